"""Time dprt_march alone on config c2 (or a given edge/size) -- a kernel-iteration helper, not the bench."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.geom import auto_camera
from paper_2501_01628_b200.volume import blob_field, decompose, default_tf

ap = argparse.ArgumentParser()
ap.add_argument("--edge", type=int, default=512)
ap.add_argument("--W", type=int, default=1920)
ap.add_argument("--H", type=int, default=1080)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--no-skip", action="store_true")
ap.add_argument("--threshold", type=float, default=0.1)
ap.add_argument("--field", choices=["blobs", "ml"], default="blobs")
ap.add_argument("--rgb8", action="store_true", help="time dprt_march_rgb8 (the single-rank bench step)")
ap.add_argument("--wide", action="store_true", help="RGBA march forced onto the wide-brick addressing")
ap.add_argument("--half-quads", action="store_true", help="opt-in fp16 coefficient quads")
args = ap.parse_args()
d = torch.device("cuda", 0)
if args.field == "ml":
    from paper_2501_01628_b200.volume import marschner_lobb_field

    f = marschner_lobb_field((args.edge + 1,) * 3)
else:
    f = blob_field((args.edge + 1,) * 3, seed=1)
dec = decompose(f, 1)
cam = auto_camera(f.bounds(), args.W, args.H)
tf = default_tf(threshold=args.threshold)
b = dev.DeviceBrick(dec.brick(0), d, half_quads=args.half_quads).generate(f)
dtf = dev.DeviceTF(tf, d)
p = torch.empty(args.W * args.H * 4, dtype=torch.float32, device=d)
s = torch.empty(args.W * args.H, dtype=torch.int32, device=d)
dev.march(b, cam, dtf, 1.0, 0.99, p, args.W, args.H, samples=s, skip=not args.no_skip)
torch.cuda.synchronize()
owned = int(s.sum().item())
hit = int((s > 0).sum().item())
frame = torch.empty(args.W * args.H * 3, dtype=torch.uint8, device=d)


def step():
    if args.rgb8:
        dev.march_rgb8(b, cam, dtf, 1.0, 0.99, (0.05, 0.06, 0.08), frame, args.W, args.H, skip=not args.no_skip)
    else:
        dev.march(b, cam, dtf, 1.0, 0.99, p, args.W, args.H, skip=not args.no_skip, force_wide=args.wide)


for _ in range(3):
    step()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(args.iters):
    step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / args.iters
a = p.view(-1, 4)[:, 3]
print(f"edge {args.edge} {args.W}x{args.H} skip={not args.no_skip}: march {ms:.4f} ms; rays hitting brick {hit}, "
      f"owned samples {owned} ({owned / max(hit, 1):.0f}/ray); pixels A>=0.99: {int((a >= 0.99).sum())}, "
      f"A>0: {int((a > 0).sum())}; {owned / ms / 1e6:.1f} G owned samples/s")
import ctypes
from paper_2501_01628_b200 import _lib
cnt = (ctypes.c_uint64 * 4)()
_lib.check(_lib.lib().dprt_march_counters(0, cnt, 1), "counters")
if any(cnt):
    launches = args.iters + 4
    print("per frame: shaded samples %.1fM, contributing %.1fM, skip steps %.1fM, rays %.0fK" %
          tuple(v / launches / s for v, s in zip(cnt, (1e6, 1e6, 1e6, 1e3))))
