"""How much of a single-rank frame is the march kernel's tail?  Times K fused RGB8 frames (c2) issued
(a) back to back on one stream and (b) alternating over S streams with one brick handle per stream
(each handle has its own tile counter), so frame k+1's CTAs can take the SMs frame k's finished CTAs
free.  A measurement helper, not the bench."""
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
ap.add_argument("--iters", type=int, default=40)
ap.add_argument("--streams", type=int, default=2)
args = ap.parse_args()
d = torch.device("cuda", 0)
f = blob_field((args.edge + 1,) * 3, seed=1)
dec = decompose(f, 1)
cam = auto_camera(f.bounds(), args.W, args.H)
tf = default_tf()
S = args.streams
bricks = [dev.DeviceBrick(dec.brick(0), d).generate(f) for _ in range(S)]
dtf = dev.DeviceTF(tf, d)
frames = [torch.empty(args.W * args.H * 3, dtype=torch.uint8, device=d) for _ in range(S)]
streams = [torch.cuda.Stream(d) for _ in range(S)]
bg = (0.05, 0.06, 0.08)


def one(k, multi):
    i = k % S if multi else 0
    if multi:
        with torch.cuda.stream(streams[i]):
            dev.march_rgb8(bricks[i], cam, dtf, 1.0, 0.99, bg, frames[i], args.W, args.H)
    else:
        dev.march_rgb8(bricks[0], cam, dtf, 1.0, 0.99, bg, frames[0], args.W, args.H)


def run(multi):
    main = torch.cuda.current_stream(d)
    for k in range(6):
        one(k, multi)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    if multi:
        for s in streams:
            s.wait_event(e0)
    for k in range(args.iters):
        one(k, multi)
    if multi:
        for s in streams:
            ev = torch.cuda.Event()
            ev.record(s)
            main.wait_event(ev)
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / args.iters


for rep in range(3):
    a = run(False)
    b = run(True)
    print(f"rep {rep}: one stream {a:.4f} ms/frame ({1e3 / a:.0f} fps); {S} streams {b:.4f} ms/frame "
          f"({1e3 / b:.0f} fps); gain {a / b:.3f}x")
ref = frames[0].clone()
torch.cuda.synchronize()
for i in range(1, S):
    assert torch.equal(frames[i], ref), "frames differ between streams"
print("frames identical across streams")
