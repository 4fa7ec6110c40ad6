"""Config 4 on one B200: a lander-like anisotropic field (1536x768x384 voxels, spacing (1,1,2), lopsided
16-blob mixture), 8 UNEVEN bricks from the mass-balanced kd split, and an orbiting camera (36 frames,
10 deg yaw steps, 20 deg pitch; the viewer's orbit parametrisation).  Per frame: every
rank's march timed alone (the 8 ranks share this GPU, one after another), the visibility order checked
against the oracle's independent kd order, and on every 6th frame every brick's per-pixel sample
ownership checked integer-exactly against the oracle.  Reports per-frame max / mean rank time (the
sort-last load imbalance) and writes gpurun_out/c4_orbit.json."""
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch

import oracle
from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.geom import orbit_camera
from paper_2501_01628_b200.volume import BrickDesc, blob_field, decompose, default_tf
from scenes import cam_array, oracle_brick

W, H = 1920, 1080
d = torch.device("cuda", 0)
f = blob_field((1536, 768, 384), seed=7, spacing=(1.0, 1.0, 2.0), lopsided=True)
whole = dev.DeviceBrick(BrickDesc.whole(f, 0), d).generate(f)
mask = torch.from_numpy(whole.download() >= np.float32(0.1))
whole.close()


def mass(axis, lo, hi):
    sub = mask[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
    return sub.sum(dim=tuple(a for a in range(3) if a != 2 - axis)).to(torch.int64).numpy()


dec = decompose(f, 8, "mass", mass)
_, nodes = oracle.kd_leaves(f.dims, f.spacing, 8, "mass", field=mask.numpy().astype(np.float32))
tf = default_tf()
dtf = dev.DeviceTF(tf, d)
bricks = [dev.DeviceBrick(dec.brick(r), d).generate(f) for r in range(8)]
part = torch.empty(W * H * 4, dtype=torch.float32, device=d)
samp = torch.empty(W * H, dtype=torch.int32, device=d)
bb = f.bounds()
out = {"field": list(f.dims), "spacing": list(f.spacing), "bricks": dec.boxes,
       "brick_cells": [int(np.prod([h - l for l, h in zip(lo, hi)])) for lo, hi in dec.boxes], "frames": []}
for i in range(36):
    cam = orbit_camera(bb.center(), 1.2 * bb.diagonal(), math.radians(10.0 * i), math.radians(20.0), 45.0, W / H)
    order = dec.visibility_order(cam.position)
    assert order == oracle.kd_order(nodes, 8, cam.position, f.origin, f.spacing), f"frame {i}: order"
    times = []
    exact = None
    for r in range(8):
        for _ in range(2):
            dev.march(bricks[r], cam, dtf, 1.0, 0.99, part, W, H)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            dev.march(bricks[r], cam, dtf, 1.0, 0.99, part, W, H)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 5)
        if i % 6 == 0:
            dev.march(bricks[r], cam, dtf, 1.0, 0.99, part, W, H, samples=samp)
            got = samp.view(H, W).cpu().numpy().astype(np.uint32)
            want = oracle.sample_counts(oracle_brick(dec, r), cam_array(cam), 1.0, W, H)
            ok = bool(np.array_equal(got, want))
            assert ok, f"frame {i} brick {r}: ownership"
            exact = (exact is None or exact) and ok
    rec = {"frame": i, "order": order, "rank_ms": times, "max_ms": max(times), "mean_ms": sum(times) / 8,
           "ownership_exact": exact}
    out["frames"].append(rec)
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in rec.items() if k != "rank_ms"}),
          flush=True)
mx = [r["max_ms"] for r in out["frames"]]
mean = [r["mean_ms"] for r in out["frames"]]
out["summary"] = {"max_rank_ms_mean": sum(mx) / len(mx), "imbalance_mean": sum(a / b for a, b in zip(mx, mean)) / len(mx)}
print(json.dumps(out["summary"]))
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/c4_orbit.json").write_text(json.dumps(out, indent=1))
