"""Ray cycling vs sort-last marching work on ONE B200 (schedule simulated serially, one brick per rank):
for each hop of the cycle, every rank's accumulate-mode march of the batch it holds is timed alone
(CUDA events); the cycle's critical path is sum over hops of the slowest rank, its total work the sum of
all marches.  Sort-last: every rank marches its whole footprint once (critical path = slowest rank).
Default TF (low opacity) and an opaque TF (early termination pays), 8 bricks of a 1025^3 field, 1920x1080."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.compositor import assign_rows
from paper_2501_01628_b200.geom import auto_camera
from paper_2501_01628_b200.volume import TransferFunction1D, blob_field, decompose, default_tf

d = torch.device("cuda", 0)
W, H, R = 1920, 1080, 8
f = blob_field((1025, 1025, 1025), seed=1)
dec = decompose(f, R)
cam = auto_camera(f.bounds(), W, H)
order = dec.visibility_order(cam.position)
pos = {s: i for i, s in enumerate(order)}
blocks = assign_rows(H, R)
bricks = [dev.DeviceBrick(dec.brick(r), d).generate(f) for r in range(R)]
x = np.linspace(0, 1, 256)
opaque = TransferFunction1D(np.column_stack([x, 1 - x, 0.5 + 0 * x, np.where(x < 0.1, 0.0, 0.6)]).astype(np.float32))


def timed(fn, reps=3):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {"R": R, "W": W, "H": H, "order": order, "cases": []}
for name, tf in (("default_tf", default_tf()), ("opaque_tf", opaque)):
    dtf = dev.DeviceTF(tf, d)
    part = torch.empty(W * H * 4, dtype=torch.float32, device=d)
    sl = [timed(lambda r=r: dev.march(bricks[r], cam, dtf, 1.0, 0.99, part, W, H)) for r in range(R)]
    # cycle: state per batch; hop k: rank at position q marches the batch of origin position (q - k) mod R
    states = {b: torch.zeros((blocks[b][1] - blocks[b][0]) * W * 8, dtype=torch.float32, device=d) for b in range(R)}
    hops = []
    for k in range(R):
        times = []
        for r in range(R):
            po = (pos[r] - k) % R
            b = order[po]
            rows = blocks[b]
            n = (rows[1] - rows[0]) * W
            seg = states[b][: n * 4] if pos[r] >= po else states[b][n * 4:]
            snap = seg.clone()

            def go(r=r, seg=seg, snap=snap, rows=rows):
                seg.copy_(snap)  # every timed repetition starts from the same accumulated state
                dev.march(bricks[r], cam, dtf, 1.0, 0.99, seg, W, H, accum=True, rows=rows)
            t_copy = timed(lambda seg=seg, snap=snap: seg.copy_(snap))
            times.append(max(timed(go) - t_copy, 0.0))
        hops.append(times)
    rec = {"tf": name, "sort_last_rank_ms": sl, "sort_last_critical_ms": max(sl), "sort_last_total_ms": sum(sl),
           "cycle_hop_ms": hops, "cycle_critical_ms": sum(max(h) for h in hops),
           "cycle_total_ms": sum(sum(h) for h in hops)}
    out["cases"].append(rec)
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in rec.items()
                      if k not in ("cycle_hop_ms", "sort_last_rank_ms")}), flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/cycle_bench.json").write_text(json.dumps(out, indent=1))
