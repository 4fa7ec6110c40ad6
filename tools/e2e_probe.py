"""Where the e2e frame time goes (c2, one rank): the bench's e2e loop at several step counts, plus the
GPU-side interval between consecutive frames' march launches (events on the render stream)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.engine import RenderOptions, VolumeRenderer
from paper_2501_01628_b200.transport import SoloEndpoint

d = torch.device("cuda", 0)
f, dec, cam, tf = bench.workload(1)
brick = dev.DeviceBrick(dec.brick(0), d).generate(f)
r = VolumeRenderer(SoloEndpoint(d), brick, dec, tf, bench.BACKGROUND)
opts = RenderOptions(dt=bench.DT, ert=bench.ERT)
pinned_tf = torch.from_numpy(tf.as_f32().reshape(-1)).pin_memory()
W, H = bench.W, bench.H
hosts = [torch.empty((H, W, 3), dtype=torch.uint8).pin_memory() for _ in range(3)]


def run(steps, depth, with_tf=True, events=None):
    inflight = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(steps):
        if with_tf:
            r.dtf.update(tf, staging=pinned_tf)
        if events is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            events.append(e)
        inflight.append(r.render_to_host(cam, W, H, hosts[k % (depth + 1)], opts))
        if len(inflight) > depth:
            inflight.pop(0).wait()
    while inflight:
        inflight.pop(0).wait()
    return (time.perf_counter() - t0) / steps * 1e3


run(10, 2)
for steps in (20, 100, 400):
    for depth in (1, 2):
        print(f"steps {steps:4d} depth {depth}: {run(steps, depth):.4f} ms/frame e2e")
print(f"no TF upload, 400 steps depth 2: {run(400, 2, with_tf=False):.4f} ms/frame")
ev = []
run(200, 2, events=ev)
gaps = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(len(ev) - 1))
print(f"GPU frame-start intervals: median {gaps[len(gaps) // 2]:.4f} ms, p10 {gaps[len(gaps) // 10]:.4f}, "
      f"p90 {gaps[9 * len(gaps) // 10]:.4f}")
# host cost alone: issue without waiting (GPU queue fills), 50 frames
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(50):
    r.dtf.update(tf, staging=pinned_tf)
    r.render_to_host(cam, W, H, hosts[k % 3], opts)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host issue cost: {(t1 - t0) / 50 * 1e3:.4f} ms/frame; device drain {(time.perf_counter() - t0) / 50 * 1e3:.4f} ms/frame")
