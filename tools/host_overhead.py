"""Host-side cost per frame of the public render call (cProfile over 300 render_to_host calls, c2)."""
import cProfile
import pstats
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
opts = RenderOptions()
pinned_tf = torch.from_numpy(tf.as_f32().reshape(-1)).pin_memory()
hosts = [torch.empty((bench.H, bench.W, 3), dtype=torch.uint8).pin_memory() for _ in range(2)]
for k in range(10):
    r.dtf.update(tf, staging=pinned_tf)
    r.render_to_host(cam, bench.W, bench.H, hosts[k % 2], opts).wait()
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
prev = None
for k in range(300):
    r.dtf.update(tf, staging=pinned_tf)
    hf = r.render_to_host(cam, bench.W, bench.H, hosts[k % 2], opts)
    if prev is not None:
        prev.wait()
    prev = hf
prev.wait()
pr.disable()
print(f"{(time.perf_counter() - t0) / 300 * 1e3:.3f} ms per frame (profiled)")
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
