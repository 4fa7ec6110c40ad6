"""Host time to issue one e2e frame (TF staging + render_to_host with two frames in flight, c2) vs the
time spent waiting for frame k-2's bytes: is the end-to-end loop host-bound?  (Measurement helper.)"""
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
opts = RenderOptions(frames_in_flight=2)
pinned_tf = torch.from_numpy(tf.as_f32().reshape(-1)).pin_memory()
hosts = [torch.empty((bench.H, bench.W, 3), dtype=torch.uint8).pin_memory() for _ in range(3)]
inflight = []
issue, wait = [], []
for k in range(400):
    t0 = time.perf_counter()
    r.dtf.update(tf, staging=pinned_tf)
    hf = r.render_to_host(cam, bench.W, bench.H, hosts[k % 3], opts, verify=True)
    t1 = time.perf_counter()
    inflight.append(hf)
    if len(inflight) > 2:
        inflight.pop(0).wait()
    t2 = time.perf_counter()
    if k >= 50:
        issue.append(t1 - t0)
        wait.append(t2 - t1)
for hf in inflight:
    hf.wait()
n = len(issue)
print(f"per frame: host issue {sum(issue) / n * 1e6:.1f} us, wait {sum(wait) / n * 1e6:.1f} us, "
      f"total {(sum(issue) + sum(wait)) / n * 1e6:.1f} us")
