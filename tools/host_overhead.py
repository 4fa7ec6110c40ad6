"""Host-side cost per frame of the public calls (config 2): the time the host spends issuing a frame, measured
while the GPU is busy (no synchronisation inside the loop, so the host never waits for the device):

* ``dev.march_rgb8``  -- the ctypes call into dprt_march_rgb8 (argument packing, device bind, launch);
* ``VolumeRenderer.render``  -- the engine's frame (frames in flight, no digest at one rank);
* ``VolumeRenderer.render_to_host``  -- plus the read-back enqueue;
and a cProfile of the last one.  Writes gpurun_out/host_overhead.json."""
import cProfile
import json
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch

import bench
from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.engine import RenderOptions, VolumeRenderer
from paper_2501_01628_b200.transport import SoloEndpoint

d = torch.device("cuda", 0)
wl = bench.build_workload("c2", 1, "even")
cam, W, H = wl.cams[0], wl.W, wl.H
brick = dev.DeviceBrick(wl.dec.brick(0), d).generate(wl.field)
r = VolumeRenderer(SoloEndpoint(d), brick, wl.dec, wl.tf, bench.BACKGROUND)
opts = RenderOptions(frames_in_flight=2)
frame8 = torch.empty(W * H * 3, dtype=torch.uint8, device=d)
hosts = [torch.empty((H, W, 3), dtype=torch.uint8).pin_memory() for _ in range(3)]
out = {}


def per_call_us(fn, n=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    host = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    return host


out["march_rgb8_call_us"] = per_call_us(lambda: dev.march_rgb8(brick, cam, r.dtf, 1.0, 0.99, bench.BACKGROUND, frame8, W, H))
out["render_call_us"] = per_call_us(lambda: r.render(cam, W, H, opts, verify=False))
pending = []


def to_host():
    pending.append(r.render_to_host(cam, W, H, hosts[len(pending) % 3], opts))
    if len(pending) > 2:
        pending.pop(0)  # dropped, not waited: the host does not block on the device here


out["render_to_host_call_us"] = per_call_us(to_host)
out["gpu_frame_ms_for_scale"] = 0.23
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    to_host()
pr.disable()
torch.cuda.synchronize()
print(json.dumps(out))
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "host_overhead.json").write_text(json.dumps(out, indent=1))
