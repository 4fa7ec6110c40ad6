"""March one brick of a bench workload a few times (an ncu target; nothing is printed but the timing):

    python tools/march_one.py --config c3 --strategy even --rank 5 --launches 4
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
from paper_2501_01628_b200 import device as dev

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--strategy", default="even")
ap.add_argument("--rank", type=int, default=5)
ap.add_argument("--ranks", type=int, default=8)
ap.add_argument("--launches", type=int, default=4)
a = ap.parse_args()
d = torch.device("cuda", 0)
wl = bench.build_workload(a.config, a.ranks, a.strategy, mass_device=d)
torch.cuda.empty_cache()
b = dev.DeviceBrick(wl.dec.brick(a.rank), d).generate(wl.field)
dtf = dev.DeviceTF(wl.tf, d)
p = torch.empty(wl.W * wl.H * 4, dtype=torch.float32, device=d)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(a.launches):
    if i == a.launches - 1:
        e0.record()
    dev.march(b, wl.cams[0], dtf, 1.0, 0.99, p, wl.W, wl.H)
e1.record()
torch.cuda.synchronize()
print(f"{a.config} {a.strategy} rank {a.rank}: last launch {e0.elapsed_time(e1):.3f} ms")
