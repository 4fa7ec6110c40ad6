"""bench.py's p2p_push leg alone: the fused march + exchange of one config-3 rank emulated on one GPU.

    python tools/push_bench.py [--strategy even|mass] [--rank 5]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench

ap = argparse.ArgumentParser()
ap.add_argument("--strategy", default="even")
ap.add_argument("--rank", type=int, default=5)
a = ap.parse_args()
d = torch.device("cuda", 0)
wl = bench.build_workload("c3", 8, a.strategy, mass_device=d)
torch.cuda.empty_cache()
print(json.dumps(bench.push_leg(wl, a.rank, d)))
