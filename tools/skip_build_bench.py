"""Cost of the TF-dependent skip-distance rebuild on the c2 brick and one config-3 brick: march time with a
fresh TF version every launch (rebuild + march) minus the march alone (CUDA events).

    python tools/skip_build_bench.py
"""
import itertools
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
from paper_2501_01628_b200 import device as dev

d = torch.device("cuda", 0)
out = {}
for cfg, R, rank in (("c2", 1, 0), ("c3", 8, 5)):
    wl = bench.build_workload(cfg, R, "even")
    b = dev.DeviceBrick(wl.dec.brick(rank), d).generate(wl.field)
    dtf = dev.DeviceTF(wl.tf, d)
    part = torch.empty(wl.W * wl.H * 4, dtype=torch.float32, device=d)
    cam = wl.cams[0]
    versions = itertools.count(10 ** 6)

    def run(fresh, n=10):
        for _ in range(2):
            dev.march(b, cam, dtf, 1.0, 0.99, part, wl.W, wl.H)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            if fresh:
                dtf.version = next(versions)  # same table, new tag: the brick rebuilds its skip distances
            dev.march(b, cam, dtf, 1.0, 0.99, part, wl.W, wl.H)
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / n

    m, r = run(False), run(True)
    out[cfg] = {"march_ms": m, "march_with_rebuild_ms": r, "rebuild_ms": r - m}
    b.close()
    torch.cuda.empty_cache()
print(json.dumps(out))
