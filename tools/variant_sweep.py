"""Kernel-variant sweep on one B200: each libdprt_cuda.so variant (tools/build_variant.py) timed in its own
process on config 2 (dprt_march_rgb8, the bench step's launch) and on config 3's slowest bricks (RGBA
partial march: even rank 5, mass-balanced rank 7), CUDA events, same box.

    python tools/variant_sweep.py base.so other.so ...   (paths relative to tools/variants/ or absolute)
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

CHILD = r'''
import json, sys, torch
sys.path.insert(0, %r)
import bench
from paper_2501_01628_b200 import device as dev
d = torch.device("cuda", 0)
out = {}
def timed(fn, n):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / n
wl = bench.build_workload("c2", 1, "even")
br = dev.DeviceBrick(wl.dec.brick(0), d).generate(wl.field)
dtf = dev.DeviceTF(wl.tf, d)
fr = torch.empty(wl.W * wl.H * 3, dtype=torch.uint8, device=d)
out["c2"] = min(timed(lambda: dev.march_rgb8(br, wl.cams[0], dtf, 1.0, 0.99, (0.05, 0.06, 0.08), fr, wl.W, wl.H), 100) for _ in range(3))
br.close(); del br; torch.cuda.empty_cache()
import os
ALL = os.environ.get("SWEEP_ALL_RANKS") == "1"
for strat, rank in (("even", 5), ("mass", 7)):
    wl = bench.build_workload("c3", 8, strat, mass_device=d)
    torch.cuda.empty_cache()
    part = torch.empty(wl.W * wl.H * 4, dtype=torch.float32, device=d)
    per = {}
    for r in (range(8) if ALL else [rank]):
        br = dev.DeviceBrick(wl.dec.brick(r), d).generate(wl.field)
        per[r] = min(timed(lambda: dev.march(br, wl.cams[0], dtf, 1.0, 0.99, part, wl.W, wl.H), 20) for _ in range(2))
        br.close(); del br; torch.cuda.empty_cache()
    if ALL:  # the 8-GPU frame's march critical path and every rank
        out[f"c3_{strat}_max"] = max(per.values())
        out[f"c3_{strat}_ranks"] = [round(per[r], 4) for r in range(8)]
    else:
        out[f"c3_{strat}_r{rank}"] = per[rank]
    del part; torch.cuda.empty_cache()
print("RESULT " + json.dumps(out))
''' % str(ROOT)

res = {}
for v in sys.argv[1:]:
    path = Path(v) if Path(v).is_absolute() else ROOT / "tools" / "variants" / v
    env = dict(os.environ, DPRT_CUDA_LIB=str(path))
    p = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True, env=env)
    line = [ln for ln in p.stdout.splitlines() if ln.startswith("RESULT ")]
    res[path.name] = json.loads(line[0][7:]) if line else {"error": p.stderr[-800:]}
    print(path.name, json.dumps(res[path.name]), flush=True)
Path(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "variant_sweep.json").write_text(json.dumps(res, indent=1))
