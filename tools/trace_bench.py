"""Time the triangle traversal leg of bench.py (dprt_trace_nearest vs the reference's numba slot) with the
library selected by DPRT_CUDA_LIB (kernel variants from tools/build_variant.py)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench

d = torch.device("cuda", 0)
for n_tri in (int(a) for a in (sys.argv[1:] or ["200000"])):
    print(json.dumps(bench.triangle_trace_leg(d, n_tri=n_tri)), flush=True)
