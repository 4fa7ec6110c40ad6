"""Measured RGBA error of the opt-in fp16 quads against the oracle over the randomized sweep's scenes, next
to the f32 quads' error and the stated bound (test_gpu_fuzz.half_quad_bound).  (GPU helper.)"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch

import oracle
import test_gpu_fuzz as tf_fuzz
from paper_2501_01628_b200 import device as dev
from scenes import ert_edge_pixels, oracle_partials

d = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
worst = {False: 0.0, True: 0.0}
ratio = 0.0
for seed in range(n):
    f, dec, cam, tf, dt, ert, W, H, bg = tf_fuzz._random_case(seed)
    vox = oracle.generate_field(f.dims, f.blobs)
    ref, _ = oracle_partials(vox, dec, cam, tf, dt, ert, W, H)
    dtf = dev.DeviceTF(tf, d)
    bound = tf_fuzz.half_quad_bound(tf)
    for half in (False, True):
        for r in range(dec.P):
            b = dev.DeviceBrick(dec.brick(r), d, half_quads=half).generate(f)
            p = torch.empty(H * W * 4, dtype=torch.float32, device=d)
            dev.march(b, cam, dtf, dt, ert, p, W, H)
            torch.cuda.synchronize()
            b.close()
            got = p.view(H, W, 4).cpu().numpy().astype(np.float64)
            err = np.abs(got - ref[r]).max(axis=2)
            edge = ert_edge_pixels(got[..., 3], ref[r][..., 3], ert, eps=1e-2)
            e = float(err[~edge].max(initial=0))
            worst[half] = max(worst[half], e)
            if half:
                ratio = max(ratio, e / bound)
print(f"{n} scenes: max |dRGBA| off ERT edges: f32 quads {worst[False]:.3e}, fp16 quads {worst[True]:.3e}; "
      f"worst fp16 error / stated bound = {ratio:.3f}")
