import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import oracle
import test_gpu_fuzz as t
from paper_2501_01628_b200 import device as dev
from scenes import oracle_partials
d = torch.device("cuda", 0)
for seed in (3828, 4627):
    f, dec, cam, tf, dt, ert, W, H, bg = t._random_case(seed)
    vox = oracle.generate_field(f.dims, f.blobs)
    for e in (ert, 1.0):
        ref, _ = oracle_partials(vox, dec, cam, tf, dt, e, W, H)
        dtf = dev.DeviceTF(tf, d)
        worst = 0
        for r in range(dec.P):
            b = dev.DeviceBrick(dec.brick(r), d).generate(f)
            p = torch.empty(H * W * 4, dtype=torch.float32, device=d)
            dev.march(b, cam, dtf, dt, e, p, W, H)
            torch.cuda.synchronize(); b.close()
            got = p.view(H, W, 4).cpu().numpy().astype(np.float64)
            err = np.abs(got - ref[r]).max(axis=2)
            i = np.unravel_index(np.argmax(err), err.shape)
            if err.max() > worst:
                worst = err.max(); info = (r, i, got[i], ref[r][i])
        print(seed, "ert", e, "max err %.3e" % worst, "brick/pixel", info[0], info[1], "gpu A %.6f oracle A %.6f" % (info[2][3], info[3][3]))
