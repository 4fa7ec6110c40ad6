"""Config 3's field split into 8 kd bricks balanced by non-empty voxel count (GPU mass function): print each
brick's cells and apron-quad count (which bricks exceed 2^31 quads and run the wide addressing)."""
import sys, json
sys.path.insert(0, "/root/repo")
import torch
from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.volume import blob_field, decompose
d = torch.device("cuda", 0)
f = blob_field((2049, 2049, 2049), seed=1)
m = dev.field_mass_function(f, d, 0.1)
dec = decompose(f, 8, "mass", m)
for r, (lo, hi) in enumerate(dec.boxes):
    n = 1
    for a in range(3): n *= hi[a] - lo[a] + 3
    print(r, lo, hi, "cells", [hi[a]-lo[a] for a in range(3)], "quad voxels %.2fG" % (n / 1e9))
