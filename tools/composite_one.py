"""One 4K, 8-fragment full-frame composite (for ncu): seeded premultiplied RGBA, alpha <= 0.5."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2501_01628_b200 import device as dev

d = torch.device("cuda", 0)
W, H, P = 3840, 2160, 8
g = torch.Generator(device=d).manual_seed(1)
frags = []
for _ in range(P):
    a = torch.rand(W * H, 1, device=d, generator=g) * 0.5
    frags.append(torch.cat([torch.rand(W * H, 3, device=d, generator=g) * a, a], 1).reshape(-1).contiguous())
rgb = torch.empty(W * H * 3, dtype=torch.uint8, device=d)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    dev.composite(frags, (0.1, 0.2, 0.3), rgb8=rgb)
torch.cuda.synchronize()
print("ok")
