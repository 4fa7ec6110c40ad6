"""March time vs view direction (orbit around the field centre) on config 2's 512^3 brick at 1080p."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.geom import orbit_camera
from paper_2501_01628_b200.volume import blob_field, decompose, default_tf

W, H = 1920, 1080
d = torch.device("cuda", 0)
f = blob_field((513, 513, 513), seed=1)
dec = decompose(f, 1)
b = dev.DeviceBrick(dec.brick(0), d).generate(f)
dtf = dev.DeviceTF(default_tf(), d)
p = torch.empty(W * H * 4, dtype=torch.float32, device=d)
bb = f.bounds()
for yaw in (0, 30, 45, 60, 90, 135, 180, 270):
    for pitch in (20,):
        cam = orbit_camera(bb.center(), 1.35 * bb.diagonal(), math.radians(yaw), math.radians(pitch), 45.0, W / H)
        for _ in range(3):
            dev.march(b, cam, dtf, 1.0, 0.99, p, W, H)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            dev.march(b, cam, dtf, 1.0, 0.99, p, W, H)
        e1.record()
        torch.cuda.synchronize()
        vd = cam.view_dir
        print(f"yaw {yaw:3d} pitch {pitch}: dir ({vd[0]:+.2f},{vd[1]:+.2f},{vd[2]:+.2f}) march {e0.elapsed_time(e1) / 10:.3f} ms")
