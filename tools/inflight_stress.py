"""Stress the frames-in-flight hazards: a long random sequence of camera moves, TF
switches (staged and plain) and brick rewrites rendered with 2 and 3 frames in flight must give exactly the
bytes of the stream-ordered render of the same sequence.  (GPU helper; tests/test_gpu_inflight.py is the
short committed version.)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
import torch

from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.engine import RenderOptions, VolumeRenderer
from paper_2501_01628_b200.geom import orbit_camera
from paper_2501_01628_b200.transport import SoloEndpoint
from paper_2501_01628_b200.volume import blob_field, decompose, default_tf
from scenes import dense_tf

d = torch.device("cuda", 0)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(11)
f = blob_field((193, 161, 129), seed=4)
W, H = 480, 360
b = f.bounds()
tfs = [default_tf(), dense_tf(), default_tf(threshold=0.3), dense_tf(64)]
script = []
for k in range(N):
    cam = orbit_camera(b.center(), b.diagonal() * rng.uniform(0.9, 2.0), rng.uniform(0, 6.28), rng.uniform(-1, 1),
                       40.0, W / H)
    script.append((cam, int(rng.integers(0, len(tfs))), bool(rng.random() < 0.5),
                   int(rng.integers(1, 50)) if rng.random() < 0.05 else None, bool(rng.random() < 0.1)))


def run(n):
    dec = decompose(f, 1)
    brick = dev.DeviceBrick(dec.brick(0), d).generate(f)
    r = VolumeRenderer(SoloEndpoint(d), brick, dec, tfs[0], (0.05, 0.06, 0.08))
    opts = RenderOptions(frames_in_flight=n)
    hosts = [torch.empty((H, W, 3), dtype=torch.uint8).pin_memory() for _ in range(N)]
    pending = []
    for k, (cam, ti, staged, seed, device_read) in enumerate(script):
        if seed is not None:
            brick.generate(blob_field(f.dims, seed=seed))
        tf = tfs[ti]
        if staged:
            r.dtf.update(tf, staging=torch.from_numpy(tf.as_f32().reshape(-1).copy()).pin_memory())
        else:
            r.dtf.update(tf)
        r.tf = tf
        if device_read:  # a device-side consumer of the frame instead of the read-back
            res = r.render(cam, W, H, opts, verify=False)
            res.wait_ready()
            hosts[k].copy_(res.rgb8.cpu())
            pending.append(None)
        else:
            pending.append(r.render_to_host(cam, W, H, hosts[k], opts, verify=False))
    for hf in pending:
        if hf is not None:
            hf.wait()
    r.join()
    torch.cuda.synchronize()
    brick.close()
    return [h.numpy().copy() for h in hosts]


want = run(1)
for n in (2, 3):
    got = run(n)
    bad = [k for k in range(N) if not np.array_equal(got[k], want[k])]
    print(f"frames in flight {n}: {N - len(bad)}/{N} frames byte-identical" + (f"; differ: {bad[:10]}" if bad else ""))
