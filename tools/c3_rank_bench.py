"""Config 3's per-GPU work measured on ONE B200: each of the 8 ranks' 1024^3-cell bricks of the 2048^3
blob field marched at 3840x2160 (dprt_march alone, CUDA events), one rank at a time, plus the rank's
compositing kernel (8 fragments of its 270-row block).  The NVLink exchange cannot run on one GPU; its
algorithmic bytes are reported.  Writes gpurun_out/c3_ranks.json."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.geom import auto_camera
from paper_2501_01628_b200.volume import blob_field, decompose, default_tf

ranks = [int(r) for r in sys.argv[1].split(",")] if len(sys.argv) > 1 and sys.argv[1] != "all" else list(range(8))
STRATEGY = sys.argv[2] if len(sys.argv) > 2 else "even"  # even: 2x2x2 bricks of 1024^3 cells; mass: balanced
HALF = len(sys.argv) > 3 and sys.argv[3] == "half"      # opt-in fp16 quads
W, H = 3840, 2160
d = torch.device("cuda", 0)
f = blob_field((2049, 2049, 2049), seed=1)
if STRATEGY == "mass":  # kd split balanced by voxels >= the TF's alpha threshold (counted on the GPU)
    dec = decompose(f, 8, "mass", dev.field_mass_function(f, d, 0.1))
    torch.cuda.empty_cache()
else:
    dec = decompose(f, 8)
cam = auto_camera(f.bounds(), W, H)
tf = default_tf()
dtf = dev.DeviceTF(tf, d)
part = torch.empty(W * H * 4, dtype=torch.float32, device=d)
peak = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
order = dec.visibility_order(cam.position)
out = {"W": W, "H": H, "field": list(f.dims), "order": order, "strategy": STRATEGY, "ranks": []}
for r in ranks:
    desc = dec.brick(r)
    t0 = time.time()
    b = dev.DeviceBrick(desc, d, half_quads=HALF).generate(f)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    for _ in range(3):
        dev.march(b, cam, dtf, 1.0, 0.99, part, W, H)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    it = 10
    e0.record()
    for _ in range(it):
        dev.march(b, cam, dtf, 1.0, 0.99, part, W, H)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    rect = b.footprint(cam, W, H)
    fp = max(0, rect[2] - rect[0]) * max(0, rect[3] - rect[1])
    alg = desc.stored_bytes + 16 * fp + 16 * tf.n
    rec = {"rank": r, "box": dec.boxes[r], "march_ms": ms, "footprint_px": fp, "algorithmic_bytes": alg,
           "achieved_GBps": alg / ms / 1e6, "frac_hbm": alg / ms / 1e6 / peak, "generate_s": gen_s}
    print(json.dumps(rec), flush=True)
    out["ranks"].append(rec)
    b.close()
    del b
    torch.cuda.empty_cache()
# one rank's compositing kernel: 8 fragments of a 270-row block
rows = H // 8
frags = [part[: rows * W * 4].clone() for _ in range(8)]
rgb = torch.empty(rows * W * 3, dtype=torch.uint8, device=d)
for _ in range(3):
    dev.composite(frags, (0.05, 0.06, 0.08), rgb8=rgb)
# graph-timed: 20 launches per replay (no Python launch overhead in the kernel time)
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for _ in range(20):
        dev.composite(frags, (0.05, 0.06, 0.08), rgb8=rgb)
g.replay()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
out["composite_rank_ms"] = e0.elapsed_time(e1) / 20
out["exchange_bytes_per_rank"] = int(7 / 8 * W * H * 16)
out["rgb8_into_root_bytes"] = int(7 / 8 * W * H * 3)
mx = max(x["march_ms"] for x in out["ranks"])
out["max_rank_march_ms"] = mx
print(json.dumps({k: v for k, v in out.items() if k != "ranks"}))
Path("gpurun_out").mkdir(exist_ok=True)
Path(f"gpurun_out/c3_ranks{'' if STRATEGY == 'even' else '_' + STRATEGY}.json").write_text(json.dumps(out, indent=1))
