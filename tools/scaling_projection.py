"""bench.py's weak-scaling workloads (N = 1, 2, 4, 8: one 512^3-cell brick per GPU, 1920x1080) measured
rank by rank on ONE B200, plus a stated projection of the N-GPU frame.

Measured here (CUDA events, each rank's work alone): the march of every rank's brick (band-clipped RGBA
partial, as the multi-rank step runs it) and the p2p blend kernel of every rank's row block over its
clipped fragments (local copies stand in for the peers' buffers).  Not measurable on one GPU: the NVLink
transfer and the two stream-ordered barriers.  Projection = max march + 2 x barrier + max(blend kernel,
clipped fragment bytes / peer bandwidth), with the barrier latency and the 770 GB/s peer bandwidth
(B200_PROFILING.md) as stated assumptions.  Writes gpurun_out/scaling_projection.json."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch

import bench
from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.compositor import assign_rows, clip_rows

BARRIER_US = 12.0  # assumed NCCL 4-byte all-reduce on NVSwitch (stream-ordered device barrier)
PEER_GBS = 770.0
d = torch.device("cuda", 0)
W, H = bench.W, bench.H


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def graph_timed(fn, reps=20):
    """Kernel time of short launches: captured in a CUDA graph (Python launch overhead excluded)."""
    fn()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(reps):
            fn()
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


STRATEGY = sys.argv[1] if len(sys.argv) > 1 else "even"  # kd split of bench.py's field: even | mass
out = {"W": W, "H": H, "assumptions": {"barrier_us": BARRIER_US, "peer_GBps": PEER_GBS}, "strategy": STRATEGY,
       "runs": []}
for N in (1, 2, 4, 8):
    f, dec, cam, tf = bench.workload(N, STRATEGY, d)
    dtf = dev.DeviceTF(tf, d)
    bands = [tuple(dev.desc_footprint(dec.brick(s), cam, W, H)[1::2]) for s in range(N)]
    parts, march_ms = [], []
    for r in range(N):
        b = dev.DeviceBrick(dec.brick(r), d).generate(f)
        p = torch.zeros(W * H * 4, dtype=torch.float32, device=d)
        if N == 1:
            frame = torch.empty(W * H * 3, dtype=torch.uint8, device=d)
            march_ms.append(timed(lambda: dev.march_rgb8(b, cam, dtf, bench.DT, bench.ERT, bench.BACKGROUND, frame, W, H)))
        else:
            march_ms.append(timed(lambda: dev.march(b, cam, dtf, bench.DT, bench.ERT, p, W, H, band_clear=True)))
        parts.append(p)
        b.close()
        torch.cuda.empty_cache()
    rec = {"N": N, "field": list(f.dims), "march_ms": march_ms, "max_march_ms": max(march_ms),
           "bands": bands}
    if N > 1:
        order = dec.visibility_order(cam.position)
        blocks = assign_rows(H, N)
        blend_ms, moved = [], []
        for j in range(N):
            rows = blocks[j]
            npix = (rows[1] - rows[0]) * W
            frags, ranges, nbytes = [], [], 0
            for s in order:
                c = clip_rows(rows, bands[s])
                if c:
                    frags.append(parts[s][c[0] * W * 4: c[1] * W * 4])
                    ranges.append(((c[0] - rows[0]) * W, (c[1] - rows[0]) * W))
                    if s != j:
                        nbytes += (c[1] - c[0]) * W * 16
            tile = torch.empty(npix * 3, dtype=torch.uint8, device=d)
            blend_ms.append(graph_timed(lambda: dev.composite(frags, bench.BACKGROUND, rgb8=tile, ranges=ranges,
                                                              npix=npix)))
            moved.append(nbytes + (npix * 3 if j else 0))
        xfer_ms = max(moved) / (PEER_GBS * 1e9) * 1e3
        comp_ms = max(max(blend_ms), xfer_ms)
        frame_ms = max(march_ms) + 2 * BARRIER_US / 1e3 + comp_ms
        rec.update({"blend_kernel_ms": blend_ms, "peer_bytes_per_rank": moved, "peer_transfer_ms": xfer_ms,
                    "projected_frame_ms": frame_ms, "projected_fps": 1e3 / frame_ms})
    else:
        rec.update({"projected_frame_ms": max(march_ms), "projected_fps": 1e3 / max(march_ms)})
    out["runs"].append(rec)
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in rec.items()
                      if k in ("N", "max_march_ms", "peer_transfer_ms", "projected_frame_ms", "projected_fps")}),
          flush=True)
    del parts
    torch.cuda.empty_cache()
Path("gpurun_out").mkdir(exist_ok=True)
Path(f"gpurun_out/scaling_projection{'' if STRATEGY == 'even' else '_' + STRATEGY}.json").write_text(json.dumps(out, indent=1))
