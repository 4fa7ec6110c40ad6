"""Config-5 style compositing sweep on ONE GPU: the blend+tone-map kernel each rank runs after the
exchange (P fragments of its row block) and the whole-frame blend, at 1080p / 4K / 8K and P = 2, 4, 8.
HBM GB/s = (16 B x P fragments + 3 B RGB8 [+16 B RGBA]) per pixel / kernel time.  NVLink transfer time
is not measurable on one GPU; the algorithmic exchange bytes per rank are printed for reference."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2501_01628_b200 import device as dev

d = torch.device("cuda", 0)
peak = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else 6650.0
out = []
for (W, H) in ((1920, 1080), (3840, 2160), (7680, 4320)):
    for P in (2, 4, 8):
        npix = W * H
        g = torch.Generator(device=d).manual_seed(P)
        frags = []
        for r in range(P):
            a = torch.rand(npix, 1, device=d, generator=g) * 0.5
            frags.append(torch.cat([torch.rand(npix, 3, device=d, generator=g) * a, a], 1).reshape(-1).contiguous())
        rows = H // P
        blk = [f[: rows * W * 4] for f in frags]  # one rank's row block of every fragment
        rgb = torch.empty(npix * 3, dtype=torch.uint8, device=d)
        res = {"W": W, "H": H, "P": P}
        for name, fr, n in (("rank_block", blk, rows * W), ("full_frame", frags, npix)):
            o = rgb[: n * 3]
            for _ in range(3):
                dev.composite(fr, (0.1, 0.1, 0.1), rgb8=o)
            # the launches are captured in a CUDA graph: a small tile's kernel is shorter than one
            # Python-side launch, so back-to-back host launches would time the host, not the kernel
            it = 20
            s_ = torch.cuda.Stream()
            s_.wait_stream(torch.cuda.current_stream())
            g_ = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_, stream=s_):
                for _ in range(it):
                    dev.composite(fr, (0.1, 0.1, 0.1), rgb8=o)
            g_.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            g_.replay()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / it
            nbytes = n * (16 * P + 3)
            res[name] = {"ms": ms, "GBps": nbytes / ms / 1e6, "frac_hbm": nbytes / ms / 1e6 / peak}
        res["exchange_bytes_per_rank"] = int((1 - 1 / P) * npix * 16)
        res["rgb8_into_root"] = int((P - 1) / P * npix * 3)
        out.append(res)
        print(json.dumps(res))
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/composite_sweep.json").write_text(json.dumps(out, indent=1))
