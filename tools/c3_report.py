"""Render profiles/r01_c3_per_rank.md from a c3_rank_bench.py JSON (run here, no GPU)."""
import json
import sys
from pathlib import Path

src = Path(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_c3_ranks_beam.json")
d = json.loads(src.read_text())
peak = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
hist = sys.argv[2] if len(sys.argv) > 2 else ""
L = ["# Round 1 — config 3 per-rank work on one B200 (`tools/c3_rank_bench.py`)", "",
     "2048^3 blob field (seed 1), kd split into 8 bricks of 1024^3 cells (+1 ghost: 1026^3 voxels, 4.33 GB f32),",
     "3840x2160, auto camera, dt = 1 voxel, ERT 0.99, default TF.  Each rank's `dprt_march` timed alone with CUDA",
     "events (10 launches after 3 warm-up).  `frac` uses the SURVEY §8(d) algorithmic bytes (whole brick + 16 B x",
     "footprint + TF) over the measured HBM peak: with exact empty-space skipping a brick's empty macrocells",
     "are never read, so `frac` > 1 on light bricks means the whole-brick byte count is not what the kernel",
     f"streams; the heavy bricks set the frame time.  Raw numbers: `{src.name}`.", "",
     "| rank | cells lo..hi | footprint px | march ms | §8(d) GB/s | frac |", "|---|---|---|---|---|---|"]
for r in d["ranks"]:
    lo, hi = r["box"]
    L.append(f"| {r['rank']} | {lo}..{hi} | {r['footprint_px']:,} | {r['march_ms']:.3f} | {r['achieved_GBps']:.0f} | "
             f"{r['frac_hbm']:.2f} |")
mx = d["max_rank_march_ms"]
# band-clipped exchange: every brick's footprint rows, host geometry only
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_01628_b200 import device as dev  # noqa: E402
from paper_2501_01628_b200.compositor import assign_rows, clip_rows  # noqa: E402
from paper_2501_01628_b200.geom import auto_camera  # noqa: E402
from paper_2501_01628_b200.volume import blob_field, decompose  # noqa: E402

_f = blob_field(tuple(d["field"]), seed=1)
_dec = decompose(_f, 8)
_cam = auto_camera(_f.bounds(), d["W"], d["H"])
_bands = [tuple(dev.desc_footprint(_dec.brick(s), _cam, d["W"], d["H"])[1::2]) for s in range(8)]
_blocks = assign_rows(d["H"], 8)
clip_recv = max(sum((c[1] - c[0]) * d["W"] * 16 for s in range(8) if s != j
                    for c in [clip_rows(_blocks[j], _bands[s])] if c) for j in range(8))
tot = sum(r["algorithmic_bytes"] for r in d["ranks"])
ex = (d["exchange_bytes_per_rank"] + d["rgb8_into_root_bytes"]) / 770e9 * 1e3
fr = mx + ex + d["composite_rank_ms"]
L += ["", f"Visibility order (front to back): {d['order']}.  Slowest rank: {mx:.3f} ms{hist}.",
      f"Frame-level march roofline with 8 GPUs: {tot / 1e9:.2f} GB algorithmic / (8 x {mx:.3f} ms) = "
      f"{tot / 8 / mx / 1e6:.0f} GB/s per GPU = **{tot / 8 / mx / 1e6 / peak:.2f}** of the measured {peak:.0f} GB/s "
      "HBM peak (north star: >= 0.60).",
      f"One rank's compositing kernel (8 fragments of its 270-row block, 4K): {d['composite_rank_ms'] * 1e3:.1f} us.",
      f"Exchange per rank (not measurable on one GPU): {d['exchange_bytes_per_rank'] / 1e6:.1f} MB of RGBA f32 "
      f"fragments, {d['rgb8_into_root_bytes'] / 1e6:.1f} MB of RGB8 tiles into rank 0 -> ~{ex:.3f} ms at the 770 GB/s",
      "peer bandwidth of B200_PROFILING.md.  Projected 8-GPU frame ~= slowest march + exchange + composite",
      f"~= {fr:.2f} ms (~{1e3 / fr:.0f} frames/s; a projection, not a measurement).",
      f"With the band-clipped exchange (each brick's footprint rows only) the most any rank reads is "
      f"{clip_recv / 1e6:.1f} MB -> ~{(clip_recv + d['rgb8_into_root_bytes'] / 7) / 770e9 * 1e3:.3f} ms, projected frame "
      f"~= {mx + (clip_recv + d['rgb8_into_root_bytes'] / 7) / 770e9 * 1e3 + d['composite_rank_ms']:.2f} ms."]
Path("profiles/r01_c3_per_rank.md").write_text("\n".join(L) + "\n")
print("\n".join(L[-7:]))
