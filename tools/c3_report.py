"""Render profiles/r01_c3_per_rank.md from c3_rank_bench.py JSONs -- the even 2x2x2 split and the split
balanced by non-empty voxel count (run here, no GPU).

    python tools/c3_report.py [even.json] [mass.json] [history]
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2501_01628_b200 import device as dev  # noqa: E402
from paper_2501_01628_b200.compositor import assign_rows, clip_rows  # noqa: E402
from paper_2501_01628_b200.geom import auto_camera  # noqa: E402
from paper_2501_01628_b200.volume import BrickDesc, blob_field  # noqa: E402

even_src = Path(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_c3_ranks_beam.json")
mass_src = Path(sys.argv[2] if len(sys.argv) > 2 else "profiles/r01_c3_ranks_mass.json")
hist = sys.argv[3] if len(sys.argv) > 3 else ""
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
PEER = 770e9


def section(d, src, title, note):
    L = [f"## {title}", "", note + f"  Raw numbers: `{src.name}`.", "",
         "| rank | cells lo..hi | stored voxels | footprint px | march ms | §8(d) GB/s | frac |", "|---|---|---|---|---|---|---|"]
    f = blob_field(tuple(d["field"]), seed=1)
    cam = auto_camera(f.bounds(), d["W"], d["H"])
    bands = []
    for r in d["ranks"]:
        lo, hi = r["box"]
        desc = BrickDesc(f.dims, tuple(lo), tuple(hi), 1, f.origin, f.spacing)
        sd = desc.stored_dims
        bands.append(tuple(dev.desc_footprint(desc, cam, d["W"], d["H"])[1::2]))
        L.append(f"| {r['rank']} | {lo}..{hi} | {sd[0]}x{sd[1]}x{sd[2]} | {r['footprint_px']:,} | {r['march_ms']:.3f} | "
                 f"{r['achieved_GBps']:.0f} | {r['frac_hbm']:.2f} |")
    mx = d["max_rank_march_ms"]
    blocks = assign_rows(d["H"], 8)
    clip_recv = max(sum((c[1] - c[0]) * d["W"] * 16 for s in range(8) if s != j
                        for c in [clip_rows(blocks[j], bands[s])] if c) for j in range(8))
    tot = sum(r["algorithmic_bytes"] for r in d["ranks"])
    mean = sum(r["march_ms"] for r in d["ranks"]) / len(d["ranks"])
    ex = (d["exchange_bytes_per_rank"] + d["rgb8_into_root_bytes"]) / PEER * 1e3
    exc = (clip_recv + d["rgb8_into_root_bytes"] / 7) / PEER * 1e3
    L += ["", f"Visibility order (front to back): {d['order']}.  Slowest rank: {mx:.3f} ms (mean {mean:.3f}, "
              f"imbalance {mx / mean:.2f}).",
          f"Frame-level march roofline with 8 GPUs: {tot / 1e9:.2f} GB algorithmic / (8 x {mx:.3f} ms) = "
          f"{tot / 8 / mx / 1e6:.0f} GB/s per GPU = **{tot / 8 / mx / 1e6 / peak:.2f}** of the measured {peak:.0f} GB/s "
          "HBM peak (north star: >= 0.60" + ("; above 1 because exact skipping never reads empty macrocells)."
                                              if tot / 8 / mx / 1e6 / peak > 1 else ")."),
          f"Projected 8-GPU frame (a projection, not a measurement): slowest march + exchange at the {PEER / 1e9:.0f} GB/s "
          f"peer bandwidth of B200_PROFILING.md + one rank's blend ({d['composite_rank_ms'] * 1e3:.1f} us) ~= "
          f"{mx + ex + d['composite_rank_ms']:.2f} ms with the full exchange ({d['exchange_bytes_per_rank'] / 1e6:.1f} MB "
          f"per rank), {mx + exc + d['composite_rank_ms']:.2f} ms (~{1e3 / (mx + exc + d['composite_rank_ms']):.0f} frames/s) "
          f"with the band-clipped exchange (at most {clip_recv / 1e6:.1f} MB per rank).", ""]
    return L


L = ["# Round 1 — config 3 per-rank work on one B200 (`tools/c3_rank_bench.py`)", "",
     "2048^3 blob field (seed 1), 8 kd bricks (+1 ghost voxel), 3840x2160, auto camera, dt = 1 voxel, ERT 0.99,",
     "default TF.  Each rank's `dprt_march` (RGBA partial) timed alone with CUDA events (10 launches after 3",
     "warm-up).  `frac` uses the SURVEY §8(d) algorithmic bytes (whole brick + 16 B x footprint + TF) over the",
     "measured HBM peak: exact empty-space skipping never reads a brick's empty macrocells, so `frac` > 1 on",
     "light bricks means the whole-brick byte count is not what the kernel streams; the slowest rank sets the",
     "frame.  ncu of the slowest even brick: `r01_c3r5_ncu.txt` (5.36 TB/s of DRAM traffic, 0.82 of the peak).", ""]
even = json.loads(even_src.read_text())
L += section(even, even_src, "even split (2x2x2 bricks of 1024^3 cells)",
             "SURVEY §8(a6)'s plan for config 3." + (f"  History of the slowest rank: {hist}." if hist else ""))
if mass_src.exists():
    mass = json.loads(mass_src.read_text())
    L += section(mass, mass_src, "split balanced by non-empty voxel count (`decompose(..., \"mass\")`)",
                 "The kd cuts fall where the integer count of voxels >= 0.1 (the default TF's alpha threshold; "
                 "`device.field_mass_function`, on the GPU) balances; the largest brick then holds more than 2^31 "
                 "apron quads and marches with 64-bit z-plane offsets (`march_beam_kernel<true>`).")
half_note = ROOT / "profiles" / "r01_c3_half_quads.md"  # the opt-in fp16-quad numbers, kept alongside
if half_note.exists():
    L += ["", half_note.read_text().strip()]
(ROOT / "profiles" / "r01_c3_per_rank.md").write_text("\n".join(L) + "\n")
print("\n".join(L))
