"""Render profiles/r01_scaling_projection.md from scaling_projection.py's JSONs (even and mass splits;
run here, no GPU)."""
import json
from pathlib import Path

P = Path(__file__).resolve().parent.parent / "profiles"


def table(d):
    L = ["| N | field | max march ms | mean march ms | max blend ms | peer MB per rank (max) | peer transfer ms | "
         "projected frame ms | projected frames/s |", "|---|---|---|---|---|---|---|---|---|"]
    for r in d["runs"]:
        mm = r["march_ms"]
        if r["N"] == 1:
            L.append(f"| 1 | {r['field']} | {max(mm):.3f} | {sum(mm) / len(mm):.3f} | — | — | — | "
                     f"{r['projected_frame_ms']:.3f} | {r['projected_fps']:.0f} |")
        else:
            L.append(f"| {r['N']} | {r['field']} | {max(mm):.3f} | {sum(mm) / len(mm):.3f} | {max(r['blend_kernel_ms']):.4f} | "
                     f"{max(r['peer_bytes_per_rank']) / 1e6:.1f} | {r['peer_transfer_ms']:.3f} | "
                     f"{r['projected_frame_ms']:.3f} | {r['projected_fps']:.0f} |")
    f1 = d["runs"][0]["projected_fps"]
    L.append("")
    L.append("Per-rank marches: " + "; ".join(f"N={r['N']}: " + ", ".join(f"{x:.3f}" for x in r["march_ms"])
                                         for r in d["runs"][1:]) + " ms.")
    L.append("Projected weak-scaling efficiency (frames/s at N over N = 1, both stream-ordered): "
             + ", ".join(f"N={r['N']}: {r['projected_fps'] / f1:.2f}" for r in d["runs"][1:]) + ".")
    return L


even = json.loads((P / "r01_scaling_projection.json").read_text())
mass = json.loads((P / "r01_scaling_projection_mass.json").read_text())
L = ["# Round 1 — bench.py's weak-scaling workloads measured rank by rank on one B200 (`tools/scaling_projection.py`)", "",
     "The field grows with N (512^3 cells per rank, doubled along x, y, z in turn), 1920x1080, default TF.  Measured",
     "(CUDA events, each rank's work alone on this GPU): every rank's march (N = 1: the fused RGB8 march; N > 1: the",
     "band-cleared RGBA partial) and every rank's blend kernel over its row block's band-clipped fragments",
     "(graph-timed).  **Projection** (not a measurement): frame = max march + 2 x 12 us barrier (assumed NCCL 4-byte",
     "all-reduce) + max(blend kernel, clipped peer bytes / 770 GB/s).  Raw: `r01_scaling_projection[_mass].json`.", "",
     "## kd split balanced by non-empty voxel count (`--decomposition mass`, bench.py's default for N > 1)", ""]
L += table(mass)
L += ["", "## even kd split (every rank 512^3 cells, `--decomposition even`)", ""]
L += table(even)
L += ["", "The slowest rank sets the frame.  With even bricks the N = 8 ranks' marches spread 0.08-0.21 ms (the 16 blobs",
      "are not spread evenly over the eight octants); the mass split (integer counts of voxels >= 0.1, the TF's",
      "alpha threshold, computed on the GPU by `device.field_mass_function`) brings the slowest N = 8 rank from",
      f"{max(even['runs'][3]['march_ms']):.3f} to {max(mass['runs'][3]['march_ms']):.3f} ms; at N = 2 the even cut happens "
      "to be the better one for this view.",
      "bench.py's N = 1 line runs two frames in flight (DESIGN.md §4.3c: ~4640 frames/s measured), which this",
      "stream-ordered projection does not include; the N > 1 step is stream-ordered (pipelining it needs the march",
      "to leave SMs to the exchange's kernels), so a driver-computed efficiency against the N = 1 line reads lower."]
(P / "r01_scaling_projection.md").write_text("\n".join(L) + "\n")
