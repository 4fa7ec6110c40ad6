"""Render a bench.py JSON line (the default N = 1 run) into a markdown summary for profiles/.

    python tools/bench_summary.py profiles/r02_bench_default.log profiles/r02_summary.md [host_overhead.json]
"""
import json
import sys

d = json.loads([ln for ln in open(sys.argv[1]) if ln.startswith("{")][-1])
out = sys.argv[2]
r = d["roofline"]
L = ["# Round 2 — measurement summary (one B200, `gpurun`)\n",
     f"Source: `python bench.py` → `{sys.argv[1].split('/')[-1]}` (the JSON line); clocks during the timed region "
     f"{d['clocks']['sm_mhz']}/{d['clocks']['sm_max_mhz']} MHz, reasons {d['clocks']['reasons']}.\n",
     "## c2 (BASELINE configs[1]: 512³ brick, 1920×1080)\n", "| key | value |", "|---|---|",
     f"| value (device frames/s, 2 in flight) | {d['value']:.0f} ({d['ms_per_step']:.4f} ms/frame) |",
     f"| e2e (render_to_host, host buffers) | {d['e2e']['value']:.0f} frames/s |",
     f"| api_e2e (Frame.render + map_frame: .array / .pixels) | {d['api_e2e']['value']:.0f} / "
     f"{d['api_e2e']['value_pixels_bytes']:.0f} frames/s |",
     f"| march kernel (events, one launch) | {r['kernel_ms']:.4f} ms |",
     f"| §8(d) bytes → frac | {r['algorithmic_bytes'] / 1e6:.1f} MB → {r['frac']:.3f} of {r['peak']} GB/s |",
     f"| needed bytes (f32 of the shaded macrocells + output + TF) → frac_needed | {r['needed_bytes'] / 1e6:.1f} MB → "
     f"{r['frac_needed']:.3f} |"]
if r.get("traffic"):
    L.append(f"| DRAM traffic (ncu child, one launch) → frac_traffic | {r['traffic'] / 1e6:.1f} MB → {r['frac_traffic']:.3f} |")
if r.get("issue_roofline"):
    L.append(f"| issue slots | {r['issue_roofline']['frac']:.3f} of {r['issue_roofline']['how']} |")
L.append(f"| shaded / contributing samples | {r['shaded_samples'] / 1e6:.2f} M / {r['contributing_samples'] / 1e6:.2f} M; "
         f"{r['shaded_samples_per_s'] / 1e9:.1f} G shaded samples/s |")
if r.get("thread_instructions_per_shaded_sample"):
    L.append(f"| instructions per shaded sample | {r['thread_instructions_per_shaded_sample']:.1f} thread, "
             f"{r['warp_instructions_per_shaded_sample']:.2f} warp |")
cpu = d.get("cpu_baseline")
if cpu:
    L.append(f"| CPU baseline (C oracle, {cpu['cores']} threads, {cpu.get('host', {}).get('cpu_model')}) | "
             f"{cpu['value']:.2f} frames/s |")
L.append("")
if "c3_per_rank" in d:
    L.append("## config 3 on one GPU (8 bricks of the 2048³ field at 3840×2160, each marched alone)\n")
    for s, c in d["c3_per_rank"].items():
        f = c["frame_roofline_per_gpu"]
        s8 = f.get("frac_survey_8d_bytes", f.get("frac"))
        L.append(f"### {s} split — slowest rank {c['slowest_rank']}: {c['slowest_march_ms']:.3f} ms (mean "
                 f"{c['mean_march_ms']:.3f}); frame frac_needed {f['frac_needed']:.3f}, §8(d) bytes {s8:.2f}; clocks "
                 f"{c['clocks']['sm_mhz']} MHz {c['clocks']['reasons']}\n")
        L.append("| rank | march ms | needed MB | shaded M | G samples/s | frac_needed |")
        L.append("|---|---|---|---|---|---|")
        for x in c["ranks"]:
            L.append(f"| {x['rank']} | {x['kernel_ms']:.3f} | {x['needed_bytes'] / 1e6:.0f} | {x['shaded_samples'] / 1e6:.1f} | "
                     f"{x['shaded_samples'] / x['kernel_ms'] / 1e6:.0f} | {x['frac_needed']:.3f} |")
        pu = c.get("p2p_push_slowest_rank")
        if pu:
            L.append(f"Fused march + exchange (p2p_push) of rank {pu['rank']}, inboxes local: push march "
                     f"{pu['push_march_ms']:.3f} ms vs {pu['local_band_march_ms']:.3f} ms into a local band-clipped "
                     f"partial ({pu['push_over_local']:.3f}x); owner wait + blend {pu['owner_wait_and_blend_ms']:.4f} ms vs "
                     f"bare blend {pu['owner_plain_blend_ms']:.4f} ms; {pu['fragment_bytes_pushed'] / 1e6:.1f} MB pushed.")
        L.append("")
    ev = d["c3_per_rank"].get("even", {})
    if ev.get("cpu_baseline"):
        L.append(f"Config-3 CPU baseline: {ev['cpu_baseline']['value']:.4f} frames/s ({ev['cpu_baseline']['sample']}).")
    if ev.get("reference_gather"):
        L.append(f"The reference's own gather_to_root + _assemble_tiles (4K, 8 ranks, `baseline/_ref`): "
                 f"{ev['reference_gather']['ms']:.1f} ms.\n")
if "c3_family_one_rank" in d:
    o = d["c3_family_one_rank"]
    L.append(f"## config-3 family at one rank (one 1024³ brick, 3840×2160; the N > 1 lines' weak-scaling reference)\n\n"
             f"{o['value']:.0f} frames/s ({o['ms_per_step']:.4f} ms/frame, two in flight); clocks "
             f"{o['clocks']['sm_mhz']} MHz {o['clocks']['reasons']}.\n")
if "c4_orbit" in d:
    c4 = d["c4_orbit"]
    L.append(f"## config 4 (8 uneven bricks, orbit frames 0, 6, …, 30)\n\nmean slowest-rank march "
             f"{c4['mean_slowest_ms']:.3f} ms, mean imbalance {c4['mean_imbalance']:.2f}, {c4['distinct_orders']} distinct "
             "visibility orders.\n")
    L += ["| frame | order | slowest ms | mean ms |", "|---|---|---|---|"]
    L += [f"| {f['frame']} | {f['order']} | {f['max_ms']:.3f} | {f['mean_ms']:.3f} |" for f in c4["frames"]]
    L.append("")
if "c5_blend" in d:
    L.append(f"## config 5 per-rank blend ({d['c5_blend']['what']})\n")
    L += ["| frame | P | ms | GB/s | of HBM peak |", "|---|---|---|---|---|"]
    L += [f"| {x['image'][0]}x{x['image'][1]} | {x['P']} | {x['ms']:.4f} | {x['GBps']:.0f} | {x['frac_hbm']:.2f} |"
          for x in d["c5_blend"]["rows"]]
    L.append("")
if len(sys.argv) > 3:
    h = json.load(open(sys.argv[3]))
    L.append("## host work per frame (`tools/host_overhead.py`, GPU busy, no sync in the loop)\n")
    L.append(f"dprt_march_rgb8 call {h['march_rgb8_call_us']:.1f} µs, VolumeRenderer.render {h['render_call_us']:.1f} µs, "
             f"render_to_host {h['render_to_host_call_us']:.1f} µs (the GPU frame is ~210 µs).\n")
open(out, "w").write("\n".join(L) + "\n")
