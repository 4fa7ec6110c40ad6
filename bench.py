"""Frames/s of the sort-last DVR path (render + composite) on B200 -- the BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--composite MODE]

N=1 workload = BASELINE config 2: a 512^3 f32 blob field as one brick, 1920x1080, dt = 1 voxel, ERT 0.99,
the SURVEY §8(d) transfer function, auto-framing camera.  N>1 (torchrun, one process per GPU, NCCL):
weak scaling: the field grows with N (512^3 cells per rank), kd-split into N bricks balanced by non-empty
voxel count (``--decomposition mass``, the default; ``even`` gives every rank 512^3 cells), composited
at 1920x1080.  A step is
one frame: march this rank's brick -> sort-last composite -> RGB8 frame on rank 0.  The brick (512 MiB)
is larger than L2 (126 MB), so no flush is needed between steps.  At one rank, frames are marched two in
flight on lane streams (``--frames-in-flight``); the timed region ends after every frame
has completed.

``--impl reference`` times the reference-side CPU implementation of the path on the host cores: the
reference (arxiv/paper_2501_01628) has no volume renderer, so this is the C oracle port
(oracle/dvr_oracle.c, OpenMP, all host threads) on a bounded row sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "frames/sec (render+composite) at 1/2/4/8 B200; HBM and NVLink GB/s vs peak"
UNIT = "frames/s"
FIELD_EDGE = 512
W, H = 1920, 1080
DT, ERT = 1.0, 0.99
BACKGROUND = (0.05, 0.06, 0.08)
MASS_THRESHOLD = 0.1  # default_tf(): alpha is 0 below this value


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def field_dims(n_ranks: int):
    """Cells split evenly by the kd rule: 512 cells per rank along successively doubled axes."""
    cells = [FIELD_EDGE, FIELD_EDGE, FIELD_EDGE]
    r = n_ranks
    axis = 0
    while r > 1:
        cells[axis] *= 2
        r //= 2
        axis = (axis + 1) % 3
    return tuple(c + 1 for c in cells)


def workload(n_ranks: int, strategy: str = "even", device=None):
    """The field, its kd decomposition over n_ranks, camera and TF.  ``strategy`` "mass" balances the
    bricks by non-empty voxel count (voxels >= the TF's alpha threshold, counted on ``device``)."""
    from paper_2501_01628_b200.geom import auto_camera
    from paper_2501_01628_b200.volume import blob_field, decompose, default_tf

    f = blob_field(field_dims(n_ranks), seed=1, n_blobs=16)
    if strategy == "mass" and n_ranks > 1:
        from paper_2501_01628_b200 import device as dev

        dec = decompose(f, n_ranks, "mass", dev.field_mass_function(f, device, MASS_THRESHOLD))
    else:
        dec = decompose(f, n_ranks)
    cam = auto_camera(f.bounds(), W, H)
    return f, dec, cam, default_tf()


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons DURING the timed region: NVML polled every 1 ms from a
    thread (the timed region is only milliseconds long), plus the recipe's nvidia-smi -lms 200 stream."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.nvml = []          # (sm_mhz, max_mhz, reason bitmask)
        self._stop = threading.Event()
        self._poll = None
        self.error = None

    def _nvml_handle(self):
        import pynvml

        pynvml.nvmlInit()
        try:
            import torch

            bus = getattr(torch.cuda.get_device_properties(self.index), "pci_bus_id", None)
            if bus is not None:
                dom = getattr(torch.cuda.get_device_properties(self.index), "pci_domain_id", 0)
                dev = getattr(torch.cuda.get_device_properties(self.index), "pci_device_id", 0)
                return pynvml.nvmlDeviceGetHandleByPciBusId(f"{dom:08x}:{bus:02x}:{dev:02x}.0")
        except Exception:  # noqa: BLE001 - fall back to the index
            pass
        return pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _sample(self):
        import pynvml

        self.nvml.append((pynvml.nvmlDeviceGetClockInfo(self._h, pynvml.NVML_CLOCK_SM), self._mx,
                          pynvml.nvmlDeviceGetCurrentClocksEventReasons(self._h)))

    def _poll_nvml(self):
        try:
            while not self._stop.is_set():
                self._sample()
                time.sleep(0.001)
        except Exception as exc:  # noqa: BLE001 - NVML unavailable: the nvidia-smi stream remains
            self.error = f"{type(exc).__name__}: {exc}"

    def __enter__(self):
        try:  # NVML set up synchronously, so polling covers the whole timed region
            import pynvml

            self._h = self._nvml_handle()
            self._mx = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self._poll = threading.Thread(target=self._poll_nvml, daemon=True)
            self._poll.start()
        except Exception as exc:  # noqa: BLE001
            self.error = f"{type(exc).__name__}: {exc}"
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self._stop.set()
        if self._poll is not None:
            self._poll.join(1)
            try:
                self._sample()  # the clock right at the end of the timed region
            except Exception:  # noqa: BLE001
                pass
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}
        if self.nvml:
            for _, _, r in self.nvml:
                reasons.update(n for n, b in bits.items() if r & b)
            return {"sm_mhz": statistics.median(c for c, _, _ in self.nvml), "sm_max_mhz": float(self.nvml[0][1]),
                    "reasons": sorted(reasons), "samples": len(self.nvml), "source": "nvml 1 ms poll + nvidia-smi",
                    "smi_samples": len(sm)}
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvidia-smi", "nvml_error": self.error}


def cpu_baseline(vox: np.ndarray, dec, cam, tf, target_s: float = 12.0):
    """The oracle (C, OpenMP, all host threads) on a row sample of the same frame; frames/s extrapolated
    from the sampled fraction of rows."""
    import oracle

    oracle.build_oracle()
    threads = oracle.max_threads()
    ca = oracle.camera_array(cam.position, cam.view_dir, cam.up, cam.fov_y, cam.aspect)
    lo, hi = dec.boxes[0]
    f = dec.field
    ob = oracle.OracleBrick(f.dims, lo, hi, 1, f.origin, f.spacing)
    tfa = tf.as_f32()
    # calibrate on a sparse sample, then size the stride for ~target_s of CPU work
    stride = 64
    t0 = time.perf_counter()
    oracle.render_brick(vox, ob, ca, tfa, tf.vmin, tf.vmax, DT, ERT, W, H, rows=(0, H, stride), nthreads=threads)
    t_cal = time.perf_counter() - t0
    rows_cal = len(range(0, H, stride))
    per_row = t_cal / rows_cal
    nrows = int(max(rows_cal, min(H, target_s / max(per_row, 1e-9))))
    stride = max(1, H // nrows)
    t0 = time.perf_counter()
    oracle.render_brick(vox, ob, ca, tfa, tf.vmin, tf.vmax, DT, ERT, W, H, rows=(0, H, stride), nthreads=threads)
    dt = time.perf_counter() - t0
    rows = len(range(0, H, stride))
    fps = (rows / H) / dt
    return {"value": fps, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"every {stride}th row ({rows}/{H} rows of the 1920x1080 frame, {dt:.1f} s), frames/s "
                      f"extrapolated by the row fraction; oracle/dvr_oracle.c f64, OpenMP {threads} threads"}


def run_reference(args):
    """--impl reference: the CPU port of the path, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    f, dec, cam, tf = workload(1)
    log(f"[reference] generating {f.dims} field on the host")
    oracle.build_oracle()
    vox = oracle.generate_field(f.dims, f.blobs, nthreads=oracle.max_threads())
    threads = oracle.max_threads()
    ca = oracle.camera_array(cam.position, cam.view_dir, cam.up, cam.fov_y, cam.aspect)
    lo, hi = dec.boxes[0]
    ob = oracle.OracleBrick(f.dims, lo, hi, 1, f.origin, f.spacing)
    # whole frames per step (~0.5 s on 16 threads) unless K + W is large: then every stride-th row, so the
    # arm stays around a minute; thin samples would under-state the CPU (few rows per OpenMP thread)
    stride = max(1, -(-(args.warmup + args.steps) // 120))
    rows = len(range(0, H, stride))
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.render_brick(vox, ob, ca, tf.as_f32(), tf.vmin, tf.vmax, DT, ERT, W, H, rows=(i % stride, H, stride),
                            nthreads=threads)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    frame_s = sum(times) / len(times) * H / rows
    fps = 1.0 / frame_s
    sample = (f"each step renders every {stride}th row ({rows}/{H} rows, offset by step) of the c2 frame; "
              f"frames/s = row fraction / step time; oracle/dvr_oracle.c, OpenMP {threads} threads")
    line = {"impl": "reference", "metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": frame_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c2: 512^3 f32 blob field, 1 brick, 1920x1080, dt=1 voxel, ERT 0.99",
                       "image": [W, H], "field": list(f.dims)},
            "cpu_baseline": {"value": fps, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2501_01628_b200 import device as dev
    from paper_2501_01628_b200.engine import RenderOptions, VolumeRenderer
    from paper_2501_01628_b200.transport import SoloEndpoint, init_dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        backend = os.environ.get("DPRT_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            ep = init_dist("nccl")
            device = ep.device
        else:
            # functional test hook only (tests/test_gpu_multiprocess.py): gloo control plane, ranks
            # possibly sharing a GPU -- never a measurement
            from paper_2501_01628_b200.transport import DistEndpoint

            device = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
            torch.cuda.set_device(device)
            dist.init_process_group(backend)
            ep = DistEndpoint(device=device)
    else:
        device = torch.device("cuda", 0)
        torch.cuda.set_device(device)
        ep = SoloEndpoint(device)
    rank, R = ep.rank, ep.R
    f, dec, cam, tf = workload(R, args.decomposition, device)
    desc = dec.brick(rank)
    brick = dev.DeviceBrick(desc, device).generate(f)
    renderer = VolumeRenderer(ep, brick, dec, tf, BACKGROUND)
    skip = not args.no_skip
    # one rank: frames in flight on lane streams (frame k+1's beams start on the SMs frame k's last beams
    # leave idle); every frame is still complete and checked byte-identical in tests
    fif = args.frames_in_flight if R == 1 else 1
    opts = RenderOptions(dt=DT, ert=ERT, composite=args.composite, skip_empty=skip, fragment_dtype=args.fragments,
                         frames_in_flight=fif)
    stream = torch.cuda.current_stream(device)
    torch.cuda.synchronize(device)

    def barrier():
        if R > 1:
            dist.barrier()
        torch.cuda.synchronize(device)

    def step():
        renderer.render(cam, W, H, opts, verify=False)

    # ---- device-resident throughput (value)
    for _ in range(args.warmup):
        step()
    renderer.join(stream)
    barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device.index) as clocks:
        barrier()
        start.record(stream)
        for _ in range(args.steps):
            step()
        renderer.join(stream)  # every frame in flight is complete before the end event
        end.record(stream)
        barrier()
    ms = start.elapsed_time(end)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=device)
    if R > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_step = float(ms_t.item()) / args.steps
    fps = 1000.0 / ms_step

    # ---- compositing exchange alone (N > 1): fragments over NVLink + blend + gather, max over ranks
    nvlink = None
    if R > 1:
        order = renderer.decomposition.visibility_order(cam.position)
        comp = renderer.compositor
        # the step's exchange: footprint-row bands when the mode clips them (RenderOptions.clip_exchange)
        bands = renderer._bands(cam, W, H) if comp.clips_bands() else None
        cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier()
        for a_, b_ in cev:
            a_.record(stream)
            comp.composite(renderer.partial, order, BACKGROUND, bands=bands)
            b_.record(stream)
        barrier()
        cms = torch.tensor([sum(a_.elapsed_time(b_) for a_, b_ in cev) / len(cev)], dtype=torch.float64,
                           device=device)
        dist.all_reduce(cms, op=dist.ReduceOp.MAX)
        comp_ms = float(cms.item())
        # fragment bytes this rank moved (sent, or read from peers in p2p mode) + its RGB8 tile; max over ranks
        moved = torch.tensor([float(comp.last_bytes)], dtype=torch.float64, device=device)
        dist.all_reduce(moved, op=dist.ReduceOp.MAX)
        frag_bytes = int(moved.item())
        full_bytes = int((1 - 1 / R) * W * H * (8 if args.fragments == "f16" else 16))  # unclipped fragments/rank
        gather_bytes = int((R - 1) / R * W * H * 3)          # RGB8 tiles into rank 0
        achieved_nv = frag_bytes / (comp_ms * 1e-3) / 1e9
        nvlink = {"bound": "nvlink", "achieved": achieved_nv, "peak": 770.0, "unit": "GB/s",
                  "frac": achieved_nv / 770.0, "peak_kind": "measured peer copy per direction (B200_PROFILING.md)",
                  "composite_ms": comp_ms, "fragment_bytes_per_rank": frag_bytes,
                  "unclipped_fragment_bytes_per_rank": full_bytes, "rgb8_into_root": gather_bytes,
                  "mode": comp.mode, "clipped_to_footprint_rows": bands is not None}

    # ---- marcher alone, CUDA events on its launch stream (roofline): K back-to-back launches of the same
    # call the step makes (the fused RGB8 march at one rank; the band-cleared RGBA-partial march otherwise)
    # between one event pair, so the average is the kernel's launch duration without per-event gaps
    partial = renderer.partial
    frame8 = torch.empty(W * H * 3, dtype=torch.uint8, device=device)
    clip = R > 1 and renderer.compositor.clips_bands()
    m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    m0.record(stream)
    for _ in range(args.steps):
        if R == 1:
            dev.march_rgb8(brick, cam, renderer.dtf, DT, ERT, BACKGROUND, frame8, W, H, skip=skip)
        else:
            dev.march(brick, cam, renderer.dtf, DT, ERT, partial, W, H, skip=skip, band_clear=clip)
    m1.record(stream)
    barrier()
    march_ms = m0.elapsed_time(m1) / args.steps
    rect = brick.footprint(cam, W, H)
    fp_px = max(0, rect[2] - rect[0]) * max(0, rect[3] - rect[1])
    alg_bytes = desc.stored_bytes + 16 * fp_px + 16 * tf.n
    peak, peak_kind = load_peaks()
    achieved = alg_bytes / (march_ms * 1e-3) / 1e9
    traffic = None
    tr = ROOT / "profiles" / "march_traffic.json"
    if tr.exists():
        t = json.loads(tr.read_text())
        if t.get("workload") == "c2" and R == 1:
            traffic = t.get("dram_bytes_per_launch")

    # ---- end to end through the public API with host buffers
    pinned_tf = torch.from_numpy(tf.as_f32().reshape(-1)).pin_memory()
    host_frame = torch.empty((H, W, 3), dtype=torch.uint8).pin_memory()
    from paper_2501_01628_b200.device import camera_struct
    import ctypes

    h2d = pinned_tf.numel() * 4 + ctypes.sizeof(camera_struct(cam))
    d2h = W * H * 3 if rank == 0 else 0

    depth = 2  # frames in flight: the host waits for frame k-2's bytes while k-1 and k are queued
    host_frames = [host_frame] + [torch.empty((H, W, 3), dtype=torch.uint8).pin_memory() for _ in range(depth)]
    inflight = []

    def e2e_step(k):
        # per step: TF H2D from pinned memory, collective render (digest verified), RGB8 frame D2H into
        # pinned memory on a side stream; the host waits for frame k-depth's bytes while later frames render
        renderer.dtf.update(tf, staging=pinned_tf)
        hf = renderer.render_to_host(cam, W, H, host_frames[k % (depth + 1)] if rank == 0 else None, opts, verify=True)
        inflight.append(hf)
        if len(inflight) > depth:
            inflight.pop(0).wait()

    def drain():
        while inflight:
            inflight.pop(0).wait()

    for k in range(args.warmup):
        e2e_step(k)
    drain()
    barrier()
    t0 = time.perf_counter()
    for k in range(args.steps):
        e2e_step(k)
    drain()
    barrier()
    e2e_s = time.perf_counter() - t0
    e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device=device)
    if R > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_fps = args.steps / float(e2e_t.item())

    cpu = None
    if rank == 0 and R == 1 and not args.no_cpu_baseline:
        log("[bench] timing the CPU oracle on a row sample")
        vox = brick.download()
        cpu = cpu_baseline(vox, dec, cam, tf)

    if rank == 0:
        # per frame: R == 1 -> march_beam alone (background fill and tone map fused into it); R > 1 ->
        # march_beam + composite (plus the 8-byte tile-counter memset and, at R > 1, the partial band memset
        # and NCCL's own kernels)
        launches = args.steps * (1 if R == 1 else 2)
        line = {
            "metric": METRIC, "value": fps * 1.0, "unit": UNIT, "n_gpus": R, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": ("c2: 512^3 f32 blob field (seed 1, 16 blobs), 1 brick per GPU, 1920x1080, "
                                    "dt=1 voxel, ERT 0.99, SURVEY 8(d) TF, auto camera") if R == 1 else
                                   (f"weak scaling of c2: {'x'.join(str(c - 1) for c in f.dims)}-cell f32 blob field "
                                    f"(seed 1, 16 blobs), {R} kd bricks ({args.decomposition}), 1920x1080, dt=1 voxel, "
                                    "ERT 0.99, SURVEY 8(d) TF, auto camera"),
                       "field": list(f.dims), "bricks": R, "decomposition": args.decomposition if R > 1 else "whole",
                       "image": [W, H], "composite": renderer.compositor.mode,
                       "fragments": args.fragments, "frames_in_flight": fif,
                       "empty_space_skipping": skip, "l2": "inputs larger than L2 (brick 512 MiB/GPU), no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": "march_beam_kernel", "kernel_ms": march_ms, "algorithmic_bytes": alg_bytes,
                         "footprint_px": fp_px},
            "e2e": {"value": e2e_fps, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "compositor_roofline": nvlink,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    brick.close()
    if R > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--composite", default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-skip", action="store_true", help="disable exact empty-space skipping")
    ap.add_argument("--decomposition", default="mass", choices=["even", "mass"],
                    help="N > 1: kd split of the field, even cells or balanced by non-empty voxel count")
    ap.add_argument("--frames-in-flight", type=int, default=2,
                    help="single rank: frames marched concurrently on lane streams (1 = stream-ordered)")
    ap.add_argument("--fragments", default="f32", choices=["f32", "f16"],
                    help="exchanged RGBA fragment format at N > 1 (f16: half the bytes, fp16 tolerance)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
