"""Frames/s of the sort-last DVR path (render + composite) on B200 -- the BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config auto|c1..c5]
                    [--per-rank] [--composite MODE] [--decomposition even|mass]

Workloads (BASELINE.json ``configs``):
  c1  64^3 blob field split into N bricks (2 at N = 2), 256x256 (the reference's CPU-runnable case)
  c2  512^3 cells per rank (weak scaling), 1920x1080 -- the N = 1 default: BASELINE configs[1]
  c3  1024^3 cells per rank, kd-doubled along x, y, z (N = 8: the 2048^3 field of configs[2]),
      3840x2160 -- the N > 1 default
  c4  lander-like anisotropic 1536x768x384 field (spacing 1,1,2), N uneven mass-balanced bricks, an
      orbiting camera (step k = orbit frame k mod 36)
  c5  compositing only: random premultiplied RGBA partials (alpha <= 0.5) of a 3840x2160 frame
``--per-rank`` (N = 1, c3 / c4): every rank's brick of the N = 8 decomposition marched alone on this GPU,
one after another; ``value`` is then 1000 / (slowest rank's march ms) -- the march critical path of the
8-GPU frame, not a whole frame.

A step is one frame: march this rank's brick -> sort-last composite -> RGB8 frame on rank 0.  Every brick
is larger than L2 (126 MB), so no flush is needed between steps.  At one rank frames are marched two in
flight on lane streams; the timed region ends after every frame has completed.

N > 1: launched by the driver as ``torchrun --nproc-per-node N bench.py --gpus N`` (one process per GPU,
NCCL).  ``python bench.py --gpus N`` without torchrun launches those N ranks itself (torch.distributed.run
on 127.0.0.1); with fewer visible GPUs than N the ranks share GPUs over a gloo control plane and the line
says ``"measurement": false`` (a functional run, never a number).

``--impl reference`` times the reference-side CPU implementation of the path on the host cores: the
reference (arxiv/paper_2501_01628) has no volume renderer, so this is the C oracle port
(oracle/dvr_oracle.c, OpenMP, all host threads) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "frames/sec (render+composite) at 1/2/4/8 B200; HBM and NVLink GB/s vs peak"
UNIT = "frames/s"
DT, ERT = 1.0, 0.99
BACKGROUND = (0.05, 0.06, 0.08)
MASS_THRESHOLD = 0.1  # default_tf(): alpha is 0 below this value
CONFIGS = ("c1", "c2", "c3", "c4", "c5")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# --------------------------------------------------------------------------------------------------
# workloads


def field_dims(edge: int, n_ranks: int):
    """``edge`` cells per axis per rank, doubled along x, y, z in turn (the kd split's order): N = 8 at
    edge 1024 is the 2048^3 field of config 3."""
    cells = [edge, edge, edge]
    r, axis = n_ranks, 0
    while r > 1:
        cells[axis] *= 2
        r //= 2
        axis = (axis + 1) % 3
    return tuple(c + 1 for c in cells)


@dataclass
class Workload:
    cfg: str
    field: object
    dec: object
    cams: list
    tf: object
    W: int
    H: int
    strategy: str
    text: str
    scaling: str
    gen: dict = field(default_factory=dict)  # the spatialField generator parameters (api_e2e)
    extra: dict = field(default_factory=dict)

    def config(self, R: int, **more) -> dict:
        """The ``config`` object of the JSON line -- identical in both arms for the same arguments."""
        f = self.field
        d = {"workload": self.text, "field": list(f.dims), "spacing": list(f.spacing), "bricks": R,
             "decomposition": self.strategy if R > 1 else "whole", "image": [self.W, self.H],
             "dt_voxels": DT, "ert": ERT, "cameras": len(self.cams),
             "l2": ("inputs larger than L2 (every brick > 126 MB), no flush"
                    if min(self.dec.brick(r).stored_bytes for r in range(self.dec.P)) > 126e6 else
                    "bricks fit in L2 (no flush): a parity-size config, not a headline number")}
        d.update(self.extra)
        d.update(more)
        return d


def build_workload(cfg: str, R: int, strategy: str, device=None, mass_device=None) -> Workload:
    """The field, its kd decomposition over R bricks, camera(s), TF and frame size of a BASELINE config.
    ``strategy`` "mass" balances the bricks by non-empty voxel count (voxels >= the TF's alpha threshold,
    counted on ``mass_device`` -- the GPU -- or on the host through the oracle when it is None)."""
    from paper_2501_01628_b200.geom import auto_camera, orbit_camera
    from paper_2501_01628_b200.volume import blob_field, decompose, default_tf

    tf = default_tf()
    if cfg == "c1":
        f, W, H = blob_field((65, 65, 65), seed=1, n_blobs=16), 256, 256
        text = "c1: 64^3 f32 blob field (seed 1, 16 blobs), kd bricks, 256x256"
        scaling = "strong"
    elif cfg in ("c2", "c3"):
        edge, (W, H) = (512, (1920, 1080)) if cfg == "c2" else (1024, (3840, 2160))
        f = blob_field(field_dims(edge, R), seed=1, n_blobs=16)
        cells = "x".join(str(c - 1) for c in f.dims)
        text = (f"{cfg}: {cells}-cell f32 blob field (seed 1, 16 blobs) = {edge}^3 cells per GPU, {R} kd brick"
                f"{'s' if R > 1 else ''}, {W}x{H}")
        if cfg == "c3" and R == 8:
            text += " (BASELINE config 3: 2048^3 / 8 x B200 / 4K)"
        scaling = "weak"
    elif cfg == "c4":
        f, W, H = blob_field((1536, 768, 384), seed=7, spacing=(1.0, 1.0, 2.0), lopsided=True), 1920, 1080
        text = "c4: lander-like 1536x768x384 field, spacing (1,1,2), lopsided 16-blob mixture, orbit camera, 1920x1080"
        scaling = "strong"
    else:
        raise ValueError(cfg)
    text += f", dt=1 voxel, ERT 0.99, SURVEY 8(d) TF"
    mass = None
    if strategy == "mass" and R > 1:
        if mass_device is not None:
            from paper_2501_01628_b200 import device as dev

            mass = dev.field_mass_function(f, mass_device, MASS_THRESHOLD)
        else:
            mass = host_mass_function(f, MASS_THRESHOLD)
    dec = decompose(f, R, strategy if R > 1 else "even", mass)
    if cfg == "c4":
        bb = f.bounds()
        cams = [orbit_camera(bb.center(), 1.2 * bb.diagonal(), math.radians(10.0 * i), math.radians(20.0), 45.0,
                             W / H) for i in range(36)]
    else:
        cams = [auto_camera(f.bounds(), W, H)]
    gen = {"seed": 7, "lopsided": True} if cfg == "c4" else {"seed": 1, "lopsided": False}
    return Workload(cfg, f, dec, cams, tf, W, H, strategy if R > 1 else "whole", text, scaling, gen)


def host_mass_function(f, tau: float, chunk: int = 64):
    """Mass function of the mass-weighted kd split on the host (CPU arm only): the oracle generates the
    field in z-chunks of voxel planes and only the 1-byte mask is kept (config 3: 8.6 GB, not 34 GB)."""
    import oracle

    nx, ny, nz = f.dims
    mask = np.empty((nz, ny, nx), np.bool_)
    for z0 in range(0, nz, chunk):
        z1 = min(nz, z0 + chunk)
        vox = oracle.generate_field(f.dims, f.blobs, (0, 0, z0), (nx, ny, z1 - z0), nthreads=oracle.max_threads(),
                                    fast=True)
        mask[z0:z1] = vox >= np.float32(tau)
        del vox

    def mass(axis, lo, hi):
        sub = mask[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        return sub.sum(axis=tuple(a for a in range(3) if a != 2 - axis), dtype=np.int64)

    return mass


# --------------------------------------------------------------------------------------------------
# clocks


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
        self._mark = 0

    def _nvml_handle(self):
        import pynvml

        pynvml.nvmlInit()
        try:
            import torch

            props = torch.cuda.get_device_properties(self.index)
            bus = getattr(props, "pci_bus_id", None)
            if bus is not None:
                dom = getattr(props, "pci_domain_id", 0)
                dev = getattr(props, "pci_device_id", 0)
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

    def mark(self) -> None:
        """The timed region starts now: the NVML summary covers only the samples from here on."""
        self._mark = len(self.nvml)

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
        nv = self.nvml[self._mark:] or self.nvml[-1:]
        if nv:
            for _, _, r in nv:
                reasons.update(n for n, b in bits.items() if r & b)
            return {"sm_mhz": statistics.median(c for c, _, _ in nv), "sm_max_mhz": float(nv[0][1]),
                    "reasons": sorted(reasons), "samples": len(nv), "source": "nvml 1 ms poll + nvidia-smi",
                    "smi_samples": len(sm)}
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvidia-smi", "nvml_error": self.error}


def host_info() -> dict:
    cpu = "unknown"
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                cpu = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_count": os.cpu_count(), "cpu_model": cpu}


# --------------------------------------------------------------------------------------------------
# CPU baselines (oracle = the reference-side CPU implementation of the path; test infrastructure)


def cpu_baseline_rows(vox: np.ndarray, wl: Workload, target_s: float = 12.0):
    """Single-brick workload: the oracle (C, OpenMP, all host threads) on a row sample of the frame;
    frames/s extrapolated from the sampled fraction of rows."""
    import oracle

    oracle.build_oracle()
    threads = oracle.max_threads()
    cam = wl.cams[0]
    ca = oracle.camera_array(cam.position, cam.view_dir, cam.up, cam.fov_y, cam.aspect)
    lo, hi = wl.dec.boxes[0]
    f = wl.field
    ob = oracle.OracleBrick(f.dims, lo, hi, 1, f.origin, f.spacing)
    tfa = wl.tf.as_f32()
    W, H = wl.W, wl.H
    stride = 64
    t0 = time.perf_counter()
    oracle.render_brick(vox, ob, ca, tfa, wl.tf.vmin, wl.tf.vmax, DT, ERT, W, H, rows=(0, H, stride), nthreads=threads)
    per_row = (time.perf_counter() - t0) / len(range(0, H, stride))
    nrows = int(max(len(range(0, H, stride)), min(H, target_s / max(per_row, 1e-9))))
    stride = max(1, H // nrows)
    t0 = time.perf_counter()
    oracle.render_brick(vox, ob, ca, tfa, wl.tf.vmin, wl.tf.vmax, DT, ERT, W, H, rows=(0, H, stride), nthreads=threads)
    dt = time.perf_counter() - t0
    rows = len(range(0, H, stride))
    return {"value": (rows / H) / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"every {stride}th row ({rows}/{H} rows of the {W}x{H} frame, {dt:.1f} s), frames/s "
                      f"extrapolated by the row fraction; oracle/dvr_oracle.c f64, OpenMP {threads} threads",
            "host": host_info()}


def cpu_baseline_lattice(wl: Workload, cam, stride: int = 8, keep: bool = False, bricks=None):
    """Multi-brick workload (config 3 / 4): the oracle renders every brick's partial on the strided pixel
    lattice (every ``stride``-th pixel in x and y: 1/stride^2 of the frame), composites them in visibility
    order and tone maps.  Bricks are generated on the host one at a time (oracle fast generator,
    bit-identical to the scalar one); only the rendering + compositing is timed.  ``keep`` returns the
    host bricks for repeated steps (config 3 holds 8 x 4.3 GB)."""
    import oracle

    oracle.build_oracle()
    threads = oracle.max_threads()
    f, dec, tf = wl.field, wl.dec, wl.tf
    ca = oracle.camera_array(cam.position, cam.view_dir, cam.up, cam.fov_y, cam.aspect)
    parts, gen_s, render_s = {}, 0.0, 0.0
    held = bricks if bricks is not None else {}
    for r in range(dec.P):
        lo, hi = dec.boxes[r]
        ob = oracle.OracleBrick(f.dims, lo, hi, 1, f.origin, f.spacing)
        vox = held.get(r)
        if vox is None:
            t0 = time.perf_counter()
            vox = oracle.generate_field(f.dims, f.blobs, ob.stored_lo, ob.stored_dims, nthreads=threads, fast=True)
            gen_s += time.perf_counter() - t0
        t0 = time.perf_counter()
        parts[r] = oracle.render_lattice(vox, ob, ca, tf.as_f32(), tf.vmin, tf.vmax, DT, ERT, wl.W, wl.H,
                                         stride, stride, nthreads=threads)
        render_s += time.perf_counter() - t0
        if keep:
            held[r] = vox
        del vox
    t0 = time.perf_counter()
    order = dec.visibility_order(cam.position)
    rgb8 = oracle.tone_map_rgb8(oracle.composite([parts[r] for r in range(dec.P)], order, BACKGROUND))
    step_s = render_s + time.perf_counter() - t0
    frac = 1.0 / (stride * stride)
    res = {"value": frac / step_s, "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"every {stride}th pixel in x and y (1/{stride * stride} of the {wl.W}x{wl.H} frame), all "
                     f"{dec.P} bricks rendered + over-composited + tone mapped: {step_s:.2f} s, frames/s "
                     f"extrapolated by the pixel fraction; host brick generation ({gen_s:.1f} s) untimed; "
                     f"oracle/dvr_oracle.c f64, OpenMP {threads} threads",
           "host": host_info(), "step_s": step_s}
    return res, rgb8, held


def ref_gather_baseline(W: int, H: int, R: int) -> Optional[dict]:
    """The REFERENCE's own image-assembly step: every rank's f64 RGB row tile through
    `gather_to_root` + `_assemble_tiles` (pkg/src/dprt/engine.py:443-456,485, transport.py:465-475) on
    its in-process transport (`run_collective` threads), from the unmodified install in baseline/_ref;
    rank 0's time, best of 3.  None when the install is absent."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "dprt").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/dprt_numba_cache")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        from dprt import engine as ref_engine, transport as ref_transport
    except Exception as exc:  # noqa: BLE001
        return {"unavailable": f"{type(exc).__name__}: {exc}"}

    def body(ep):
        row0, row1 = ref_engine.assign_pixels(W, H, ep.R)[ep.rank]
        fb = np.full((row1 - row0, W, 3), 0.5)
        times = []
        for _ in range(3):
            ref_transport.barrier(ep)
            t0 = time.perf_counter()
            tiles = ref_transport.gather_to_root(ep, ref_engine._tile_bytes(row0, row1, fb))
            if ep.rank == 0:
                ref_engine._assemble_tiles(tiles, W, H)
            times.append(time.perf_counter() - t0)
        return min(times)

    res = ref_transport.run_collective(R, body)
    return {"ms": res[0] * 1e3, "frame": [W, H], "ranks": R,
            "what": "reference gather_to_root + _assemble_tiles of f64 RGB row tiles, inproc threads, rank 0, best of 3"}


# --------------------------------------------------------------------------------------------------
# reference arm


def run_reference(args):
    """--impl reference: the CPU port of the path, rank 0 only (other ranks exit without work)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    R = args.gpus
    cfg = resolve_config(args.config, R)
    if cfg == "c5":
        line = {"impl": "reference", "unavailable": "config c5 is compositing-only; the reference has no compositor"}
        print(json.dumps(line), flush=True)
        return
    wl = build_workload(cfg, R, args.decomposition)
    threads = oracle.max_threads()
    times = []
    if R == 1 and cfg != "c4":
        log(f"[reference] generating the {wl.field.dims} field on the host")
        f = wl.field
        vox = oracle.generate_field(f.dims, f.blobs, nthreads=threads, fast=True)
        lo, hi = wl.dec.boxes[0]
        ob = oracle.OracleBrick(f.dims, lo, hi, 1, f.origin, f.spacing)
        cam = wl.cams[0]
        ca = oracle.camera_array(cam.position, cam.view_dir, cam.up, cam.fov_y, cam.aspect)
        # whole frames per step (~0.5 s at c2 on 16 threads) unless K + W is large: then every stride-th row,
        # so the arm stays around a minute; thin samples would under-state the CPU (few rows per thread)
        stride = max(1, -(-(args.warmup + args.steps) // 120)) if cfg == "c2" else max(1, wl.H // 135)
        rows = len(range(0, wl.H, stride))
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            oracle.render_brick(vox, ob, ca, wl.tf.as_f32(), wl.tf.vmin, wl.tf.vmax, DT, ERT, wl.W, wl.H,
                                rows=(i % stride, wl.H, stride), nthreads=threads)
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
        frame_s = sum(times) / len(times) * wl.H / rows
        sample = (f"each step renders every {stride}th row ({rows}/{wl.H} rows, offset by step) of the frame; "
                  f"frames/s = row fraction / step time; oracle/dvr_oracle.c f64, OpenMP {threads} threads")
    else:
        # multi-brick: the strided 1/64 pixel lattice of the composited frame, all bricks per step; the host
        # bricks are generated once (untimed) and kept
        held = {}
        for i in range(args.warmup + args.steps):
            cam = wl.cams[i % len(wl.cams)]
            res, _, held = cpu_baseline_lattice(wl, cam, 8, keep=True, bricks=held)
            if i >= args.warmup:
                times.append(res["step_s"])
        frame_s = sum(times) / len(times) * 64
        sample = res["sample"]
    fps = 1.0 / frame_s
    line = {"impl": "reference", "metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": R,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": frame_s * 1e3, "higher_is_better": True,
            "scaling": wl.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": wl.config(R),
            "cpu_baseline": {"value": fps, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                             "host": host_info()},
            "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------------------
# our arm: measurement legs


def resolve_config(cfg: str, R: int) -> str:
    if cfg == "auto":
        return "c2" if R == 1 else "c3"
    return cfg


def spin_up(step, n: int, device, R: int = 1, min_s: float = 0.2) -> int:
    """The W warm-up steps, then more until the GPU has been busy for ``min_s``: an idle GPU lowers its SM
    clock and the first milliseconds after idle run slower (measured on c2: the first 20-frame region after
    0.5 s idle +6 %, later regions not), so a timed region that follows set-up or another leg's host work
    would otherwise start below the clock a sustained run holds.  The extra count is derived from the
    slowest rank's W-step time, so every rank runs the same number of (collective) steps.  ``step(k)``."""
    import torch
    import torch.distributed as dist

    for k in range(n):  # W steps (first-frame set-up included)
        step(k)
    torch.cuda.synchronize(device)
    m = max(n, 4)  # steady-state step time
    t0 = time.perf_counter()
    for k in range(n, n + m):
        step(k)
    torch.cuda.synchronize(device)
    per = (time.perf_counter() - t0) / m
    if R > 1:
        t = torch.tensor([per], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        per = float(t.item())
    extra = min(int(math.ceil(min_s / max(per, 1e-5))), 20000)
    for k in range(n + m, n + m + extra):
        step(k)
    return n + m + extra


def events_ms(fn, steps: int, stream) -> float:
    import torch

    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b) / steps


def graph_ms(fn, steps: int, device) -> float:
    """Per-launch device ms of ``fn`` captured ``steps`` times into one CUDA graph (replay timed by events):
    kernels of a few microseconds are otherwise separated by host launch gaps."""
    import torch

    side = torch.cuda.Stream(device)
    side.wait_stream(torch.cuda.current_stream(device))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for _ in range(steps):
            fn()
    g.replay()
    torch.cuda.synchronize(device)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.current_stream(device)
    a.record(st)
    g.replay()
    b.record(st)
    b.synchronize()
    return a.elapsed_time(b) / steps


def march_leg(dev, brick, desc, cam, dtf, tf, W, H, steps, fused: bool, partial=None, band_clear=False) -> dict:
    """The march kernel alone (CUDA events on its launch stream, K back-to-back launches of the call the
    step makes) + the instrumented march (needed bytes, shaded samples).  SURVEY §8(d) roofline."""
    import torch

    device = brick.device
    stream = torch.cuda.current_stream(device)
    frame8 = torch.empty(W * H * 3, dtype=torch.uint8, device=device) if fused else None

    def once():
        if fused:
            dev.march_rgb8(brick, cam, dtf, DT, ERT, BACKGROUND, frame8, W, H)
        else:
            dev.march(brick, cam, dtf, DT, ERT, partial, W, H, band_clear=band_clear)

    for _ in range(3):
        once()
    torch.cuda.synchronize(device)
    ms = events_ms(once, steps, stream)
    st = dev.march_stats(brick, cam, dtf, DT, ERT, W, H)
    rect = brick.footprint(cam, W, H)
    fp_px = max(0, rect[2] - rect[0]) * max(0, rect[3] - rect[1])
    alg = desc.stored_bytes + 16 * fp_px + 16 * tf.n
    out_bytes = 3 * W * H if fused else 16 * fp_px
    needed = st["needed_bytes"] + out_bytes + 16 * tf.n
    peak, kind = load_peaks()
    achieved = alg / (ms * 1e-3) / 1e9
    ach_needed = needed / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": None, "peak_kind": peak_kind_text(kind), "kernel": "march_beam_kernel", "kernel_ms": ms,
            "algorithmic_bytes": alg, "footprint_px": fp_px,
            "needed_bytes": needed, "achieved_needed": ach_needed, "frac_needed": ach_needed / peak,
            "needed_macrocells": st["macrocells"], "shaded_samples": st["shaded_samples"],
            "contributing_samples": st["contributing_samples"],
            "shaded_samples_per_s": st["shaded_samples"] / (ms * 1e-3)}


def peak_kind_text(kind: str) -> str:
    return "measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs)" if kind == "measured" else \
        "fallback 6.65 TB/s (B200_PROFILING.md)"


def measure_traffic(cfg: str, timeout: int = 240) -> dict:
    """DRAM bytes + warp instructions of ONE march launch of this workload, from an ncu child process
    (``--metrics`` pass on a separate single-GPU run of ``bench.py --traffic-probe``; the bench's own
    timings are never taken under the profiler)."""
    ncu = os.environ.get("NCU") or "/usr/local/cuda/bin/ncu"
    if not Path(ncu).exists():
        return {"error": "ncu not found"}
    metrics = ("dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,"
               "smsp__thread_inst_executed.sum")
    log_file = Path(os.environ.get("TMPDIR", "/tmp")) / f"dprt_traffic_{os.getpid()}.csv"
    cmd = [ncu, "--metrics", metrics, "--clock-control", "none", "-k", "regex:march_beam_kernel", "-s", "3",
           "-c", "1", "--csv", "--log-file", str(log_file), sys.executable, str(Path(__file__).resolve()),
           "--traffic-probe", "--config", cfg]
    try:
        p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    except subprocess.TimeoutExpired:
        return {"error": f"ncu child timed out after {timeout} s"}
    if p.returncode != 0 or not log_file.exists():
        return {"error": f"ncu child rc={p.returncode}: {(p.stderr or p.stdout)[-300:]}"}
    import csv

    vals = {}
    with open(log_file) as fh:
        rows = [r for r in csv.reader(ln for ln in fh if not ln.startswith("=="))]
    hdr = rows[0]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        name, unit, v = d.get("Metric Name"), d.get("Metric Unit"), d.get("Metric Value", "").replace(",", "")
        try:
            x = float(v)
        except ValueError:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
                 "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0}.get(unit, 1.0)
        vals[name] = x * scale
    log_file.unlink(missing_ok=True)
    if "dram__bytes_read.sum" not in vals:
        return {"error": "ncu produced no dram metrics"}
    return {"dram_bytes": vals["dram__bytes_read.sum"] + vals.get("dram__bytes_write.sum", 0.0),
            "dram_read_bytes": vals["dram__bytes_read.sum"], "warp_instructions": vals.get("smsp__inst_executed.sum"),
            "thread_instructions": vals.get("smsp__thread_inst_executed.sum"),
            "ncu_kernel_s": vals.get("gpu__time_duration.sum"),
            "source": "ncu --metrics child run of bench.py --traffic-probe (1 launch after 3, cold cache, serialised)"}


def traffic_probe(args):
    """Hidden mode for measure_traffic: the workload's brick and a few march launches, nothing else."""
    import torch

    from paper_2501_01628_b200 import device as dev

    d = torch.device("cuda", 0)
    torch.cuda.set_device(d)
    wl = build_workload(args.config, 1, "even")
    desc = wl.dec.brick(0)
    brick = dev.DeviceBrick(desc, d).generate(wl.field)
    dtf = dev.DeviceTF(wl.tf, d)
    frame8 = torch.empty(wl.W * wl.H * 3, dtype=torch.uint8, device=d)
    for _ in range(5):
        dev.march_rgb8(brick, wl.cams[0], dtf, DT, ERT, BACKGROUND, frame8, wl.W, wl.H)
    torch.cuda.synchronize(d)
    brick.close()


def nvlink_sweep(ep, device) -> dict:
    """Measured link peak for the compositor roofline: NCCL send/recv between rank pairs (r, r XOR 1), all
    pairs at once, both directions, 16-256 MiB messages; per-direction GB/s, best size, min over ranks."""
    import torch
    import torch.distributed as dist

    R, r = ep.R, ep.rank
    partner = r ^ 1
    stream = torch.cuda.current_stream(device)
    best = 0.0
    sizes = (16 << 20, 64 << 20, 256 << 20)
    per = {}
    for nbytes in sizes:
        s = torch.empty(nbytes // 4, dtype=torch.float32, device=device).fill_(1.0)
        q = torch.empty_like(s)
        ok = partner < R

        def once():
            if ok:
                ep.exchange([(partner, s)], [(partner, q)])

        for _ in range(2):
            once()
        dist.barrier()
        torch.cuda.synchronize(device)
        ms = events_ms(once, 5, stream) if ok else float("inf")
        gbs = nbytes / (ms * 1e-3) / 1e9 if ok else 0.0
        t = torch.tensor([gbs], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        per[nbytes >> 20] = float(t.item())
        best = max(best, per[nbytes >> 20])
        del s, q
    return {"peak_gbs": best, "per_size_MiB": per,
            "how": "NCCL batch_isend_irecv between r and r^1 (all pairs at once), per-direction GB/s, min over ranks"}


def per_rank_leg(cfg: str, strategy: str, device, steps: int, warmup: int, R_virtual: int = 8,
                 cpu: bool = False) -> dict:
    """Config 3 / 4 per-GPU work on ONE GPU: each of the R_virtual ranks' bricks generated and marched alone
    (RGBA partial, the multi-rank step's march call), CUDA events, clocks sampled; slowest rank = the
    8-GPU frame's march critical path.  Roofline per GPU over the frame: every GPU waits for the slowest."""
    import torch

    from paper_2501_01628_b200 import device as dev

    wl = build_workload(cfg, R_virtual, strategy, mass_device=device)
    torch.cuda.empty_cache()
    dtf = dev.DeviceTF(wl.tf, device)
    cam = wl.cams[0]
    W, H = wl.W, wl.H
    part = torch.empty(W * H * 4, dtype=torch.float32, device=device)
    ranks = []
    peak, kind = load_peaks()
    with ClockSampler(device.index) as clocks:
        for r in range(R_virtual):
            desc = wl.dec.brick(r)
            brick = dev.DeviceBrick(desc, device).generate(wl.field)
            m = march_leg(dev, brick, desc, cam, dtf, wl.tf, W, H, steps, fused=False, partial=part)
            m.update({"rank": r, "box": [list(map(int, wl.dec.boxes[r][0])), list(map(int, wl.dec.boxes[r][1]))]})
            ranks.append(m)
            brick.close()
            del brick
            torch.cuda.empty_cache()
    slow = max(ranks, key=lambda x: x["kernel_ms"])
    mx = slow["kernel_ms"]
    alg = sum(x["algorithmic_bytes"] for x in ranks)
    need = sum(x["needed_bytes"] for x in ranks)
    out = {"workload": wl.text, "decomposition": strategy, "order": wl.dec.visibility_order(cam.position),
           "slowest_rank": slow["rank"], "slowest_march_ms": mx,
           "mean_march_ms": sum(x["kernel_ms"] for x in ranks) / len(ranks),
           "march_critical_path_frames_per_s": 1000.0 / mx,
           "frame_roofline_per_gpu": {
               "frac_needed": need / R_virtual / (mx * 1e-3) / 1e9 / peak,
               "frac_survey_8d_bytes": alg / R_virtual / (mx * 1e-3) / 1e9 / peak,
               "slowest_rank_frac_needed": slow["frac_needed"], "slowest_rank_frac_survey_8d_bytes": slow["frac"],
               "note": "needed bytes = f32 voxels of the macrocells the march shades in (dprt_march_stats); SURVEY "
                       "8(d) bytes count whole bricks, which a skipping marcher never reads in full (above 1 on "
                       "light or oversized mass-balanced bricks)",
               "peak": peak, "peak_kind": peak_kind_text(kind),
               "how": "sum over ranks of bytes / (ranks x slowest rank's march ms) / peak: every GPU of the "
                      "frame waits for the slowest march"},
           "exchange_bytes_per_rank_unclipped": int((1 - 1 / R_virtual) * W * H * 16),
           "rgb8_into_root_bytes": int((R_virtual - 1) / R_virtual * W * H * 3),
           "ranks": [{"rank": x["rank"], "box": x["box"], "kernel_ms": x["kernel_ms"], "frac_needed": x["frac_needed"],
                      "frac_survey_8d_bytes": x["frac"], "algorithmic_bytes": x["algorithmic_bytes"],
                      "needed_bytes": x["needed_bytes"], "footprint_px": x["footprint_px"],
                      "shaded_samples": x["shaded_samples"], "contributing_samples": x["contributing_samples"],
                      "shaded_samples_per_s": x["shaded_samples_per_s"]} for x in ranks],
           "clocks": clocks.summary()}
    if cfg == "c3":
        log(f"[bench] {cfg} fused march + exchange (p2p_push) of the slowest rank, emulated on this GPU")
        out["p2p_push_slowest_rank"] = push_leg(wl, slow["rank"], device)
    if cpu:
        log(f"[bench] {cfg} CPU baseline (oracle, strided 1/64 pixel lattice, {R_virtual} bricks)")
        res, _, _ = cpu_baseline_lattice(wl, cam, 8)
        out["cpu_baseline"] = res
        g = ref_gather_baseline(W, H, R_virtual)
        if g is not None:
            out["reference_gather"] = g
    return out


def push_leg(wl: "Workload", rank: int, device, steps: int = 10) -> dict:
    """The fused march + exchange (p2p_push) of one config-3 rank on ONE GPU: its brick
    marched with every row block pushed into that block owner's inbox slot (all eight inboxes local here, so
    this times the kernel's work, not NVLink) and the same march into a local band-clipped partial; then the
    owner side -- the epoch-flag wait and the blend of one row block from the eight inbox slots, tone-mapped
    into the frame with the completion signal -- against the plain ranged blend.  Stream-ordered on one
    stream: every wait is satisfied when issued (no kernel waits on another)."""
    import torch

    from paper_2501_01628_b200 import device as dev
    from paper_2501_01628_b200.p2p import PushLayout

    P, W, H = wl.dec.P, wl.W, wl.H
    cam = wl.cams[0]
    dtf = dev.DeviceTF(wl.tf, device)
    L = PushLayout(P, W, H, 16)
    inbox = [torch.zeros(L.inbox_pixels() * 4, dtype=torch.float32, device=device) for _ in range(P)]
    flags = [torch.zeros(L.flag_words(), dtype=torch.int32, device=device) for _ in range(P)]
    ib, fb = [t.data_ptr() for t in inbox], [t.data_ptr() for t in flags]
    bands = [tuple(dev.desc_footprint(wl.dec.brick(s), cam, W, H)[1::2]) for s in range(P)]
    order = wl.dec.visibility_order(cam.position)
    brick = dev.DeviceBrick(wl.dec.brick(rank), device).generate(wl.field)
    part = torch.empty(W * H * 4, dtype=torch.float32, device=device)
    frame = torch.empty(W * H * 3, dtype=torch.uint8, device=device)
    stream = torch.cuda.current_stream(device)
    epoch = [0]

    def push():
        epoch[0] += 1
        dst, fl = L.march_targets(ib, fb, rank, epoch[0])
        dev.march_push(brick, cam, dtf, DT, ERT, W, H, L.row_start, dst, fl, fb[rank] + L.counter_offset(0), epoch[0],
                       band_clear=True)

    def local():
        dev.march(brick, cam, dtf, DT, ERT, part, W, H, band_clear=True)

    owner = 0
    rows = L.blocks[owner]
    npix = (rows[1] - rows[0]) * W

    def blend_push():
        # the owner's side of frame `epoch`: every source's flag was raised by `prime` below
        dev.wait_flags(device.index, fb[owner], P, epoch[0])
        ptrs, ranges, _ = L.fragments(ib[owner], owner, epoch[0], order, bands)
        dev.composite_signal(device.index, ptrs, npix, BACKGROUND, frame.data_ptr() + 3 * rows[0] * W, 0, ranges,
                             fb[owner] + L.counter_offset(1), [fb[0] + 4 * (P + owner)], epoch[0])

    def blend_plain():
        ptrs, ranges, _ = L.fragments(ib[owner], owner, epoch[0], order, bands)
        dev.composite_ptrs(device.index, ptrs, npix, BACKGROUND, rgb8_ptr=frame.data_ptr() + 3 * rows[0] * W,
                           ranges=ranges)

    for _ in range(3):
        push()
        local()
    torch.cuda.synchronize(device)
    with ClockSampler(device.index) as clocks:
        push_ms = events_ms(push, steps, stream)
        local_ms = events_ms(local, steps, stream)
        # raise every source's flag of the current epoch (the other ranks' marches, already complete)
        for s in range(P):
            for w in range(P):
                flags[w][s] = epoch[0]
        torch.cuda.synchronize(device)
        wait_blend_ms = graph_ms(blend_push, 20, device)
        blend_ms = graph_ms(blend_plain, 20, device)
    brick.close()
    sent = sum((min(b[1], bands[rank][1]) - max(b[0], bands[rank][0])) * W for j, b in enumerate(L.blocks)
               if j != rank and min(b[1], bands[rank][1]) > max(b[0], bands[rank][0]))
    return {"rank": rank, "push_march_ms": push_ms, "local_band_march_ms": local_ms,
            "push_over_local": push_ms / local_ms,
            "owner_wait_and_blend_ms": wait_blend_ms, "owner_plain_blend_ms": blend_ms,
            "fragment_bytes_pushed": 16 * sent,
            "note": "one GPU: the eight inboxes are local, so this is the kernels' own cost; on 8 GPUs the pushed "
                    "rows cross NVLink during the march instead of after it (DESIGN.md §6)",
            "clocks": clocks.summary()}


def push_frames_leg(renderer, cams, W: int, H: int, opts, steps: int, warmup: int, stream, device) -> dict:
    """N > 1, every rank on its own GPU: the same frames rendered with the fused march + exchange
    (composite='p2p_push': the march writes its row blocks into their owners' inboxes over
    NVLink, no per-frame collective), timed like ``value`` (CUDA events on the rank's stream, max over
    ranks).  Reported beside ``value``, never instead of it.  The outcome is combined over a gloo group: a
    rank whose flag wait failed (its CUDA context is then gone) still reports, and cannot hang its peers
    inside an NCCL collective."""
    import dataclasses

    import torch
    import torch.distributed as dist

    g = dist.new_group(backend="gloo")
    ms, err = float("inf"), ""
    try:
        po = dataclasses.replace(opts, composite="p2p_push")
        for k in range(warmup):
            renderer.render(cams[k % len(cams)], W, H, po, verify=False)
        torch.cuda.synchronize(device)
        dist.barrier(group=g)
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for k in range(steps):
            renderer.render(cams[k % len(cams)], W, H, po, verify=False)
        end.record(stream)
        torch.cuda.synchronize(device)
        ms = start.elapsed_time(end) / steps
    except Exception as ex:  # reported in the line; the main measurement above stands
        err = f"{type(ex).__name__}: {ex}"[:400]
    lost = 0.0
    if err:
        try:  # does this rank's CUDA context still work?
            torch.cuda.synchronize(device)
            torch.zeros(1, device=device).item()
        except Exception:  # noqa: BLE001
            lost = 1.0
    t = torch.tensor([ms, 0.0 if not err else 1.0, lost], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=g)
    errs = [None] * dist.get_world_size()
    dist.all_gather_object(errs, err, group=g)
    out = {"composite": "p2p_push", "ms_per_step_max_over_ranks": None, "value": None,
           "how": "renderer.render(..., composite='p2p_push') x steps after warmup, CUDA events, max over ranks"}
    if t[1] == 0:
        out["ms_per_step_max_over_ranks"] = float(t[0])
        out["value"] = 1000.0 / float(t[0])
    else:
        out["errors"] = {r: e for r, e in enumerate(errs) if e}
        out["cuda_context_lost"] = bool(t[2])
    return out


def c3_one_rank_leg(device, steps: int = 20, warmup: int = 3) -> dict:
    """The N > 1 workload family (config-3 family: 1024^3 cells per rank at 3840x2160) at ONE rank -- one
    1024^3 brick, the single-rank fused frame, two frames in flight like ``value`` -- so that the N > 1 lines
    (weak scaling of this family) have a same-workload N = 1 reference; the N = 1 ``value`` itself is
    BASELINE's config 2."""
    import torch

    from paper_2501_01628_b200 import device as dev
    from paper_2501_01628_b200.engine import RenderOptions, VolumeRenderer
    from paper_2501_01628_b200.transport import SoloEndpoint

    wl = build_workload("c3", 1, "even")
    brick = dev.DeviceBrick(wl.dec.brick(0), device).generate(wl.field)
    renderer = VolumeRenderer(SoloEndpoint(device), brick, wl.dec, wl.tf, BACKGROUND)
    opts = RenderOptions(dt=DT, ert=ERT, frames_in_flight=2)
    stream = torch.cuda.current_stream(device)
    for _ in range(warmup):
        renderer.render(wl.cams[0], wl.W, wl.H, opts, verify=False)
    renderer.join(stream)
    torch.cuda.synchronize(device)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device.index) as clocks:
        start.record(stream)
        for _ in range(steps):
            renderer.render(wl.cams[0], wl.W, wl.H, opts, verify=False)
        renderer.join(stream)
        end.record(stream)
        torch.cuda.synchronize(device)
    ms = start.elapsed_time(end) / steps
    brick.close()
    del renderer, brick
    torch.cuda.empty_cache()
    return {"workload": wl.text, "value": 1000.0 / ms, "unit": UNIT, "ms_per_step": ms, "steps": steps,
            "frames_in_flight": 2, "config": wl.config(1), "clocks": clocks.summary(),
            "note": "same-workload N = 1 reference for the N > 1 lines (weak scaling of the config-3 family); "
                    "value_N / value_1 across the driver's N = 1 (config 2) and N > 1 lines compares different "
                    "workloads"}


def c4_orbit_leg(device, steps: int = 5, every: int = 6) -> dict:
    """Config 4 on one GPU: the lander-like field's 8 uneven mass-balanced bricks all resident, every
    ``every``-th frame of the 36-frame orbit; per frame every rank's march timed alone (the sort-last frame
    waits for the slowest) and the visibility order recorded.  Reports the load imbalance the orbit causes."""
    import torch

    from paper_2501_01628_b200 import device as dev

    wl = build_workload("c4", 8, "mass", mass_device=device)
    torch.cuda.empty_cache()
    dtf = dev.DeviceTF(wl.tf, device)
    bricks = [dev.DeviceBrick(wl.dec.brick(r), device).generate(wl.field) for r in range(8)]
    part = torch.empty(wl.W * wl.H * 4, dtype=torch.float32, device=device)
    stream = torch.cuda.current_stream(device)
    frames = []
    with ClockSampler(device.index) as clocks:
        for i in range(0, len(wl.cams), every):
            cam = wl.cams[i]
            ms = []
            for b in bricks:
                for _ in range(2):
                    dev.march(b, cam, dtf, DT, ERT, part, wl.W, wl.H)
                torch.cuda.synchronize(device)
                ms.append(events_ms(lambda: dev.march(b, cam, dtf, DT, ERT, part, wl.W, wl.H), steps, stream))
            frames.append({"frame": i, "order": wl.dec.visibility_order(cam.position), "max_ms": max(ms),
                           "mean_ms": sum(ms) / len(ms), "rank_ms": ms})
    for b in bricks:
        b.close()
    del bricks, part
    torch.cuda.empty_cache()
    return {"workload": wl.text + ", 8 mass-balanced bricks", "bricks": [[list(map(int, lo)), list(map(int, hi))]
                                                                       for lo, hi in wl.dec.boxes],
            "frames": frames, "mean_slowest_ms": sum(f["max_ms"] for f in frames) / len(frames),
            "mean_imbalance": sum(f["max_ms"] / f["mean_ms"] for f in frames) / len(frames),
            "distinct_orders": len({tuple(f["order"]) for f in frames}), "clocks": clocks.summary()}


def c5_blend_leg(device, steps: int = 20) -> dict:
    """Config 5's per-rank compute on one GPU: the blend + tone map of a rank's row block from P fragments
    (what each rank runs after the exchange), 1080p-8K x P = 2, 4, 8; bytes = 16 B x P fragments in + 3 B
    out per pixel, GB/s against the HBM copy peak."""
    import torch

    from paper_2501_01628_b200 import device as dev

    peak, kind = load_peaks()
    rows = []
    stream = torch.cuda.current_stream(device)
    g = torch.Generator(device=device)
    g.manual_seed(5)
    with ClockSampler(device.index) as clocks:
        for (W, H) in ((1920, 1080), (3840, 2160), (7680, 4320)):
            for P in (2, 4, 8):
                n = (H // P) * W
                nbytes = 16 * P * n + 3 * n
                # rotate over enough fragment sets that consecutive launches never find their inputs in L2
                nsets = max(2, -(-3 * 126_000_000 // nbytes))
                sets = [[torch.rand(n * 4, generator=g, device=device) * 0.5 for _ in range(P)] for _ in range(nsets)]
                out = torch.empty(n * 3, dtype=torch.uint8, device=device)
                k = [0]

                def fn():
                    dev.composite(sets[k[0] % nsets], BACKGROUND, rgb8=out)
                    k[0] += 1

                for _ in range(3):
                    fn()
                torch.cuda.synchronize(device)
                ms = graph_ms(fn, max(steps, 2 * nsets), device)
                rows.append({"image": [W, H], "P": P, "block_px": n, "ms": ms, "GBps": nbytes / (ms * 1e-3) / 1e9,
                             "frac_hbm": nbytes / (ms * 1e-3) / 1e9 / peak, "input_sets": nsets})
                del sets, out
    return {"what": "per-rank blend + tone map of a row block (H/P rows) from P fp32 RGBA fragments; "
                    "launches captured in one CUDA graph, replay timed with CUDA events (no host launch gaps between "
                    "these 10-90 us kernels), rotating over input sets > 3x L2 so no launch reads L2-resident "
                    "fragments", "rows": rows,
            "peak": peak, "peak_kind": peak_kind_text(kind), "clocks": clocks.summary()}


def triangle_trace_leg(device, n_tri: int = 200_000, W: int = 1920, H: int = 1080, steps: int = 10) -> Optional[dict]:
    """SURVEY §8(f) row 4 (triangle half): the reference's own per-rank compute slot -- numba
    trace_nearest_batch / trace_any_batch over its BVH (pkg/src/dprt/bvh.py:284-311) -- against
    dprt_trace_nearest / dprt_trace_any (csrc/trace.cu, bit-identical) on the same Accel and the same
    1920x1080 primary rays of the reference's auto camera; the reference install in baseline/_ref builds the
    scene and BVH and runs the CPU side (one thread, as each rank runs it).  None without that install."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "dprt").exists():
        return None
    import torch

    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/dprt_numba_cache")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    from dprt import bvh as ref_bvh, cli as ref_cli, engine as ref_engine, scene as ref_scene

    from paper_2501_01628_b200 import trace

    sc = ref_scene.generate_uneven_cloud(7, n_tri, 8)
    acc = ref_bvh.build_bvh(sc.triangles)
    cam = ref_cli.default_camera(sc, W, H)

    class _Ep:
        rank, R = 0, 1

    prim = ref_engine.gen_primary_batch(_Ep(), cam, W, H)
    n = len(prim)
    args = (acc.node_lo, acc.node_hi, acc.node_left, acc.node_right, acc.node_first, acc.node_count, acc.root,
            acc.tri_v, acc.tri_id)
    # CPU: the numba slot on every 50th ray (a sample spread over the frame; compile excluded)
    sel = np.arange(0, n, 50)
    k = len(sel)
    s_org, s_dir = np.ascontiguousarray(prim.org[sel]), np.ascontiguousarray(prim.dirn[sel])
    s_t0, s_t1 = np.ascontiguousarray(prim.tmin[sel]), np.ascontiguousarray(prim.tmax[sel])
    bt, bi = np.full(k, np.inf), np.full(k, trace.MISS_ID, np.int64)
    ref_bvh.trace_nearest_batch(*args, s_org[:64], s_dir[:64], s_t0[:64], s_t1[:64], bt[:64], bi[:64])
    bt[:], bi[:] = np.inf, trace.MISS_ID
    t0 = time.perf_counter()
    ref_bvh.trace_nearest_batch(*args, s_org, s_dir, s_t0, s_t1, bt, bi)
    cpu_s = time.perf_counter() - t0
    # GPU: all rays, device resident, events
    b = trace.DeviceBvh.from_accel(acc, device)
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
    org, dirn, tmin, tmax = dv(prim.org), dv(prim.dirn), dv(prim.tmin), dv(prim.tmax)
    best_t = torch.full((n,), float("inf"), dtype=torch.float64, device=device)
    best_id = torch.full((n,), int(trace.MISS_ID), dtype=torch.int64, device=device)

    def once():
        best_t.fill_(float("inf"))
        best_id.fill_(int(trace.MISS_ID))
        b.trace_nearest(org, dirn, tmin, tmax, best_t, best_id)

    for _ in range(3):
        once()
    torch.cuda.synchronize(device)
    ms = events_ms(once, steps, torch.cuda.current_stream(device))
    sel_t = torch.from_numpy(sel).to(device)
    same = bool(np.array_equal(best_t[sel_t].cpu().numpy().view(np.uint64), bt.view(np.uint64)) and
                np.array_equal(best_id[sel_t].cpu().numpy(), bi))
    hits = int((best_id != int(trace.MISS_ID)).sum().item())
    return {"what": "nearest-hit traversal of the reference's BVH (200k-triangle uneven cloud, one rank) for the "
                    f"{W}x{H} primary rays of its auto camera",
            "rays": n, "hits": hits, "gpu_ms": ms, "gpu_rays_per_s": n / (ms * 1e-3),
            "reference_numba_rays_per_s": k / cpu_s, "reference_sample_rays": k,
            "speedup": (n / (ms * 1e-3)) / (k / cpu_s), "bit_identical_on_sample": same,
            "timing": "GPU: CUDA events over 10 launches incl. the 2 result resets; CPU: one numba call over every "
                      "50th ray, 1 thread (each reference rank runs its slot on one thread)"}


def composite_sweep(ep, device, sizes, modes, steps: int) -> list:
    """Config 5: random premultiplied RGBA partials (alpha <= 0.5), every rank composites with each mode;
    device ms per frame (max over ranks), fragment bytes moved, GB/s."""
    import torch
    import torch.distributed as dist

    from paper_2501_01628_b200.compositor import Compositor

    out = []
    R = ep.R
    g = torch.Generator(device=device)
    for (W, H) in sizes:
        for mode in modes:
            g.manual_seed(1234 + ep.rank)
            comp = Compositor(ep, W, H, mode, device)
            part = comp.shared_partial()
            if part is None:
                part = torch.empty(W * H * 4, dtype=torch.float32, device=device)
            rgba = torch.rand(W * H * 4, generator=g, device=device, dtype=torch.float32)
            a = rgba[3::4] * 0.5
            rgba[0::4] *= a
            rgba[1::4] *= a
            rgba[2::4] *= a
            rgba[3::4] = a
            part.copy_(rgba)
            del rgba
            order = list(range(R))[::-1]
            for _ in range(2):
                comp.composite(part, order, BACKGROUND)
            if R > 1:
                dist.barrier()
            torch.cuda.synchronize(device)
            ms = events_ms(lambda: comp.composite(part, order, BACKGROUND), steps, torch.cuda.current_stream(device))
            t = torch.tensor([ms, float(comp.last_bytes)], dtype=torch.float64, device=device)
            if R > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            out.append({"image": [W, H], "mode": comp.mode, "ms": float(t[0]), "fragment_bytes_per_rank": int(t[1]),
                        "GBps_per_rank": float(t[1]) / (float(t[0]) * 1e-3) / 1e9 if t[0] > 0 else None})
            comp.close() if hasattr(comp, "close") else None
            del comp, part
            torch.cuda.empty_cache()
    return out


# --------------------------------------------------------------------------------------------------
# our arm


def launch_ranks(args) -> int:
    """``--gpus N`` without a launcher: run the N ranks under torch.distributed.run (127.0.0.1)."""
    import torch

    n_dev = torch.cuda.device_count()
    env = dict(os.environ)
    if n_dev < args.gpus:
        log(f"[bench] {args.gpus} ranks on {n_dev} visible GPU(s): ranks share GPUs over a gloo control plane "
            "(functional run, not a measurement)")
        env["DPRT_BENCH_BACKEND"] = "gloo"
    else:
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2501_01628_b200 import device as dev
    from paper_2501_01628_b200.engine import RenderOptions, VolumeRenderer
    from paper_2501_01628_b200.transport import DistEndpoint, SoloEndpoint, init_dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    shared = False
    backend = "none"
    if world > 1:
        backend = os.environ.get("DPRT_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            ep = init_dist("nccl")
            device = ep.device
        else:
            # functional mode: gloo control plane, ranks possibly sharing a GPU -- never a measurement
            device = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
            torch.cuda.set_device(device)
            dist.init_process_group(backend)
            ep = DistEndpoint(device=device)
            shared = torch.cuda.device_count() < world
    else:
        device = torch.device("cuda", 0)
        torch.cuda.set_device(device)
        ep = SoloEndpoint(device)
    rank, R = ep.rank, ep.R
    if args.gpus != R and not (args.gpus == 1 and R == 1):
        log(f"[bench] note: --gpus {args.gpus} but WORLD_SIZE {R}; reporting n_gpus = {R}")
    cfg = resolve_config(args.config, R)
    if cfg == "c5":
        return run_c5(args, ep, device, R, shared, backend)
    if args.per_rank:
        return run_per_rank(args, device, cfg)

    wl = build_workload(cfg, R, args.decomposition, mass_device=device)
    torch.cuda.empty_cache()
    f, dec, tf, W, H = wl.field, wl.dec, wl.tf, wl.W, wl.H
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
    cams = wl.cams
    torch.cuda.synchronize(device)

    def barrier():
        if R > 1:
            dist.barrier()
        torch.cuda.synchronize(device)

    k_step = [0]

    def step():
        renderer.render(cams[k_step[0] % len(cams)], W, H, opts, verify=False)
        k_step[0] += 1

    # ---- device-resident throughput (value); the clock sampler starts first, so its own start-up (NVML,
    # nvidia-smi) overlaps the warm-up rather than the timed region
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device.index) as clocks:
        warm = spin_up(lambda k: step(), args.warmup, device, R)
        renderer.join(stream)
        barrier()
        k_step[0] = 0
        clocks.mark()
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
    cam = cams[0]

    # ---- compositing exchange alone (N > 1): fragments over NVLink + blend + gather, max over ranks; the
    # link peak measured in the same run (NCCL send/recv sweep)
    nvlink = None
    if R > 1:
        order = renderer.decomposition.visibility_order(cam.position)
        comp = renderer.compositor
        bands = renderer._bands(cam, W, H) if comp.clips_bands() else None
        barrier()
        comp_ms = events_ms(lambda: comp.composite(renderer.partial, order, BACKGROUND, bands=bands), args.steps,
                            stream)
        cms = torch.tensor([comp_ms, float(comp.last_bytes)], dtype=torch.float64, device=device)
        dist.all_reduce(cms, op=dist.ReduceOp.MAX)
        comp_ms, frag_bytes = float(cms[0]), int(cms[1])
        full_bytes = int((1 - 1 / R) * W * H * (8 if args.fragments == "f16" else 16))
        gather_bytes = int((R - 1) / R * W * H * 3)
        link = nvlink_sweep(ep, device) if not shared else {"peak_gbs": None, "how": "ranks share a GPU"}
        achieved_nv = frag_bytes / (comp_ms * 1e-3) / 1e9
        lp = link.get("peak_gbs")
        nvlink = {"bound": "nvlink", "achieved": achieved_nv, "peak": lp, "unit": "GB/s",
                  "frac": achieved_nv / lp if lp else None, "peak_kind": link["how"], "link_sweep": link,
                  "composite_ms": comp_ms, "fragment_bytes_per_rank": frag_bytes,
                  "unclipped_fragment_bytes_per_rank": full_bytes, "rgb8_into_root": gather_bytes,
                  "mode": comp.mode, "clipped_to_footprint_rows": bands is not None}

    # ---- marcher alone (roofline) + instrumented march (needed bytes, shaded samples)
    barrier()
    roof = march_leg(dev, brick, desc, cam, renderer.dtf, tf, W, H, args.steps, fused=(R == 1),
                     partial=renderer.partial, band_clear=R > 1 and renderer.compositor.clips_bands())
    if R > 1:
        t = torch.tensor([roof["kernel_ms"]], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        roof["kernel_ms_max_over_ranks"] = float(t.item())

    # ---- end to end through the engine's host-buffer call (render_to_host)
    pinned_tf = torch.from_numpy(tf.as_f32().reshape(-1)).pin_memory()
    from paper_2501_01628_b200.device import camera_struct
    import ctypes

    h2d = pinned_tf.numel() * 4 + ctypes.sizeof(camera_struct(cam))
    d2h = W * H * 3 if rank == 0 else 0
    depth = 2  # frames in flight: the host waits for frame k-2's bytes while k-1 and k are queued
    host_frames = [torch.empty((H, W, 3), dtype=torch.uint8).pin_memory() for _ in range(depth + 1)]
    inflight = []

    def e2e_step(k):
        renderer.dtf.update(tf, staging=pinned_tf)
        hf = renderer.render_to_host(cams[k % len(cams)], W, H, host_frames[k % (depth + 1)] if rank == 0 else None,
                                     opts, verify=True)
        inflight.append(hf)
        if len(inflight) > depth:
            inflight.pop(0).wait()

    def drain():
        while inflight:
            inflight.pop(0).wait()

    def timed_host(fn, n) -> float:
        barrier()
        t0 = time.perf_counter()
        for k in range(n):
            fn(k)
        drain()
        barrier()
        s = time.perf_counter() - t0
        t = torch.tensor([s], dtype=torch.float64, device=device)
        if R > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    spin_up(e2e_step, args.warmup, device, R)
    drain()
    d2h0 = renderer.d2h_bytes
    e2e_fps = args.steps / timed_host(e2e_step, args.steps)
    if rank == 0:  # the read-back bytes actually copied (only the footprint rectangle once a buffer holds a frame)
        d2h = (renderer.d2h_bytes - d2h0) / args.steps

    # ---- end to end through the reference-facing API (Device/World/Frame -> render_frame_collective ->
    # map_frame, api.py:329-371): the transfer function is edited and re-committed every 8th frame (so the
    # TF upload and the skip-distance rebuild run inside the timed loop), pixels mapped on rank 0
    api = api_e2e(ep, device, wl, args)

    # ---- N > 1: the fused march + exchange (p2p_push) on the same frames, last (a failed flag wait ends
    # this process's CUDA context; everything measured above is already on the host)
    comp_mode = renderer.compositor.mode if R > 1 else "single (fused into the march)"
    push_frames = None
    push_env = os.environ.get("DPRT_BENCH_PUSH", "1")
    if R > 1 and push_env != "0" and (not shared or push_env == "force"):
        log("[bench] fused march + exchange (p2p_push) frames")
        push_frames = push_frames_leg(renderer, cams, W, H, opts, args.steps, max(args.warmup, 3), stream, device)
    context_lost = bool(push_frames and push_frames.get("cuda_context_lost"))

    cpu = None
    extras = {}
    if rank == 0 and R == 1 and not args.no_cpu_baseline and cfg in ("c1", "c2", "c3"):
        log("[bench] timing the CPU oracle on a row sample")
        cpu = cpu_baseline_rows(brick.download(), wl)
    if not context_lost:
        brick.close()
        del renderer, brick
        torch.cuda.empty_cache()
    if R == 1 and cfg == "c2" and not args.no_extras:
        # config 3 (the north-star target) on this one GPU: every rank's brick of the 2048^3 field marched
        # alone under clocks, even 2x2x2 and mass-balanced kd splits, + its CPU baseline
        log("[bench] config 3 per-rank leg (8 bricks of 2048^3 at 3840x2160)")
        extras["c3_per_rank"] = {s: per_rank_leg("c3", s, device, 10, 3, cpu=(s == "even") and not args.no_cpu_baseline)
                                 for s in ("even", "mass")}
        log("[bench] config-3 family at one rank (the N > 1 lines' weak-scaling reference)")
        extras["c3_family_one_rank"] = c3_one_rank_leg(device)
        log("[bench] config 4 orbit leg and config 5 blend leg")
        extras["c4_orbit"] = c4_orbit_leg(device)
        extras["c5_blend"] = c5_blend_leg(device)
        log("[bench] triangle traversal leg (the reference's numba slot vs dprt_trace_nearest)")
        tri = triangle_trace_leg(device)
        if tri is not None:
            extras["f4_triangle_trace"] = tri
    if rank == 0 and R == 1 and not args.no_traffic:
        log("[bench] ncu child: DRAM bytes of one march launch")
        tr = measure_traffic(cfg)
        if "dram_bytes" in tr:
            roof["traffic"] = tr["dram_bytes"]
            roof["frac_traffic"] = tr["dram_bytes"] / (roof["kernel_ms"] * 1e-3) / 1e9 / roof["peak"]
            if tr.get("warp_instructions") and roof["shaded_samples"]:
                # per lane-sample: a warp instruction serves up to 32 lanes' samples
                roof["warp_instructions_per_shaded_sample"] = tr["warp_instructions"] / roof["shaded_samples"]
            if tr.get("thread_instructions") and roof["shaded_samples"]:
                roof["thread_instructions_per_shaded_sample"] = tr["thread_instructions"] / roof["shaded_samples"]
            if tr.get("warp_instructions"):
                # the compute-side roofline of this latency / issue-bound kernel: warp instructions per second
                # against 4 issue slots per SM per cycle at the max SM clock
                sms = torch.cuda.get_device_properties(device).multi_processor_count
                mhz = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("sm_max_mhz", 1965.0)) \
                    if (ROOT / "MEASURED_PEAKS.json").exists() else 1965.0
                ipeak = sms * 4 * mhz * 1e6
                roof["issue_roofline"] = {"achieved_warp_inst_per_s": tr["warp_instructions"] / (roof["kernel_ms"] * 1e-3),
                                          "peak_warp_inst_per_s": ipeak,
                                          "frac": tr["warp_instructions"] / (roof["kernel_ms"] * 1e-3) / ipeak,
                                          "how": f"{sms} SMs x 4 schedulers x {mhz:.0f} MHz"}
        roof["traffic_probe"] = tr

    if rank == 0:
        # per frame: R == 1 -> march_beam alone (background fill and tone map fused into it); R > 1 ->
        # march_beam + composite (+ NCCL's own kernels for the barriers)
        launches = args.steps * (1 if R == 1 else 2)
        line = {
            "metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": R, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": wl.scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": wl.config(R),
            "run": {"warmup_steps_run": warm,
                    "warmup_rule": "W steps, then more until the GPU has been busy 0.2 s (spin_up: no timed region "
                                   "starts at an idle-lowered clock)",
                    "composite": comp_mode,
                    "fragments": args.fragments, "frames_in_flight": fif, "empty_space_skipping": skip},
            "roofline": roof,
            "e2e": {"value": e2e_fps, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "d2h_note": "the RGB8 frame is read back into reused pinned buffers: the first frame of a "
                                "buffer whole, later ones only the footprint rectangle (plus earlier rectangles) -- "
                                "outside it the march writes the background, which the buffer already holds",
                    "path": "VolumeRenderer.render_to_host (TF from pinned memory, digest verified, RGB8 read-back)"},
            "api_e2e": api,
            "gpu_launches": launches,
            "compositor_roofline": nvlink,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
            "backend": backend if R > 1 else "single",
        }
        if push_frames is not None:
            line["p2p_push_frames"] = push_frames
        if shared:
            line["measurement"] = False
            line["note"] = f"{R} ranks shared {torch.cuda.device_count()} GPU(s) over gloo: functional run only"
        line.update(extras)
        print(json.dumps(line), flush=True)
    if context_lost:  # NCCL teardown on a lost context can block: the line is out, leave now
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)
    if R > 1:
        dist.destroy_process_group()


def api_e2e(ep, device, wl: Workload, args) -> dict:
    """Frames/s through the drop-in API (api.py): Device -> spatialField / transferFunction1D / volume /
    world / camera / renderer / frame; every step render_frame_collective + map_frame(...).pixels on rank 0;
    every 8th frame the TF opacity is edited and re-committed."""
    import torch
    import torch.distributed as dist

    from paper_2501_01628_b200 import api

    d = api.Device(ep, device)
    fld = d.create("spatialField")
    fld.set_param("dims", tuple(wl.field.dims))
    fld.set_param("generator", "blobs")
    fld.set_param("seed", wl.gen["seed"])
    fld.set_param("blobCount", 16)
    fld.set_param("lopsided", wl.gen["lopsided"])
    fld.set_param("spacing", tuple(wl.field.spacing))
    fld.commit()
    tfo = d.create("transferFunction1D")
    base = wl.tf.as_f32().copy()
    tfo.set_param("table", base)
    tfo.set_param("valueRange", (wl.tf.vmin, wl.tf.vmax))
    tfo.commit()
    vol = d.create("volume")
    vol.set_param("field", fld)
    vol.set_param("transferFunction", tfo)
    vol.set_param("decomposition", wl.strategy if ep.R > 1 else "even")
    vol.commit()
    world = d.create("world")
    world.set_param("volumes", [vol])
    world.commit()
    cam0 = wl.cams[0]
    camo = d.create("camera")
    camo.set_param("position", tuple(cam0.position))
    camo.set_param("direction", tuple(cam0.view_dir))
    camo.set_param("up", tuple(cam0.up))
    camo.set_param("fovY", cam0.fov_y)
    camo.set_param("aspect", cam0.aspect)
    camo.commit()
    rend = d.create("renderer")
    rend.set_param("background", BACKGROUND)
    rend.set_param("composite", args.composite if ep.R > 1 else "auto")
    rend.set_param("dt", DT)
    rend.set_param("ert", ERT)
    rend.commit()
    frame = d.create("frame")
    frame.set_param("world", world)
    frame.set_param("camera", camo)
    frame.set_param("renderer", rend)
    frame.set_param("size", (wl.W, wl.H))
    frame.commit()
    nbytes = [0]

    def step(k):
        if k % 8 == 7:  # edit the opacity ramp: new TF contents -> upload + skip-distance rebuild
            t = base.copy()
            t[:, 3] *= 0.9 if (k // 8) % 2 == 0 else 1.0
            tfo.set_param("table", t)
            tfo.commit()
            vol.commit()
        cam = wl.cams[k % len(wl.cams)]
        if len(wl.cams) > 1:
            camo.set_param("position", tuple(cam.position))
            camo.set_param("direction", tuple(cam.view_dir))
            camo.commit()
        frame.render()
        m = api.map_frame(frame)
        if ep.rank == 0:
            px = m.pixels if as_bytes[0] else m.array  # both wait for this frame's bytes in host memory
            nbytes[0] = frame._renderer.d2h_bytes

    as_bytes = [False]
    d2h0 = [0]

    def timed() -> float:
        spin_up(step, args.warmup, device, ep.R)
        frame.wait()
        if ep.R > 1:
            dist.barrier()
        torch.cuda.synchronize(device)
        d2h0[0] = nbytes[0]
        t0 = time.perf_counter()
        for k in range(args.steps):
            step(k)
        frame.wait()
        if ep.R > 1:
            dist.barrier()
        t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=device)
        if ep.R > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return args.steps / float(t.item())

    fps = timed()            # map_frame(frame).array: the pinned frame, no bytes copy
    d2h_step = (nbytes[0] - d2h0[0]) / args.steps
    as_bytes[0] = True
    fps_bytes = timed()      # map_frame(frame).pixels: bytes, as the reference's FrameResult returns
    frame.release() if hasattr(frame, "release") else None
    world.release() if hasattr(world, "release") else None
    torch.cuda.synchronize(device)
    return {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 16 * wl.tf.n // 8 + 200, "d2h_bytes_per_step": d2h_step,
            "value_pixels_bytes": fps_bytes,
            "path": "api.Frame.render + map_frame(frame) every frame, the frame's pixels read on rank 0 (value: the "
                    "zero-copy .array view; value_pixels_bytes: .pixels as bytes like the reference); TF edited + "
                    "committed every 8th frame; one frame at a time (the app reads frame k before rendering k+1)"}


def run_per_rank(args, device, cfg: str):
    """``--per-rank``: config 3 / 4 per-GPU work of the 8-GPU frame on this one GPU (value = 1000 / slowest
    rank's march ms: the march critical path, not a whole frame)."""
    if cfg not in ("c3", "c4"):
        raise SystemExit("--per-rank applies to c3 and c4")
    strategy = args.decomposition
    res = per_rank_leg(cfg, strategy, device, args.steps, args.warmup, cpu=not args.no_cpu_baseline)
    line = {"metric": METRIC + " [per-rank march critical path on 1 GPU]", "value": res["march_critical_path_frames_per_s"],
            "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res["slowest_march_ms"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": res["workload"] + " -- each rank's brick marched alone on one GPU",
                       "decomposition": strategy, "per_rank": True},
            "per_rank": res, "clocks": res["clocks"], "cpu_baseline": res.get("cpu_baseline"),
            "gpu_launches": 8 * args.steps}
    print(json.dumps(line), flush=True)


def run_c5(args, ep, device, R, shared, backend):
    """Config 5: compositing-only sweep, 1080p-8K partials, direct-send vs binary-swap (+ p2p) at N ranks."""
    import torch
    import torch.distributed as dist

    sizes = [(1920, 1080), (3840, 2160), (7680, 4320)]
    modes = ["direct_send", "binary_swap", "p2p"] if R > 1 else ["direct_send"]
    if R > 1 and R & (R - 1):
        modes.remove("binary_swap")
    with ClockSampler(device.index) as clocks:
        rows = composite_sweep(ep, device, sizes, modes, args.steps)
    link = nvlink_sweep(ep, device) if R > 1 and not shared else None
    head = next(r for r in rows if r["image"] == [3840, 2160])
    if ep.rank == 0:
        line = {"metric": METRIC, "value": 1000.0 / head["ms"], "unit": UNIT, "n_gpus": R, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": head["ms"], "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": "c5: compositing only, random premultiplied RGBA partials (alpha <= 0.5)",
                           "headline": f"3840x2160 {head['mode']}", "sizes": sizes, "modes": modes},
                "sweep": rows, "link": link, "clocks": clocks.summary(), "backend": backend if R > 1 else "single",
                "gpu_launches": args.steps}
        if link and link.get("peak_gbs"):
            for r in rows:
                if r["GBps_per_rank"]:
                    r["frac_link"] = r["GBps_per_rank"] / link["peak_gbs"]
        if shared:
            line["measurement"] = False
        print(json.dumps(line), flush=True)
    if R > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="auto", choices=("auto",) + CONFIGS,
                    help="BASELINE config (auto: c2 at N = 1, c3 at N > 1)")
    ap.add_argument("--per-rank", action="store_true",
                    help="c3 / c4 at N = 1: every rank's brick of the 8-GPU frame marched alone on this GPU")
    ap.add_argument("--composite", default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the config-3 per-rank leg of the default N = 1 run")
    ap.add_argument("--no-traffic", action="store_true", help="skip the ncu child run that measures DRAM bytes")
    ap.add_argument("--no-skip", action="store_true", help="disable exact empty-space skipping")
    ap.add_argument("--decomposition", default="mass", choices=["even", "mass"],
                    help="N > 1: kd split of the field, even cells or balanced by non-empty voxel count")
    ap.add_argument("--frames-in-flight", type=int, default=2,
                    help="single rank: frames marched concurrently on lane streams (1 = stream-ordered)")
    ap.add_argument("--fragments", default="f32", choices=["f32", "f16"],
                    help="exchanged RGBA fragment format at N > 1 (f16: half the bytes, fp16 tolerance)")
    ap.add_argument("--traffic-probe", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.traffic_probe:
        args.config = resolve_config(args.config, 1)
        traffic_probe(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))
    run_ours(args)


if __name__ == "__main__":
    main()
