"""Per-rank sort-last DVR frame driver: march this rank's brick, composite in visibility order, gather.

Counterpart of the reference's wavefront driver (pkg/src/dprt/engine.py): ``render_volume_with``
replaces ``render_with`` (engine.py:459-488) and ``render_volume_frame`` replaces ``render_frame``
(engine.py:491-497).  The collective contract is unchanged: the render digest is verified on every rank
before any GPU work (engine.py:410-440), pixel ownership is ``assign_pixels``' row blocks
(engine.py:216-221), the frame lands on rank 0, and ``tone_map_rgb8`` is the same formula
(engine.py:500-502) -- fused into the last compositing kernel.
"""

from __future__ import annotations

import hashlib
import json
import os
import time
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np
import torch

from . import device as dev
from .compositor import Compositor, assign_rows
from .errors import ContractError, UsageError
from .geom import CameraSpec, Vec3
from .transport import RankEndpoint
from .volume import Decomposition, TransferFunction1D, visibility_order

COMPOSITE_MODES = ("auto", "direct_send", "binary_swap", "p2p", "p2p_push", "cycle")
FRAGMENT_DTYPES = {"f32": torch.float32, "f16": torch.float16}
FUSED_SLOTS = 3  # device RGB8 frames the fused single-rank path rotates through (read-back pipeline depth)

# Distinct colours for rank-ownership visualisation, one per rank modulo 8 (engine.py:41-44).
RANK_PALETTE = np.array([
    (0.90, 0.15, 0.15), (0.15, 0.55, 0.90), (0.95, 0.75, 0.10), (0.15, 0.80, 0.35),
    (0.60, 0.30, 0.85), (0.95, 0.45, 0.10), (0.20, 0.25, 0.95), (0.80, 0.80, 0.80),
], dtype=np.float64)


def assign_pixels(width: int, height: int, num_ranks: int) -> List[Tuple[int, int]]:
    """Row blocks: rank r owns rows [r*H//R, (r+1)*H//R) (engine.py:216-221)."""
    if num_ranks < 1:
        raise ValueError(f"num_ranks must be >= 1, got {num_ranks}")
    return [(r * height // num_ranks, (r + 1) * height // num_ranks) for r in range(num_ranks)]


def tone_map_rgb8(image: np.ndarray) -> np.ndarray:
    """Host twin of the fused device tone map: clamp to [0, 1], quantize half up (engine.py:500-502)."""
    return np.floor(np.clip(image, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)


@dataclass(frozen=True)
class RenderOptions:
    """DVR render options (the reference's RenderOptions, engine.py:167-174, re-scoped to volumes)."""

    dt: float = 1.0                    # lattice spacing along the ray, world units
    ert: float = 0.99                  # early ray termination threshold (per brick)
    composite: str = "auto"            # auto | direct_send | binary_swap | p2p | p2p_push | cycle (§2.10)
    skip_empty: bool = True            # exact empty-space skipping
    disable_compositing: bool = False  # debug: root shows only its own brick (negative test, engine.py:172)
    frame_index: int = 0
    keep_float: bool = False           # also return the float RGB image before quantisation on rank 0; COLLECTIVE:
                                       # it changes the exchange (RGBA gather / peer mapping), so every rank
                                       # must pass the same value (it is part of the render digest)
    collect_samples: bool = False      # also return per-pixel owned sample counts (this rank)
    mode: str = "dvr"                  # "dvr" or "rankcolor" (rank-ownership visualisation, engine.py:327-332)
    clip_exchange: bool = True         # direct-send / p2p move only each rank's footprint rows;
                                       # RenderResult.partial is then defined only inside this rank's band
    timing: bool = False               # CUDA events around march and composite (RankStats.device_times())
    fragment_dtype: str = "f32"        # "f16": half-size RGBA fragments (march output, exchange, blend input;
                                       # direct_send / p2p / auto), DESIGN.md §6
    frames_in_flight: int = 1          # single rank: > 1 marches frames on that many lane streams, so frame
                                       # k+1 starts while frame k's last beams finish; the
                                       # current stream then does not wait for the frame: use
                                       # RenderResult.ready / VolumeRenderer.join() before reading rgb8


@dataclass
class RankStats:
    """Per-rank counters plus line records in the reference's schema (engine.py:177-193)."""

    samples: int = 0
    bytes_exchanged: int = 0
    rounds: int = 0
    records: List[str] = field(default_factory=list)
    events: Optional[tuple] = None     # (march start, march end, composite end) with RenderOptions.timing
    brick_bytes: int = 0
    _samples_dev: Optional[torch.Tensor] = None

    def device_times(self) -> dict:
        """Device milliseconds of this rank's march and composite (waits for them) and the march's
        whole-brick byte rate; needs RenderOptions.timing."""
        if self.events is None:
            raise UsageError("render with RenderOptions(timing=True) to time the kernels")
        e0, e1, e2 = self.events
        e2.synchronize()
        march = e0.elapsed_time(e1)
        return {"march_ms": march, "composite_ms": e1.elapsed_time(e2),
                "brick_GBps": self.brick_bytes / (march * 1e-3) / 1e9 if march > 0 else None}

    def owned_samples(self) -> int:
        """Owned lattice samples of this rank's brick in the frame (needs collect_samples; waits)."""
        if self._samples_dev is not None:
            self.samples = int(self._samples_dev.sum(dtype=torch.int64).item())
            self._samples_dev = None
        return self.samples

    def record(self, frame: int, rays: int, nbytes: int, millis: float, **extra) -> None:
        tail = "".join(f" {k}={v}" for k, v in extra.items())
        self.records.append(f"frame={frame} round={self.rounds} raysTraced={rays} "
                            f"bytesExchanged={nbytes} millis={millis:.3f}{tail}")
        self.rounds += 1


@dataclass
class RenderResult:
    rgb8: Optional[torch.Tensor]          # rank 0: (H, W, 3) uint8 on the device; None elsewhere
    stats: RankStats
    image: Optional[np.ndarray] = None    # rank 0 with keep_float: (H, W, 3) float64
    samples: Optional[torch.Tensor] = None  # with collect_samples: (H, W) int32, this rank's brick
    partial: Optional[torch.Tensor] = None  # this rank's RGBA partial (H, W, 4) f32 (device)
    order: Optional[List[int]] = None
    ready: Optional[torch.cuda.Event] = None  # frames_in_flight > 1: rgb8 is complete once this fires

    def wait_ready(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Order ``stream`` (default: current) after this frame's device work (a no-op unless the frame
        was rendered with frames_in_flight > 1, where the current stream does not wait by itself)."""
        if self.ready is not None:
            (stream if stream is not None else torch.cuda.current_stream()).wait_event(self.ready)


_TF_HASHES: "dict[int, tuple]" = {}


def _tf_hash(tf: TransferFunction1D) -> str:
    """sha256 of the table bytes, memoised per table object (the digest is computed every frame)."""
    key = id(tf.table)
    hit = _TF_HASHES.get(key)
    if hit is not None and hit[0] is tf.table:
        return hit[1]
    h = hashlib.sha256(tf.as_f32().tobytes()).hexdigest()
    if len(_TF_HASHES) > 64:
        _TF_HASHES.clear()
    _TF_HASHES[key] = (tf.table, h)
    return h


def rankcolor_tf(tf: TransferFunction1D, rank: int) -> TransferFunction1D:
    """Rank-ownership visualisation (the reference's "rankcolor" mode, engine.py:327-332, RANK_PALETTE
    engine.py:41-44): every entry that is visible in ``tf`` becomes opaque in this rank's palette colour,
    so the composited frame shows, per pixel, the first brick in visibility order that holds visible data."""
    t = tf.as_f32().copy()
    t[:, :3] = RANK_PALETTE[rank % len(RANK_PALETTE)]
    t[:, 3] = np.where(t[:, 3] > 0.0, 1.0, 0.0)
    return TransferFunction1D(t.astype(np.float32), tf.vmin, tf.vmax)


def render_digest(cam: CameraSpec, width: int, height: int, options: RenderOptions, tf: TransferFunction1D,
                  background: Vec3, decomposition: Decomposition) -> bytes:
    """sha256 of every collective render parameter (engine.py:410-424), extended with the transfer
    function bytes, lattice, ERT, field geometry, brick table and composite mode."""
    f = decomposition.field
    doc = {
        "cam": [list(cam.position), list(cam.view_dir), list(cam.up), cam.fov_y, cam.aspect],
        "size": [width, height],
        "dt": options.dt, "ert": options.ert, "composite": options.composite,
        "skip": options.skip_empty, "disableCompositing": options.disable_compositing, "mode": options.mode,
        "clipExchange": options.clip_exchange, "fragments": options.fragment_dtype, "keepFloat": options.keep_float,
        "tf": [_tf_hash(tf), tf.vmin, tf.vmax],
        "field": [list(f.dims), list(f.origin), list(f.spacing)],
        "bricks": [[list(lo), list(hi)] for lo, hi in decomposition.boxes],
        "background": list(background),
    }
    return hashlib.sha256(json.dumps(doc, separators=(",", ":")).encode("utf-8")).digest()


def verify_collective_digest(ep: RankEndpoint, digest: bytes) -> None:
    """Fail on every rank, before any GPU work, if digests diverge (engine.py:427-440)."""
    root_digest = ep.broadcast_from_root(digest if ep.rank == 0 else None)
    votes = ep.gather_to_root(b"\x01" if root_digest == digest else b"\x00")
    verdict = json.dumps([r for r, v in enumerate(votes) if v != b"\x01"]).encode() if ep.rank == 0 else None
    bad = json.loads(ep.broadcast_from_root(verdict))
    if bad:
        raise ContractError(f"collective render parameters diverge from rank 0 on ranks {bad}")


class VolumeRenderer:
    """Per-rank state that persists across frames: device TF, partial buffer, compositor scratch.

    One instance per rank/GPU.  ``render`` is the collective frame (all ranks call it in the same
    order with the same committed parameters)."""

    def __init__(self, ep: RankEndpoint, brick: dev.DeviceBrick, decomposition: Decomposition,
                 tf: TransferFunction1D, background: Vec3 = (0.0, 0.0, 0.0)):
        if decomposition.P != ep.R:
            raise UsageError(f"decomposition has {decomposition.P} bricks for {ep.R} ranks")
        self.ep = ep
        self.brick = brick
        self.decomposition = decomposition
        self.device = brick.device
        self.set_tf(tf)
        self.background = tuple(float(c) for c in background)
        self._size = None
        self.partial = None
        self.samples = None
        self.compositor: Optional[Compositor] = None
        self._copy_stream = None
        self._pending_copy = None
        self._fused_frames = None
        self._rank_dtf = None
        self._rank_tf_src = None
        self._fused_events = [None] * FUSED_SLOTS
        self._fused_writers = [None] * FUSED_SLOTS  # lane march that last wrote each device frame
        self._fused_next = 0
        self._fused_slot = 0
        self._lanes = []  # frames in flight: lane streams (counter slots 1..), next lane
        self._lane_next = 0
        self._band_key = None
        self._band_cache = None
        self._host_keys = {}  # host frame buffer -> (W, H, background) of the full frame it last received
        self.d2h_bytes = 0    # bytes render_to_host has copied device -> host so far (its read-back traffic)

    def set_tf(self, tf: TransferFunction1D) -> None:
        # marches of frames still in flight on lane streams may read the old table: the current stream (the
        # allocator's reuse order for the tensor being dropped) waits for them first
        if getattr(self, "dtf", None) is not None:
            self.join()
        self.tf = tf
        self.dtf = dev.DeviceTF(tf, self.brick.device)

    def _ensure(self, width: int, height: int, mode: str, fragment_dtype: str = "f32") -> None:
        if fragment_dtype not in FRAGMENT_DTYPES:
            raise UsageError(f"fragment_dtype must be one of {tuple(FRAGMENT_DTYPES)}, got {fragment_dtype!r}")
        fdt = FRAGMENT_DTYPES[fragment_dtype]
        if self._size != (width, height):
            self.samples = torch.empty(height * width, dtype=torch.int32, device=self.device)
            self.compositor = None
            self._size = (width, height)
        if self.compositor is None or self.compositor.mode_requested != mode or self.compositor.fdt != fdt:
            self.compositor = Compositor(self.ep, width, height, mode, self.device, fragment_dtype=fdt)
            shared = self.compositor.shared_partial()
            self.partial = shared if shared is not None else torch.empty(height * width * 4, dtype=fdt,
                                                                          device=self.device)

    def _bands(self, cam: CameraSpec, width: int, height: int):
        """Every rank's footprint row band [y0, y1) (host geometry, identical on all ranks; cached)."""
        key = (cam, width, height)
        if self._band_key != key:
            dec = self.decomposition
            self._band_cache = [tuple(dev.desc_footprint(dec.brick(s), cam, width, height)[1::2])
                                for s in range(self.ep.R)]
            self._band_key = key
        return self._band_cache

    def render(self, cam: CameraSpec, width: int, height: int, options: RenderOptions = RenderOptions(),
               verify: bool = True) -> RenderResult:
        if options.composite not in COMPOSITE_MODES:
            raise UsageError(f"unknown composite mode {options.composite!r}; choose from {COMPOSITE_MODES}")
        if options.mode not in ("dvr", "rankcolor"):
            raise UsageError(f"unknown render mode {options.mode!r}; choose 'dvr' or 'rankcolor'")
        if options.mode == "rankcolor":
            rc = rankcolor_tf(self.tf, self.ep.rank)
            if self._rank_dtf is None or self._rank_tf_src is not self.tf:
                if self._rank_dtf is not None:
                    self.join()  # lane marches may still read the table being replaced
                self._rank_dtf = dev.DeviceTF(rc, self.device)
                self._rank_tf_src = self.tf
            dtf = self._rank_dtf
        else:
            dtf = self.dtf
        stats = RankStats()
        if verify and self.ep.R > 1:  # one rank cannot diverge from itself
            verify_collective_digest(self.ep, render_digest(cam, width, height, options, self.tf,
                                                            self.background, self.decomposition))
        self._ensure(width, height, options.composite, options.fragment_dtype)
        order = visibility_order(self.decomposition, cam.position)
        t0 = time.perf_counter()
        ev = None
        if options.timing:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record(torch.cuda.current_stream(self.device))
            stats.brick_bytes = self.brick.desc.stored_bytes
        if self.ep.R == 1 and not options.keep_float and os.environ.get("DPRT_FUSED_SINGLE", "1") != "0":
            # one rank: the composite is just over-background + tone map -> fused into the march
            # a ring of device frames so the read-backs of frames k-1, k-2 overlap the march of frame k
            lanes = self._frame_lanes(options)
            nslots = max(FUSED_SLOTS, len(lanes) + 2)
            if self._fused_frames is None or tuple(self._fused_frames[0].shape) != (height, width, 3) or \
                    len(self._fused_frames) != nslots:
                self.join()  # old frames may still be written / read back: their memory is reused
                self._fused_frames = [torch.empty((height, width, 3), dtype=torch.uint8, device=self.device)
                                      for _ in range(nslots)]
                self._fused_events = [None] * nslots
                self._fused_writers = [None] * nslots
                self._fused_next = 0
            slot = self._fused_next
            self._fused_next = (slot + 1) % nslots
            frame = self._fused_frames[slot]
            self._fused_slot = slot
            samples = self.samples if options.collect_samples else None
            if not lanes:
                if self._fused_events[slot] is not None:
                    torch.cuda.current_stream(self.device).wait_event(self._fused_events[slot])
                    self._fused_events[slot] = None
                dev.march_rgb8(self.brick, cam, dtf, options.dt, options.ert, self.background, frame.view(-1),
                               width, height, samples=samples, skip=options.skip_empty)
                ready = None
            else:
                li = self._lane_next
                self._lane_next = (li + 1) % len(lanes)
                lane = lanes[li]
                # this device frame's previous read-back and previous writer (possibly another lane)
                for key in ("_fused_events", "_fused_writers"):
                    evs = getattr(self, key)
                    if evs[slot] is not None:
                        lane.wait_event(evs[slot])
                        evs[slot] = None
                if ev is not None:
                    ev[0].record(lane)
                ready = dev.march_rgb8(self.brick, cam, dtf, options.dt, options.ert, self.background,
                                       frame.view(-1), width, height, samples=samples, skip=options.skip_empty,
                                       lane=lane, slot=li + 1)
                self._fused_writers[slot] = ready
            if ev is not None:
                st = torch.cuda.current_stream(self.device) if not lanes else lane
                ev[1].record(st)
                ev[2].record(st)
                stats.events = tuple(ev)
            stats.record(options.frame_index, width * height, 0, (time.perf_counter() - t0) * 1e3)
            res = RenderResult(rgb8=frame, stats=stats, order=order, ready=ready)
            if options.collect_samples:
                res.samples = self.samples.view(height, width)
                stats._samples_dev = res.samples
            return res
        if options.composite == "cycle" and self.ep.R > 1 and not options.disable_compositing:
            return self._render_cycle(cam, width, height, options, dtf, stats, order, ev, t0)
        bands = None
        if options.clip_exchange and self.ep.R > 1 and not options.disable_compositing and \
                self.compositor.clips_bands():
            bands = self._bands(cam, width, height)
        push = None if options.disable_compositing or self.ep.R == 1 else self.compositor.push_targets()
        if push is not None:
            # fused march + exchange: peers write this frame into rank 0's frame buffer once every rank's
            # march is done, so the previous frame's read-back must drain before this march
            if self._pending_copy is not None:
                torch.cuda.current_stream(self.device).wait_event(self._pending_copy)
                self._pending_copy = None
            row_start, dst, flag_ptrs, counter, epoch = push
            dev.march_push(self.brick, cam, dtf, options.dt, options.ert, width, height, row_start, dst, flag_ptrs,
                           counter, epoch, samples=self.samples if options.collect_samples else None,
                           skip=options.skip_empty, band_clear=bands is not None,
                           half=self.compositor.fdt == torch.float16)
        else:
            dev.march(self.brick, cam, dtf, options.dt, options.ert, self.partial, width, height,
                      samples=self.samples if options.collect_samples else None, skip=options.skip_empty,
                      band_clear=bands is not None)
        if ev is not None:
            ev[1].record(torch.cuda.current_stream(self.device))
        if options.disable_compositing:
            order = [self.ep.rank] if self.ep.R == 1 else order
        if self._pending_copy is not None:
            # the previous frame's read-back may still be draining the device frame buffer
            torch.cuda.current_stream(self.device).wait_event(self._pending_copy)
            self._pending_copy = None
        out = self.compositor.composite(self.partial, order, self.background,
                                        keep_float=options.keep_float, solo=options.disable_compositing, bands=bands)
        if ev is not None:
            ev[2].record(torch.cuda.current_stream(self.device))
            stats.events = tuple(ev)
        nbytes = self.compositor.last_bytes
        stats.bytes_exchanged += nbytes
        stats.record(options.frame_index, width * height, nbytes, (time.perf_counter() - t0) * 1e3)
        res = RenderResult(rgb8=out.rgb8, stats=stats, order=order,
                           partial=None if push is not None else self.partial.view(height, width, 4))
        if options.keep_float and out.rgba is not None:
            rgba = out.rgba.view(height, width, 4).double().cpu().numpy()
            bg = np.asarray(self.background, np.float64)
            res.image = rgba[..., :3] + (1.0 - rgba[..., 3:4]) * bg
        if options.collect_samples:
            res.samples = self.samples.view(height, width)
            stats._samples_dev = res.samples
        return res

    def _render_cycle(self, cam, width, height, options, dtf, stats, order, ev, t0) -> RenderResult:
        """Ray cycling (the reference's paradigm, engine.py:282-310, for DVR).  Rank b's
        batch = its row block.  It starts at b's position p0 in the visibility order and hops along that
        order (ring_exchange, transport.py:457-462): at each hop the holder marches its brick into the
        batch's back state B (positions >= p0) or front state F (positions < p0), continuing the rays'
        accumulated state (ERT on accumulated opacity, so rays saturated in front skip later bricks).
        After R hops the batch is home (engine.py:305-309 asserts the same); F over B + background +
        tone map gives the RGB8 tile, gathered to rank 0 like the other modes."""
        ep, R, r, W = self.ep, self.ep.R, self.ep.rank, width
        blocks = assign_rows(height, R)
        pos = {s: i for i, s in enumerate(order)}
        nxt, prv = order[(pos[r] + 1) % R], order[(pos[r] - 1) % R]
        maxn = max(b1 - b0 for b0, b1 in blocks) * W
        comp = self.compositor
        bufs = [comp._buf("cycA", max(maxn, 1) * 8), comp._buf("cycB", max(maxn, 1) * 8)]
        mine = blocks[r]
        n_mine = (mine[1] - mine[0]) * W
        bufs[0][: n_mine * 8].zero_()
        cur = 0
        sent = 0
        for k in range(R):
            po = (pos[r] - k) % R  # origin position of the batch held at this hop
            rows = blocks[order[po]]
            n = (rows[1] - rows[0]) * W
            if n:
                state = bufs[cur][: n * 8]
                seg = state[: n * 4] if pos[r] >= po else state[n * 4:]  # back (B) or front (F) segment
                smp = self.samples[rows[0] * W: rows[1] * W] if options.collect_samples else None
                dev.march(self.brick, cam, dtf, options.dt, options.ert, seg, width, height, samples=smp,
                          skip=options.skip_empty, accum=True, rows=rows)
            # hand the batch on along the visibility order; receive the one behind it
            rrows = blocks[order[(pos[r] - k - 1) % R]]
            rn = (rrows[1] - rrows[0]) * W
            ep.exchange([(nxt, bufs[cur][: n * 8])] if n else [], [(prv, bufs[1 - cur][: rn * 8])] if rn else [])
            sent += n * 32
            stats.record(options.frame_index, n, n * 32, (time.perf_counter() - t0) * 1e3)
            cur = 1 - cur
        if ev is not None:
            ev[1].record(torch.cuda.current_stream(self.device))
        tile = comp._buf("tile8", max(n_mine, 1) * 3, torch.uint8)[: n_mine * 3]
        tile_f = comp._buf("tilef", max(n_mine, 1) * 4)[: n_mine * 4] if options.keep_float else None
        if n_mine:
            home = bufs[cur][: n_mine * 8]
            dev.composite([home[n_mine * 4:], home[: n_mine * 4]], self.background, rgb8=tile, rgba=tile_f)
        if self._pending_copy is not None:
            torch.cuda.current_stream(self.device).wait_event(self._pending_copy)
            self._pending_copy = None
        comp.last_bytes = 0
        out = comp._gather_tiles(mine, tile, tile_f, blocks, options.keep_float)
        if ev is not None:
            ev[2].record(torch.cuda.current_stream(self.device))
            stats.events = tuple(ev)
        stats.bytes_exchanged += sent + comp.last_bytes
        res = RenderResult(rgb8=out.rgb8, stats=stats, order=order)
        if options.keep_float and out.rgba is not None:
            rgba = out.rgba.view(height, width, 4).double().cpu().numpy()
            res.image = rgba[..., :3] + (1.0 - rgba[..., 3:4]) * np.asarray(self.background, np.float64)
        if options.collect_samples:
            res.samples = self.samples.view(height, width)
            stats._samples_dev = res.samples
        return res

    def _frame_lanes(self, options: RenderOptions) -> list:
        """Lane streams for frames in flight (single rank, fused frame, no sample counts); [] = ordered on
        the current stream as usual."""
        n = int(options.frames_in_flight)
        if n < 1 or n >= dev.MARCH_COUNTER_SLOTS:
            raise UsageError(f"frames_in_flight must be in [1, {dev.MARCH_COUNTER_SLOTS - 1}], got {n}")
        if n == 1 or options.collect_samples:
            if self._lanes:
                self.join()
                self._lanes = []
            return []
        if len(self._lanes) != n:
            self.join()
            self._lanes = [torch.cuda.Stream(self.device) for _ in range(n)]
            self._lane_next = 0
        return self._lanes

    def join(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Order ``stream`` (default: current) after every frame still in flight on a lane stream."""
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        for i, w in enumerate(self._fused_writers):
            if w is not None:
                st.wait_event(w)
        self.brick.join_lanes(st)

    def render_to_host(self, cam: CameraSpec, width: int, height: int, host: Optional[torch.Tensor],
                       options: RenderOptions = RenderOptions(), verify: bool = True) -> "HostFrame":
        """Collective render whose RGB8 frame is copied into ``host`` (pinned, (H, W, 3) uint8, rank 0) on a
        side stream: the read-back of frame k overlaps the march of frame k+1.  ``HostFrame.wait()``
        blocks until the bytes are in host memory."""
        res = self.render(cam, width, height, options, verify)
        if res.rgb8 is None:
            return HostFrame(None, None, res)
        if host is None or tuple(host.shape) != (height, width, 3) or host.dtype != torch.uint8:
            raise UsageError("host frame must be a (H, W, 3) uint8 tensor")
        main = torch.cuda.current_stream(self.device)
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(self.device)
        if res.ready is not None:  # frames in flight: the frame's own lane event, not the current stream
            ready = res.ready
        else:
            ready = torch.cuda.Event()
            ready.record(main)
        self._copy_stream.wait_event(ready)
        # one rank: every pixel outside the brick's footprint rectangle is the tone-mapped background, written
        # by the march itself.  A host buffer that received a full frame of this size and background holds the
        # background everywhere outside the rectangles written since (FrameResult.array is read-only), so only
        # the bounding box of those and this frame's rectangle crosses PCIe
        region = None
        key = (width, height, tuple(self.background))
        ent = self._host_keys.get(host.data_ptr())
        fused = self.ep.R == 1 and res.partial is None
        rect = dev.desc_footprint(self.brick.desc, cam, width, height) if fused else None
        if fused and ent is not None and ent[0] is host and ent[1] == key:
            d = ent[2]
            region = (min(d[0], rect[0]), min(d[1], rect[1]), max(d[2], rect[2]), max(d[3], rect[3]))
        with torch.cuda.stream(self._copy_stream):
            if region is not None:
                x0, y0, x1, y1 = region
                if x1 > x0 and y1 > y0:
                    dev.copy_2d(self.device.index, host.data_ptr() + 3 * (y0 * width + x0), 3 * width,
                                res.rgb8.data_ptr() + 3 * (y0 * width + x0), 3 * width, 3 * (x1 - x0), y1 - y0,
                                stream=self._copy_stream.cuda_stream)
                    self.d2h_bytes += 3 * (x1 - x0) * (y1 - y0)
                # the rendered rectangle alone keeps non-background bytes: the next copy covers it
                ent[2] = rect
            else:
                host.copy_(res.rgb8, non_blocking=True)
                self.d2h_bytes += host.numel()
                if fused:
                    if len(self._host_keys) >= 8:  # a bounded set of recently used host buffers
                        self._host_keys.pop(next(iter(self._host_keys)))
                    self._host_keys[host.data_ptr()] = [host, key, tuple(rect)]
        done = torch.cuda.Event()
        done.record(self._copy_stream)
        if self._fused_frames is not None and res.rgb8 is self._fused_frames[self._fused_slot]:
            self._fused_events[self._fused_slot] = done  # guards only that device frame
        else:
            self._pending_copy = done
        return HostFrame(host, done, res)


@dataclass
class HostFrame:
    """A frame on its way to host memory (VolumeRenderer.render_to_host)."""

    pixels: Optional[torch.Tensor]
    event: Optional[torch.cuda.Event]
    result: RenderResult

    def wait(self) -> Optional[torch.Tensor]:
        if self.event is not None:
            self.event.synchronize()
        return self.pixels


def render_volume_with(ep: RankEndpoint, brick: dev.DeviceBrick, decomposition: Decomposition,
                       tf: TransferFunction1D, cam: CameraSpec, width: int, height: int,
                       options: RenderOptions = RenderOptions(), background: Vec3 = (0.0, 0.0, 0.0)) -> RenderResult:
    """Collective render given this rank's resident brick (the render_with slot, engine.py:459-488)."""
    return VolumeRenderer(ep, brick, decomposition, tf, background).render(cam, width, height, options)


def render_volume_frame(ep: RankEndpoint, decomposition: Decomposition, tf: TransferFunction1D,
                        cam: CameraSpec, width: int, height: int, options: RenderOptions = RenderOptions(),
                        background: Vec3 = (0.0, 0.0, 0.0), ghost: int = 1) -> RenderResult:
    """Collective render of a decomposed synthetic field (the render_frame slot, engine.py:491-497):
    each rank generates its own brick on its GPU, then renders."""
    device = ep.device if ep.device.type == "cuda" else torch.device("cuda", torch.cuda.current_device())
    brick = dev.DeviceBrick(decomposition.brick(ep.rank, ghost), device).generate(decomposition.field)
    try:
        return render_volume_with(ep, brick, decomposition, tf, cam, width, height, options, background)
    finally:
        torch.cuda.current_stream(device).synchronize()
        brick.close()
