"""Torch-facing wrappers of the C ABI: device bricks, the marcher and the compositor kernel.

PyTorch is plumbing here: it owns the device buffers (partials, TF table, frames) and supplies the
current stream; all compute is in libdprt_cuda.so.  Every call checks its status code and raises the
reference's exception classes (errors.py); there is no CPU path.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from .errors import UsageError
from .geom import CameraSpec
from .volume import BrickDesc, FieldSpec, TransferFunction1D


MARCH_COUNTER_SLOTS = _lib.MARCH_COUNTER_SLOTS  # tile queues per brick: slot 0 stream-ordered, 1.. frame lanes


def _stream(device: torch.device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _require_cuda(t: torch.Tensor, name: str, dtype: torch.dtype) -> None:
    if not t.is_cuda:
        raise UsageError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise UsageError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise UsageError(f"{name} must be contiguous")


def desc_struct(desc: BrickDesc) -> _lib.BrickDesc:
    d = _lib.BrickDesc()
    d.dims[:] = list(desc.dims)
    d.lo[:] = list(desc.lo)
    d.hi[:] = list(desc.hi)
    d.ghost = desc.ghost
    d.origin[:] = [float(v) for v in desc.origin]
    d.spacing[:] = [float(v) for v in desc.spacing]
    return d


def desc_footprint(desc: BrickDesc, cam: CameraSpec, width: int, height: int) -> Tuple[int, int, int, int]:
    """Screen rectangle [x0, y0, x1, y1) of a brick's owned box (host-only: any rank, any brick)."""
    rect = (ctypes.c_int32 * 4)()
    c = camera_struct(cam)
    d = desc_struct(desc)
    _lib.check(_lib.lib().dprt_desc_footprint(ctypes.byref(d), ctypes.byref(c), width, height, rect),
               "dprt_desc_footprint")
    return tuple(rect)


def camera_struct(cam: CameraSpec) -> _lib.Camera:
    """Host-evaluated basis and film half extents (geom.py:163-168, 250-251)."""
    f, r, u = cam.basis()
    half_w, half_h = cam.film_half_extents()
    c = _lib.Camera()
    c.pos[:] = [float(v) for v in cam.position]
    c.fwd[:] = list(f)
    c.right[:] = list(r)
    c.up[:] = list(u)
    c.half_w = half_w
    c.half_h = half_h
    return c


class DeviceBrick:
    """A rank's brick resident in HBM (stored voxels incl. ghost + macrocell min/max grid).

    Lifetime mirrors the reference's RefCounted objects (refcount.py:10-63): ``close()`` releases the
    native handle; using a closed brick raises UsageError."""

    def __init__(self, desc: BrickDesc, device: torch.device, half_quads: bool = False):
        """``half_quads`` (opt-in): the coefficient quads in fp16, half the quad bytes for memory-bound bricks
        at a stated precision cost."""
        if device.type != "cuda":
            raise UsageError("DeviceBrick needs a CUDA device")
        self.desc = desc
        self.device = device
        self.half_quads = bool(half_quads)
        self.index = device.index if device.index is not None else torch.cuda.current_device()
        d = desc_struct(desc)
        if half_quads:
            d.flags |= _lib.BRICK_HALF_QUADS
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().dprt_brick_create(self.index, ctypes.byref(d), ctypes.byref(h)), "dprt_brick_create")
        self._h = h
        # frames in flight (march_rgb8 with a lane stream): the last march event per lane stream, the TF
        # version of the last lane march and whether that march rebuilt the TF-dependent skip distances
        self._lane_reads = {}
        self._lane_version = None
        self._lane_rebuilt = False

    def join_lanes(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Make ``stream`` (default: the current stream) wait for every march still in flight on a lane
        stream.  Called before anything stream-ordered touches what those marches read: the voxels, the
        skip distances, the tile counters."""
        if not self._lane_reads:
            return
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        for ev in self._lane_reads.values():
            st.wait_event(ev)
        self._lane_reads.clear()

    @property
    def handle(self) -> ctypes.c_void_p:
        if self._h is None:
            raise UsageError("brick was released")
        return self._h

    def generate(self, f: FieldSpec) -> "DeviceBrick":
        if tuple(f.dims) != tuple(self.desc.dims):
            raise UsageError(f"field dims {f.dims} != brick grid {self.desc.dims}")
        if f.kind == "marschnerLobb":
            blobs = np.ascontiguousarray(f.ml, np.float64)  # {f_M, alpha}
            spec = _lib.FieldSpec(1, 1, ctypes.c_void_p(blobs.ctypes.data))
        else:
            blobs = np.ascontiguousarray(f.blobs, np.float64)
            spec = _lib.FieldSpec(0, blobs.shape[0], ctypes.c_void_p(blobs.ctypes.data))
        self.join_lanes()
        _lib.check(_lib.lib().dprt_brick_generate(self.handle, ctypes.byref(spec), _stream(self.device)),
                   "dprt_brick_generate")
        return self

    def upload(self, voxels) -> "DeviceBrick":
        """Stored voxels (z, y, x) from a host numpy array or a device tensor."""
        shape = tuple(reversed(self.desc.stored_dims))
        self.join_lanes()
        if isinstance(voxels, torch.Tensor):
            if tuple(voxels.shape) != shape:
                raise UsageError(f"voxel tensor {tuple(voxels.shape)} != stored {shape}")
            if voxels.is_cuda:
                _require_cuda(voxels, "voxels", torch.float32)
                rc = _lib.lib().dprt_brick_upload(self.handle, ctypes.c_void_p(voxels.data_ptr()), 1, _stream(self.device))
                _lib.check(rc, "dprt_brick_upload")
                return self
            voxels = voxels.numpy()
        arr = np.ascontiguousarray(voxels, np.float32)
        if arr.shape != shape:
            raise UsageError(f"voxel array {arr.shape} != stored {shape}")
        rc = _lib.lib().dprt_brick_upload(self.handle, ctypes.c_void_p(arr.ctypes.data), 0, _stream(self.device))
        _lib.check(rc, "dprt_brick_upload")
        torch.cuda.current_stream(self.device).synchronize()  # host array must outlive the copy
        return self

    def download_device(self) -> torch.Tensor:
        """Stored voxels (z, y, x) as a new f32 tensor on the brick's device (stream-ordered copy)."""
        out = torch.empty(tuple(reversed(self.desc.stored_dims)), dtype=torch.float32, device=self.device)
        rc = _lib.lib().dprt_brick_download(self.handle, ctypes.c_void_p(out.data_ptr()), 1, _stream(self.device))
        _lib.check(rc, "dprt_brick_download")
        return out

    def download(self) -> np.ndarray:
        out = np.empty(tuple(reversed(self.desc.stored_dims)), np.float32)
        rc = _lib.lib().dprt_brick_download(self.handle, ctypes.c_void_p(out.ctypes.data), 0, _stream(self.device))
        _lib.check(rc, "dprt_brick_download")
        return out

    @property
    def macro_shift(self) -> int:
        """log2 of the macrocell edge in cells (2 or 3, by brick size; dprt_brick_macro_shift)."""
        v = ctypes.c_int32()
        _lib.check(_lib.lib().dprt_brick_macro_shift(self.handle, ctypes.byref(v)), "dprt_brick_macro_shift")
        return int(v.value)

    def footprint(self, cam: CameraSpec, width: int, height: int):
        rect = (ctypes.c_int32 * 4)()
        c = camera_struct(cam)
        _lib.check(_lib.lib().dprt_brick_footprint(self.handle, ctypes.byref(c), width, height, rect),
                   "dprt_brick_footprint")
        return tuple(rect)

    def close(self) -> None:
        if self._h is not None:
            _lib.check(_lib.lib().dprt_brick_destroy(self._h), "dprt_brick_destroy")
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def field_mass_function(f: FieldSpec, device: torch.device, tau: float, chunk: int = 64):
    """The mass function of the mass-weighted kd split (volume.decompose) for a synthetic field, computed
    on the GPU: the field is generated in z-chunks of ``chunk`` cell planes (bit-identical to the whole
    field), thresholded at ``tau`` into a 1-byte mask kept on the device, and
    ``mass(axis, lo, hi)`` sums the voxel box [lo, hi) of the mask over the two other axes -- the same
    counts as api._mass_function's host path, without moving the field to the host."""
    from .volume import BrickDesc

    nx, ny, nz = f.dims
    mask = torch.empty((nz, ny, nx), dtype=torch.uint8, device=device)
    z = 0
    while z < nz - 1:
        z1 = min(z + chunk, nz - 1)
        b = DeviceBrick(BrickDesc(f.dims, (0, 0, z), (nx - 1, ny - 1, z1), 0, f.origin, f.spacing), device)
        try:
            vox = b.generate(f).download_device()  # voxel planes z .. z1
        finally:
            torch.cuda.current_stream(device).synchronize()
            b.close()
        last = z1 == nz - 1
        mask[z: z1 + 1 if last else z1] = (vox if last else vox[:-1]) >= tau
        del vox
        z = z1

    def mass(axis, lo, hi):
        sub = mask[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        dims = tuple(a for a in range(3) if a != 2 - axis)
        return sub.sum(dim=dims, dtype=torch.int64).cpu().numpy()

    return mass


def skip_key(tf: TransferFunction1D) -> int:
    """The bricks' TF-dependent skip distances depend on the TF only through which entries have alpha > 0,
    the entry count and the value range (skip_classify_kernel): a nonzero 63-bit digest of exactly those,
    used as the ABI's tf_version -- editing colours or scaling opacities keeps the distances, changing the
    alpha support rebuilds them."""
    import hashlib

    a = np.ascontiguousarray(tf.as_f32().reshape(-1, 4)[:, 3] > 0.0)
    h = hashlib.blake2b(digest_size=8)
    h.update(np.array([tf.n], np.int64).tobytes())
    h.update(np.array([tf.vmin, tf.vmax], np.float64).tobytes())
    h.update(np.packbits(a).tobytes())
    return (int.from_bytes(h.digest(), "little") & ((1 << 63) - 1)) | 1


class DeviceTF:
    """A transfer function table resident on one device (4 KiB for 256 entries).

    ``version`` tags what the bricks' cached skip distances depend on (``skip_key``: the alpha support and
    the value range); ``update`` re-uploads the table and recomputes the tag when the contents change.  Uploads from a pinned staging buffer alternate between
    two device tables and run on a side stream (``dprt_stage_input``, SM-driven): frame k's table is
    staged while frame k-1 still marches out of the other one, and the march of frame k waits on it."""

    def __init__(self, tf: TransferFunction1D, device: torch.device):
        self.tf = tf
        self._host = tf.as_f32().reshape(-1).copy()
        self.table = torch.from_numpy(self._host.copy()).to(device)
        self.version = skip_key(tf)
        self._tables = None        # the two staging targets (allocated on the first staged update)
        self._slot = 0
        self._side = None          # side stream for the staging copies
        self._marker = None        # main-stream event recorded at the previous staged update
        self._lane_reads = {}      # id(table) -> events of lane-stream marches that read it (frames in flight)

    def note_lane_read(self, lane: torch.cuda.Stream, event: torch.cuda.Event) -> None:
        """A march on ``lane`` (not the current stream) reads the current table until ``event`` (lanes run
        their marches in order, so the latest event per lane covers the earlier ones)."""
        self._lane_reads.setdefault(id(self.table), {})[lane.cuda_stream] = event

    def _wait_lane_reads(self, stream: torch.cuda.Stream, table: torch.Tensor) -> None:
        for ev in self._lane_reads.pop(id(table), {}).values():
            stream.wait_event(ev)

    def update(self, tf: TransferFunction1D, staging: Optional[torch.Tensor] = None) -> None:
        """New table contents (optionally copied from a pinned host staging tensor)."""
        host = tf.as_f32().reshape(-1)
        if host.shape != self._host.shape or not np.array_equal(host, self._host) or (
                tf.vmin, tf.vmax) != (self.tf.vmin, self.tf.vmax):
            self.version = skip_key(tf)
            self._host = host.copy()
            if host.shape[0] != self.table.numel():
                # lane marches may still read the old table: the current stream (its allocator's reuse
                # order) waits for them before the tensor is released
                for t in self._tables or [self.table]:
                    self._wait_lane_reads(torch.cuda.current_stream(t.device), t)
                self.table = torch.empty(host.shape[0], dtype=torch.float32, device=self.table.device)
                self._tables = None
        self.tf = tf
        if staging is not None and staging.is_pinned() and staging.numel() == host.shape[0] and \
                staging.dtype == torch.float32:
            self._stage(staging)
            return
        src = staging if staging is not None else torch.from_numpy(self._host)
        self._wait_lane_reads(torch.cuda.current_stream(self.table.device), self.table)
        self.table.copy_(src, non_blocking=staging is not None)

    def _stage(self, staging: torch.Tensor) -> None:
        d = self.table.device
        main = torch.cuda.current_stream(d)
        if self._tables is None:
            self._tables = [self.table, torch.empty_like(self.table)]
            self._side = torch.cuda.Stream(d)
            self._marker = None
        self._slot ^= 1
        dst = self._tables[self._slot]
        # the slot was last read by the march enqueued before the previous staged update: wait for
        # exactly that work (the marker), not for the march still running out of the other slot
        if self._marker is not None:
            self._side.wait_event(self._marker)
        self._wait_lane_reads(self._side, dst)  # ... and for lane-stream marches out of that slot
        self._marker = torch.cuda.Event()
        self._marker.record(main)
        _lib.check(_lib.lib().dprt_stage_input(d.index, ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(staging.data_ptr()),
                                               dst.numel() * 4, ctypes.c_void_p(self._side.cuda_stream)),
                   "dprt_stage_input")
        ready = torch.cuda.Event()
        ready.record(self._side)
        main.wait_event(ready)
        self.table = dst

    def params(self, dt: float, ert: float, flags: int = 0) -> _lib.MarchParams:
        return _lib.MarchParams(ctypes.c_void_p(self.table.data_ptr()), self.tf.n, flags, float(self.tf.vmin),
                                float(self.tf.vmax), float(dt), float(ert), self.version)


def march(brick: DeviceBrick, cam: CameraSpec, tf: DeviceTF, dt: float, ert: float, partial: torch.Tensor,
          width: int, height: int, samples: Optional[torch.Tensor] = None, skip: bool = True,
          footprint: bool = True, band_clear: bool = False, accum: bool = False,
          rows: Optional[Tuple[int, int]] = None, force_wide: bool = False, force_deep: bool = False) -> None:
    """dprt_march: the brick's full-frame premultiplied RGBA partial into ``partial`` (H*W*4 f32).
    ``band_clear``: only the footprint's row band is defined afterwards (band-clipped compositing).
    ``rows`` = (r0, r1): march only those pixel rows; ``partial`` (and ``samples``) hold just them.
    ``accum``: ``partial`` holds each ray's accumulated front-to-back state, which the march continues
    (ray cycling).  A float16 ``partial`` gets fp16 fragments (DPRT_MARCH_HALF)."""
    half = partial.dtype == torch.float16
    _require_cuda(partial, "partial", torch.float16 if half else torch.float32)
    npix = width * height if rows is None else (rows[1] - rows[0]) * width
    if rows is not None and not (0 <= rows[0] < rows[1] <= height):
        raise UsageError(f"row window {rows} outside [0, {height})")
    if partial.numel() != npix * 4:
        raise UsageError(f"partial holds {partial.numel()} floats, need {npix * 4}")
    sp = ctypes.c_void_p(0)
    if samples is not None:
        _require_cuda(samples, "samples", torch.int32)
        if samples.numel() != npix:
            raise UsageError("samples buffer must hold one count per pixel")
        sp = ctypes.c_void_p(samples.data_ptr())
    flags = (0 if skip else _lib.MARCH_NO_SKIP) | (0 if footprint else _lib.MARCH_FULL_FRAME)
    if band_clear:
        flags |= _lib.MARCH_BAND_CLEAR
    if accum:
        flags |= _lib.MARCH_ACCUM
    if half:
        flags |= _lib.MARCH_HALF
    if force_wide:  # test hook: the addressing of bricks with >= 2^31 quads
        flags |= _lib.MARCH_WIDE
    if force_deep:  # test hook: the large-brick batch / occupancy configuration
        flags |= _lib.MARCH_DEEP
    variant = os.environ.get("DPRT_MARCHER", "")
    if variant == "beam":
        flags |= _lib.MARCH_BEAM
    elif variant == "queue":
        flags |= _lib.MARCH_QUEUE
    p = tf.params(dt, ert, flags)
    if rows is not None:
        p.row0, p.row1 = int(rows[0]), int(rows[1])
    brick.join_lanes()  # counter slot 0, skip distances: ordered after frames still in flight
    c = camera_struct(cam)
    rc = _lib.lib().dprt_march(brick.handle, ctypes.byref(c), ctypes.byref(p), ctypes.c_void_p(partial.data_ptr()),
                               sp, width, height, _stream(brick.device))
    _lib.check(rc, "dprt_march")


def march_push(brick: DeviceBrick, cam: CameraSpec, tf: DeviceTF, dt: float, ert: float, width: int, height: int,
               row_start: Sequence[int], dst: Sequence[int], flag_ptrs: Sequence[int], counter_ptr: int, epoch: int,
               samples: Optional[torch.Tensor] = None, skip: bool = True, band_clear: bool = False,
               half: bool = False) -> None:
    """dprt_march_push: the fused march + exchange (DESIGN.md §6 "p2p_push").  Row block b of this brick's
    RGBA partial is written straight into ``dst[b]`` (block b's owner's inbox slot for this rank; a peer
    pointer), pixel (x, y) at element (y - row_start[b]) * W + x, and once every CTA's stores are fenced
    ``epoch`` is release-stored into every ``flag_ptrs[b]``.  ``counter_ptr``: a zeroed device word."""
    P = len(dst)
    if len(row_start) != P + 1 or len(flag_ptrs) != P:
        raise UsageError("push targets need P destinations, P flags and P + 1 row boundaries")
    sp = ctypes.c_void_p(0)
    if samples is not None:
        _require_cuda(samples, "samples", torch.int32)
        if samples.numel() != width * height:
            raise UsageError("samples buffer must hold one count per pixel")
        sp = ctypes.c_void_p(samples.data_ptr())
    flags = (0 if skip else _lib.MARCH_NO_SKIP) | (_lib.MARCH_BAND_CLEAR if band_clear else 0) | \
        (_lib.MARCH_HALF if half else 0)
    p = tf.params(dt, ert, flags)
    rows = (ctypes.c_int32 * (P + 1))(*[int(r) for r in row_start])
    dsts = (ctypes.c_void_p * P)(*[int(d) for d in dst])
    fls = (ctypes.c_void_p * P)(*[int(f) for f in flag_ptrs])
    t = _lib.PushTargets(P, 0, ctypes.cast(rows, ctypes.c_void_p), ctypes.cast(dsts, ctypes.c_void_p),
                         ctypes.cast(fls, ctypes.c_void_p), ctypes.c_void_p(counter_ptr), int(epoch) & 0xFFFFFFFF, 0)
    brick.join_lanes()
    c = camera_struct(cam)
    rc = _lib.lib().dprt_march_push(brick.handle, ctypes.byref(c), ctypes.byref(p), ctypes.byref(t), sp, width, height,
                                    _stream(brick.device))
    _lib.check(rc, "dprt_march_push")


def wait_flags(device_index: int, flags_ptr: int, n: int, epoch: int, stream: Optional[int] = None) -> None:
    """dprt_wait_flags: later work on the stream runs once the n device words at ``flags_ptr`` reach ``epoch``
    (written by other GPUs, or by work already complete -- never by work that itself waits on this stream)."""
    s = ctypes.c_void_p(stream if stream is not None else torch.cuda.current_stream(device_index).cuda_stream)
    _lib.check(_lib.lib().dprt_wait_flags(device_index, ctypes.c_void_p(flags_ptr), n, int(epoch) & 0xFFFFFFFF, s),
               "dprt_wait_flags")


def march_stats(brick: DeviceBrick, cam: CameraSpec, tf: DeviceTF, dt: float, ert: float, width: int, height: int,
                skip: bool = True) -> dict:
    """dprt_march_stats (synchronous diagnostic): what the production march reads and shades for this view --
    ``needed_voxels`` = cells of the macrocells holding a shaded sample (x 4 B: the brick bytes a perfect
    marcher must read once), ``shaded`` / ``contributing`` samples and the number of such macrocells."""
    p = tf.params(dt, ert, 0 if skip else _lib.MARCH_NO_SKIP)
    c = camera_struct(cam)
    out = (ctypes.c_uint64 * 4)()
    brick.join_lanes()
    _lib.check(_lib.lib().dprt_march_stats(brick.handle, ctypes.byref(c), ctypes.byref(p), width, height, out,
                                           _stream(brick.device)), "dprt_march_stats")
    return {"needed_voxels": int(out[0]), "needed_bytes": 4 * int(out[0]), "shaded_samples": int(out[1]),
            "contributing_samples": int(out[2]), "macrocells": int(out[3])}


def march_rgb8(brick: DeviceBrick, cam: CameraSpec, tf: DeviceTF, dt: float, ert: float, background,
               rgb8: torch.Tensor, width: int, height: int, samples: Optional[torch.Tensor] = None,
               skip: bool = True, lane: Optional[torch.cuda.Stream] = None,
               slot: int = 0) -> Optional[torch.cuda.Event]:
    """dprt_march_rgb8: single-rank frame, over-background and tone map fused into the march.

    ``lane`` (frames in flight): run the march on that stream with tile-counter ``slot`` (1..3, one per
    lane) instead of the current stream.  The lane first waits for the current stream's work so far (the
    frame's inputs are ordered as usual); the current stream does NOT wait for the march -- the returned
    event marks the frame complete.  Frames on different lanes overlap: the next frame's CTAs take the
    SMs the previous frame's last beams leave idle.  Hazards between lanes are resolved here: a march that
    (re)builds the TF-dependent skip distances, or follows one that did, first waits for the other lanes,
    and every stream-ordered march / brick write joins the lanes (``DeviceBrick.join_lanes``)."""
    _require_cuda(rgb8, "rgb8", torch.uint8)
    if rgb8.numel() != width * height * 3:
        raise UsageError("rgb8 frame must hold 3 bytes per pixel")
    sp = ctypes.c_void_p(0)
    if samples is not None:
        _require_cuda(samples, "samples", torch.int32)
        sp = ctypes.c_void_p(samples.data_ptr())
    p = tf.params(dt, ert, 0 if skip else _lib.MARCH_NO_SKIP)
    c = camera_struct(cam)
    bg = (ctypes.c_float * 3)(*[float(v) for v in background])
    if lane is None:
        if slot != 0:
            raise UsageError("counter slots other than 0 need a lane stream")
        brick.join_lanes()
        rc = _lib.lib().dprt_march_rgb8(brick.handle, ctypes.byref(c), ctypes.byref(p), bg,
                                        ctypes.c_void_p(rgb8.data_ptr()), sp, width, height, _stream(brick.device))
        _lib.check(rc, "dprt_march_rgb8")
        return None
    if not 1 <= slot < _lib.MARCH_COUNTER_SLOTS:
        raise UsageError(f"lane counter slot must be in [1, {_lib.MARCH_COUNTER_SLOTS}), got {slot}")
    main = torch.cuda.current_stream(brick.device)
    ready = torch.cuda.Event()
    ready.record(main)
    lane.wait_event(ready)
    rebuild = brick._lane_version != tf.version
    if rebuild or brick._lane_rebuilt:
        for key, ev in list(brick._lane_reads.items()):
            if key != lane.cuda_stream:
                lane.wait_event(ev)
    p.counter_slot = slot
    rc = _lib.lib().dprt_march_rgb8(brick.handle, ctypes.byref(c), ctypes.byref(p), bg,
                                    ctypes.c_void_p(rgb8.data_ptr()), sp, width, height,
                                    ctypes.c_void_p(lane.cuda_stream))
    _lib.check(rc, "dprt_march_rgb8")
    done = torch.cuda.Event()
    done.record(lane)
    brick._lane_reads[lane.cuda_stream] = done
    brick._lane_rebuilt = rebuild
    brick._lane_version = tf.version
    tf.note_lane_read(lane, done)
    return done


def composite(frags: Sequence[torch.Tensor], background=None, rgb8: Optional[torch.Tensor] = None,
              rgba: Optional[torch.Tensor] = None, ranges: Optional[Sequence[Tuple[int, int]]] = None,
              npix: Optional[int] = None) -> None:
    """dprt_composite: front-to-back 'over' of RGBA fragments (already in visibility order); writes
    tone-mapped RGB8 (needs ``background``) and/or the blended RGBA.  Without ``ranges`` the fragments
    are equally sized and cover the whole tile; with ``ranges`` fragment i holds only the tile pixels
    [lo_i, hi_i) (clear elsewhere) and ``npix`` is the tile size (dprt_composite_ranged)."""
    if not frags:
        raise UsageError("nothing to composite")
    fdt = frags[0].dtype if frags[0].dtype in (torch.float16, torch.float32) else torch.float32
    if ranges is None:
        n = frags[0].numel()
        if n % 4:
            raise UsageError("fragments must hold whole RGBA pixels")
        for i, f in enumerate(frags):
            _require_cuda(f, f"fragment {i}", fdt)
            if f.numel() != n:
                raise UsageError("fragments differ in size")
        npix = n // 4
    else:
        if npix is None or len(ranges) != len(frags):
            raise UsageError("ranged composite needs npix and one (lo, hi) range per fragment")
        for i, (f, (lo, hi)) in enumerate(zip(frags, ranges)):
            _require_cuda(f, f"fragment {i}", fdt)
            if f.numel() < 4 * (hi - lo):
                raise UsageError(f"fragment {i} holds {f.numel() // 4} pixels, range needs {hi - lo}")
        n = npix * 4
    flags = 0
    bg_arr = None
    rgb_ptr = ctypes.c_void_p(0)
    rgba_ptr = ctypes.c_void_p(0)
    if rgb8 is not None:
        _require_cuda(rgb8, "rgb8", torch.uint8)
        if rgb8.numel() != npix * 3:
            raise UsageError("rgb8 output must hold 3 bytes per pixel")
        if background is None:
            raise UsageError("tone mapping needs a background colour")
        flags |= _lib.COMPOSITE_TONEMAP
        rgb_ptr = ctypes.c_void_p(rgb8.data_ptr())
    if background is not None:
        bg_arr = (ctypes.c_float * 3)(*[float(c) for c in background])
    if rgba is not None:
        _require_cuda(rgba, "rgba", torch.float32)
        if rgba.numel() != n:
            raise UsageError("rgba output must match the fragments")
        flags |= _lib.COMPOSITE_RGBA
        rgba_ptr = ctypes.c_void_p(rgba.data_ptr())
    if fdt == torch.float16:
        flags |= _lib.COMPOSITE_HALF_IN
    ptrs = (ctypes.c_void_p * len(frags))(*[f.data_ptr() for f in frags])
    rng = None if ranges is None else (ctypes.c_int64 * (2 * len(ranges)))(*[int(v) for r in ranges for v in r])
    dev = frags[0].device
    rc = _lib.lib().dprt_composite_ranged(dev.index if dev.index is not None else torch.cuda.current_device(), ptrs,
                                          rng, len(frags), npix, bg_arr, flags, rgb_ptr, rgba_ptr, _stream(dev))
    _lib.check(rc, "dprt_composite")


def composite_ptrs(device_index: int, ptrs: Sequence[int], npix: int, background, rgb8_ptr: int = 0,
                   rgba_ptr: int = 0, stream: Optional[int] = None,
                   ranges: Optional[Sequence[Tuple[int, int]]] = None, half: bool = False) -> None:
    """Raw-pointer form for peer (IPC-mapped) fragments and outputs: the fused NVLink compositor."""
    flags = (_lib.COMPOSITE_TONEMAP if rgb8_ptr else 0) | (_lib.COMPOSITE_RGBA if rgba_ptr else 0)
    if half:
        flags |= _lib.COMPOSITE_HALF_IN
    bg_arr = (ctypes.c_float * 3)(*[float(c) for c in background]) if background is not None else None
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    rng = None if ranges is None else (ctypes.c_int64 * (2 * len(ranges)))(*[int(v) for r in ranges for v in r])
    s = ctypes.c_void_p(stream if stream is not None else torch.cuda.current_stream(device_index).cuda_stream)
    rc = _lib.lib().dprt_composite_ranged(device_index, arr, rng, len(ptrs), npix, bg_arr, flags,
                                          ctypes.c_void_p(rgb8_ptr), ctypes.c_void_p(rgba_ptr), s)
    _lib.check(rc, "dprt_composite")


def composite_signal(device_index: int, ptrs: Sequence[int], npix: int, background, rgb8_ptr: int, rgba_ptr: int,
                     ranges: Optional[Sequence[Tuple[int, int]]], counter_ptr: int, signal_ptrs: Sequence[int],
                     epoch: int, half: bool = False, stream: Optional[int] = None) -> None:
    """dprt_composite_signal: composite_ptrs whose last CTA, after every CTA fenced its stores (RGB8 rows in
    rank 0's frame over NVLink), release-stores ``epoch`` into every ``signal_ptrs`` word."""
    flags = (_lib.COMPOSITE_TONEMAP if rgb8_ptr else 0) | (_lib.COMPOSITE_RGBA if rgba_ptr else 0)
    if half:
        flags |= _lib.COMPOSITE_HALF_IN
    bg_arr = (ctypes.c_float * 3)(*[float(c) for c in background]) if background is not None else None
    arr = (ctypes.c_void_p * max(len(ptrs), 1))(*ptrs)
    rng = None if ranges is None else (ctypes.c_int64 * (2 * len(ranges)))(*[int(v) for r in ranges for v in r])
    sig = (ctypes.c_void_p * len(signal_ptrs))(*signal_ptrs)
    s = ctypes.c_void_p(stream if stream is not None else torch.cuda.current_stream(device_index).cuda_stream)
    rc = _lib.lib().dprt_composite_signal(device_index, arr, rng, len(ptrs), npix, bg_arr, flags,
                                          ctypes.c_void_p(rgb8_ptr), ctypes.c_void_p(rgba_ptr),
                                          ctypes.c_void_p(counter_ptr), sig, len(signal_ptrs),
                                          int(epoch) & 0xFFFFFFFF, s)
    _lib.check(rc, "dprt_composite_signal")


def copy_2d(device_index: int, dst: int, dst_pitch: int, src: int, src_pitch: int, width_bytes: int, rows: int,
            stream: Optional[int] = None) -> None:
    """dprt_copy_2d: ``rows`` rows of ``width_bytes`` between device and pinned host memory, stream ordered."""
    s = ctypes.c_void_p(stream if stream is not None else torch.cuda.current_stream(device_index).cuda_stream)
    _lib.check(_lib.lib().dprt_copy_2d(device_index, ctypes.c_void_p(dst), dst_pitch, ctypes.c_void_p(src), src_pitch,
                                       width_bytes, rows, s), "dprt_copy_2d")


def enable_peer(device_index: int, peer_index: int) -> None:
    """NVLink peer access from ``device_index`` to ``peer_index`` (idempotent; TransportError if impossible)."""
    _lib.check(_lib.lib().dprt_enable_peer(device_index, peer_index), "dprt_enable_peer")


def ipc_handle(device_index: int, ptr: int) -> bytes:
    buf = (ctypes.c_uint8 * 64)()
    _lib.check(_lib.lib().dprt_ipc_handle(device_index, ctypes.c_void_p(ptr), buf), "dprt_ipc_handle")
    return bytes(buf)


def ipc_open(device_index: int, handle: bytes) -> int:
    buf = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    out = ctypes.c_void_p()
    _lib.check(_lib.lib().dprt_ipc_open(device_index, buf, ctypes.byref(out)), "dprt_ipc_open")
    return int(out.value)


def ipc_close(device_index: int, ptr: int) -> None:
    _lib.check(_lib.lib().dprt_ipc_close(device_index, ctypes.c_void_p(ptr)), "dprt_ipc_close")


class DeviceBuffer:
    """Device memory from dprt_device_alloc (allocation base == pointer, so a CUDA IPC handle maps
    exactly this buffer), viewed as a torch tensor through __cuda_array_interface__."""

    def __init__(self, device: torch.device, numel: int, dtype=torch.float32):
        self.index = device.index if device.index is not None else torch.cuda.current_device()
        self.device = torch.device("cuda", self.index)
        self.numel = int(numel)
        self.dtype = dtype
        itemsize = torch.empty((), dtype=dtype).element_size()
        self.nbytes = self.numel * itemsize
        p = ctypes.c_void_p()
        _lib.check(_lib.lib().dprt_device_alloc(self.index, self.nbytes, ctypes.byref(p)), "dprt_device_alloc")
        self.ptr = int(p.value)
        typestr = {torch.float32: "<f4", torch.float16: "<f2", torch.uint8: "|u1", torch.int32: "<i4"}[dtype]
        self.__cuda_array_interface__ = {"shape": (self.numel,), "typestr": typestr, "data": (self.ptr, False),
                                         "version": 3, "strides": None}
        self.tensor = torch.as_tensor(self, device=self.device)

    def close(self) -> None:
        if self.ptr:
            torch.cuda.synchronize(self.device)
            _lib.check(_lib.lib().dprt_device_free(self.index, ctypes.c_void_p(self.ptr)), "dprt_device_free")
            self.ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
