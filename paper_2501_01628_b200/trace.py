"""Triangle traversal on the GPU -- the reference's per-rank compute slot, as a drop-in.

The reference's triangle renderer spends its per-rank time in two numba functions over a BVH's flat arrays,
``trace_nearest_batch`` and ``trace_any_batch`` (pkg/src/dprt/bvh.py:284-311), called with identical
arguments by ``engine.trace_local_round`` (engine.py:254-279) on every hop of the ray-queue cycle
(``cycle_batch``, engine.py:282-310).  This module puts both behind ``dprt_trace_nearest`` /
``dprt_trace_any`` (csrc/trace.cu), bit-identical to the reference (float64, the reference's evaluation
order, no contraction):

* ``trace_nearest_batch`` / ``trace_any_batch`` -- the same signature as the numba functions, host numpy
  arrays in, results written in place; the BVH is uploaded once per Accel and cached.  Assigning them to
  ``dprt.engine.trace_nearest_batch`` / ``trace_any_batch`` runs the reference's whole triangle renderer on
  the GPU (tests/test_gpu_trace.py does exactly that against the unmodified install).
* ``DeviceBvh`` + ``DeviceRayBatch`` -- device-resident BVH and ray batch for GPU ray cycling
  (``cycle_batch_device``): the batch stays in HBM and moves between ranks as device tensors (NCCL on a
  multi-GPU box), only the traversal slot changes per hop.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Dict, Tuple

import numpy as np
import torch

from . import _lib
from .errors import UsageError

MISS_ID = np.iinfo(np.int64).max  # bvh.py:25
MAX_DEPTH = 62                    # the traversal stack holds 64 entries (bvh.py:23): depth + 1 <= 63 < 64


def bvh_depth(left: np.ndarray, right: np.ndarray, root: int) -> int:
    """Depth of the tree (root = 0); the traversal stack needs depth + 1 entries."""
    if root < 0:
        return 0
    depth, level = 0, [int(root)]
    while level:
        nxt = []
        for n in level:
            if left[n] >= 0:
                nxt.append(int(left[n]))
            if right[n] >= 0:
                nxt.append(int(right[n]))
        if nxt:
            depth += 1
        level = nxt
    return depth


class DeviceBvh:
    """A rank's BVH (the reference's Accel arrays, bvh.py:46-60) resident on one GPU."""

    def __init__(self, node_lo, node_hi, node_left, node_right, node_first, node_count, root, tri_v, tri_id,
                 device: torch.device):
        left = np.ascontiguousarray(node_left, np.int64)
        right = np.ascontiguousarray(node_right, np.int64)
        if bvh_depth(left, right, int(root)) > MAX_DEPTH:
            raise UsageError(f"BVH deeper than {MAX_DEPTH} levels: the traversal stack holds 64 entries")
        self.device = device
        self.index = device.index if device.index is not None else torch.cuda.current_device()

        def up(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a, dt)).to(device)

        self._t = [up(node_lo, np.float64), up(node_hi, np.float64), up(left, np.int64), up(right, np.int64),
                   up(node_first, np.int64), up(node_count, np.int64), up(tri_v, np.float64), up(tri_id, np.int64)]
        n_nodes, n_prims = len(left), int(np.asarray(tri_id).shape[0])
        p = [ctypes.c_void_p(t.data_ptr()) for t in self._t]
        self.struct = _lib.Bvh(p[0], p[1], p[2], p[3], p[4], p[5], n_nodes, int(root), p[6], p[7], n_prims)

    @classmethod
    def from_accel(cls, accel, device: torch.device) -> "DeviceBvh":
        return cls(accel.node_lo, accel.node_hi, accel.node_left, accel.node_right, accel.node_first,
                   accel.node_count, accel.root, accel.tri_v, accel.tri_id, device)

    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def trace_nearest(self, org: torch.Tensor, dirn: torch.Tensor, tmin: torch.Tensor, tmax: torch.Tensor,
                      best_t: torch.Tensor, best_id: torch.Tensor) -> None:
        """Device tensors, (best_t, best_id) min-reduced in place (stream ordered)."""
        n = _check_rays(org, dirn, tmin, tmax)
        _check(best_t, torch.float64, (n,), "best_t")
        _check(best_id, torch.int64, (n,), "best_id")
        rc = _lib.lib().dprt_trace_nearest(self.index, ctypes.byref(self.struct), n, _p(org), _p(dirn), _p(tmin),
                                           _p(tmax), _p(best_t), _p(best_id), self._stream())
        _lib.check(rc, "dprt_trace_nearest")

    def trace_any(self, org: torch.Tensor, dirn: torch.Tensor, tmin: torch.Tensor, tmax: torch.Tensor,
                  occluded: torch.Tensor) -> None:
        n = _check_rays(org, dirn, tmin, tmax)
        _check(occluded, torch.uint8, (n,), "occluded")
        rc = _lib.lib().dprt_trace_any(self.index, ctypes.byref(self.struct), n, _p(org), _p(dirn), _p(tmin),
                                       _p(tmax), _p(occluded), self._stream())
        _lib.check(rc, "dprt_trace_any")


def _p(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _check(t: torch.Tensor, dtype, shape, name: str) -> None:
    if not t.is_cuda or t.dtype != dtype or tuple(t.shape) != tuple(shape) or not t.is_contiguous():
        raise UsageError(f"{name} must be a contiguous CUDA {dtype} tensor of shape {tuple(shape)}, got "
                         f"{t.dtype} {tuple(t.shape)} on {t.device}")


def _check_rays(org, dirn, tmin, tmax) -> int:
    n = int(tmin.shape[0]) if tmin.dim() == 1 else -1
    _check(org, torch.float64, (n, 3), "org")
    _check(dirn, torch.float64, (n, 3), "dirn")
    _check(tmin, torch.float64, (n,), "tmin")
    _check(tmax, torch.float64, (n,), "tmax")
    return n


# ---------------------------------------------------------------------------------------------------------
# drop-in for the numba slot (host arrays, in place)

_CACHE: Dict[Tuple[int, int], Tuple[object, DeviceBvh]] = {}


def _device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def _cached_bvh(node_lo, node_hi, node_left, node_right, node_first, node_count, root, tri_v, tri_id) -> DeviceBvh:
    """An Accel's arrays never change after build_bvh (bvh.py:105-157): upload once per array object."""
    dev = _device()
    key = (id(tri_v), dev.index)
    hit = _CACHE.get(key)
    if hit is not None and hit[0] is tri_v:
        return hit[1]
    if len(_CACHE) > 32:
        _CACHE.clear()
    b = DeviceBvh(node_lo, node_hi, node_left, node_right, node_first, node_count, root, tri_v, tri_id, dev)
    _CACHE[key] = (tri_v, b)
    return b


def _rays_to_device(org, dirn, tmin, tmax, dev):
    return [torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(dev, non_blocking=False)
            for a in (org, dirn, tmin, tmax)]


def trace_nearest_batch(node_lo, node_hi, node_left, node_right, node_first, node_count, root, tri_v, tri_id,
                        org, dirn, tmin, tmax, best_t, best_id) -> None:
    """Drop-in for bvh.trace_nearest_batch (bvh.py:284-296): min-reduce each ray's (best_t, best_id) against
    the local BVH, in place -- on the GPU."""
    n = int(np.asarray(tmin).shape[0])
    if n == 0:
        return
    b = _cached_bvh(node_lo, node_hi, node_left, node_right, node_first, node_count, root, tri_v, tri_id)
    o, d, t0, t1 = _rays_to_device(org, dirn, tmin, tmax, b.device)
    bt = torch.from_numpy(np.ascontiguousarray(best_t, np.float64)).to(b.device)
    bi = torch.from_numpy(np.ascontiguousarray(best_id, np.int64)).to(b.device)
    b.trace_nearest(o, d, t0, t1, bt, bi)
    best_t[:] = bt.cpu().numpy()
    best_id[:] = bi.cpu().numpy()


def trace_any_batch(node_lo, node_hi, node_left, node_right, node_first, node_count, root, tri_v, tri_id,
                    org, dirn, tmin, tmax, occluded) -> None:
    """Drop-in for bvh.trace_any_batch (bvh.py:299-311): OR-reduce each ray's occlusion flag, in place."""
    n = int(np.asarray(tmin).shape[0])
    if n == 0:
        return
    b = _cached_bvh(node_lo, node_hi, node_left, node_right, node_first, node_count, root, tri_v, tri_id)
    o, d, t0, t1 = _rays_to_device(org, dirn, tmin, tmax, b.device)
    occ = torch.from_numpy(np.ascontiguousarray(occluded, np.uint8)).to(b.device)
    b.trace_any(o, d, t0, t1, occ)
    occluded[:] = occ.cpu().numpy()


# ---------------------------------------------------------------------------------------------------------
# device-resident ray cycling (engine.py:282-310 with the batch in HBM)


@dataclass
class DeviceRayBatch:
    """The traversal-relevant fields of the reference's RayBatch (engine.py:47-70) on the device, packed in
    one f64 buffer per batch so a ring hop is ONE tensor exchange: columns org(3) dirn(3) tmin tmax best_t,
    then best_id (int64 bits) and occluded (0/1) as f64 bit patterns."""

    kind: int                 # engine.PRIMARY / SHADOW / REFLECTION
    buf: torch.Tensor         # (n, 11) float64
    rounds_completed: int = 0
    owner: int = 0

    COLS = 11

    @staticmethod
    def from_host(kind: int, org, dirn, tmin, tmax, best_t, best_id, occluded, device, owner: int = 0):
        n = int(np.asarray(tmin).shape[0])
        a = np.empty((n, DeviceRayBatch.COLS), np.float64)
        a[:, 0:3] = org
        a[:, 3:6] = dirn
        a[:, 6] = tmin
        a[:, 7] = tmax
        a[:, 8] = best_t
        a[:, 9] = np.ascontiguousarray(best_id, np.int64).view(np.float64)
        a[:, 10] = occluded
        return DeviceRayBatch(kind, torch.from_numpy(a).to(device), 0, owner)

    def __len__(self) -> int:
        return int(self.buf.shape[0])

    def results(self):
        """(best_t, best_id, occluded) as host arrays."""
        a = self.buf.cpu().numpy()
        return a[:, 8].copy(), a[:, 9].copy().view(np.int64), (a[:, 10] != 0).astype(np.uint8)


def _trace_device_batch(b: DeviceBvh, batch: DeviceRayBatch, shadow_kind: int) -> None:
    """One local round on the device batch: the columns are gathered into contiguous tensors, traced, and
    scattered back (the slot's arrays must be contiguous)."""
    n = len(batch)
    if n == 0:
        return
    x = batch.buf
    org, dirn = x[:, 0:3].contiguous(), x[:, 3:6].contiguous()
    tmin, tmax = x[:, 6].contiguous(), x[:, 7].contiguous()
    if batch.kind == shadow_kind:
        occ = (x[:, 10] != 0).to(torch.uint8)
        b.trace_any(org, dirn, tmin, tmax, occ)
        x[:, 10] = occ.to(torch.float64)
    else:
        bt = x[:, 8].contiguous()
        bi = x[:, 9].contiguous().view(torch.int64)
        b.trace_nearest(org, dirn, tmin, tmax, bt, bi)
        x[:, 8] = bt
        x[:, 9] = bi.view(torch.float64)


def cycle_batch_device(ep, batch: DeviceRayBatch, bvh: DeviceBvh, shadow_kind: int = 1,
                       disable_cycling: bool = False) -> DeviceRayBatch:
    """engine.cycle_batch (engine.py:282-310) with the batch on the device: R rounds of (trace locally, hand
    the batch to rank + 1) over the endpoint's data plane (device tensors: NCCL isend/irecv across GPUs,
    device copies between rank threads), so after R hops the batch is home; asserts it, like the reference."""
    rounds = 1 if disable_cycling else ep.R
    for _ in range(rounds):
        _trace_device_batch(bvh, batch, shadow_kind)
        batch.rounds_completed += 1
        if rounds > 1:
            # sizes travel on the control plane (the ring neighbours' batch lengths differ)
            n_in = int(ep.ring_exchange(str(len(batch)).encode()))
            owner_in = int(ep.ring_exchange(str(batch.owner).encode()))
            incoming = torch.empty((n_in, DeviceRayBatch.COLS), dtype=torch.float64, device=batch.buf.device)
            sends = [((ep.rank + 1) % ep.R, batch.buf)] if len(batch) else []
            recvs = [((ep.rank - 1) % ep.R, incoming)] if n_in else []
            ep.exchange(sends, recvs)
            batch = DeviceRayBatch(batch.kind, incoming, batch.rounds_completed, owner_in)
    if batch.rounds_completed != rounds:
        raise AssertionError(f"rank {ep.rank}: batch completed {batch.rounds_completed} rounds, expected {rounds}")
    if rounds > 1 and batch.owner != ep.rank:
        raise AssertionError(f"cycled batch did not return home (rank {ep.rank})")
    return batch
