"""Fused sort-last compositor over peer memory (NVLink P2P): exchange + blend + gather in one kernel.

Each rank marches straight into a buffer that every peer has mapped (CUDA IPC handles exchanged once on
the control plane).  After a stream-ordered device barrier (an NCCL all-reduce: it completes on a rank
only once every rank's march has finished), rank j launches ONE composite kernel whose P input pointers
are the peers' partial buffers offset to row block j (``assign_pixels``, engine.py:216-221), in
visibility order, and whose RGB8 output pointer is rank 0's frame at row block j.  The fragment reads
((1 - 1/P) * W * H * 16 B per rank) and the tile writes into rank 0 (3 B/px) cross NVLink inside that
kernel; a second device barrier publishes the frame to rank 0 and keeps peers from overwriting a
partial that is still being read.  This replaces both the reference's ring cycling of ray batches
(engine.py:282-310) and its linear gather_to_root of f64 tiles (engine.py:485, transport.py:465-475).
"""

from __future__ import annotations

from typing import Optional, Sequence

import torch

from . import device as dev
from .compositor import CompositeOutput, assign_rows, clip_rows
from .transport import RankEndpoint


class P2PCompositor:
    def __init__(self, ep: RankEndpoint, width: int, height: int, device: torch.device,
                 fragment_dtype: torch.dtype = torch.float32):
        """Collective.  Local failures never skip a collective call: they leave ``self.ok`` False."""
        self.ep = ep
        self.fdt = fragment_dtype
        self.px = 8 if fragment_dtype == torch.float16 else 16  # fragment bytes per pixel
        self.W = width
        self.H = height
        self.device = device
        self.index = device.index if device.index is not None else torch.cuda.current_device()
        n = width * height
        self.ok = True
        self.partial = self.frame = self.frame_rgba = None
        try:
            self.partial = dev.DeviceBuffer(device, n * 4, fragment_dtype)
            if ep.rank == 0:
                self.frame = dev.DeviceBuffer(device, n * 3, torch.uint8)
        except Exception:  # noqa: BLE001 - reported through self.ok
            self.ok = False
        self.peer_partials = ep.share_pointers(self.index, self.partial.ptr if self.partial else 0)
        self.root_frame = ep.share_pointers(self.index, self.frame.ptr if self.frame else 0)[0]
        self.ok = self.ok and all(self.peer_partials) and self.root_frame != 0
        self.root_rgba = 0
        self.last_bytes = 0

    @classmethod
    def try_create(cls, ep: RankEndpoint, width: int, height: int, device: torch.device,
                   fragment_dtype: torch.dtype = torch.float32) -> Optional["P2PCompositor"]:
        """Collectively set up peer mappings; every rank gets None if any rank cannot (no NVLink P2P,
        IPC refused, ...), so the caller can pick the NCCL exchange instead -- on every rank alike."""
        impl = cls(ep, width, height, device, fragment_dtype)
        flags = ep.all_gather_bytes(b"1" if impl.ok else b"0")
        if all(f == b"1" for f in flags):
            return impl
        impl.close()
        return None

    def _ensure_rgba(self) -> None:
        if self.root_rgba:
            return
        if self.ep.rank == 0:
            self.frame_rgba = dev.DeviceBuffer(self.device, self.W * self.H * 4)
        self.root_rgba = self.ep.share_pointers(self.index, self.frame_rgba.ptr if self.frame_rgba else 0)[0]

    def composite(self, partial: torch.Tensor, order: Sequence[int], background, keep_float: bool = False,
                  bands=None) -> CompositeOutput:
        ep = self.ep
        if keep_float:
            self._ensure_rgba()
        if partial.data_ptr() != self.partial.ptr:
            self.partial.tensor.copy_(partial)
        ep.device_barrier()  # every rank's partial is complete
        rows = assign_rows(self.H, ep.R)[ep.rank]
        npix = (rows[1] - rows[0]) * self.W
        if npix:
            off = rows[0] * self.W
            if bands is None:
                ptrs = [self.peer_partials[s] + self.px * off for s in order]
                ranges = None
            else:  # read each peer only inside its footprint rows (the rest of its partial is clear)
                ptrs, ranges = [], []
                for s in order:
                    c = clip_rows(rows, bands[s])
                    if c:
                        ptrs.append(self.peer_partials[s] + self.px * c[0] * self.W)
                        ranges.append(((c[0] - rows[0]) * self.W, (c[1] - rows[0]) * self.W))
                if not ptrs:
                    ptrs, ranges = [self.peer_partials[ep.rank]], [(0, 0)]
            dev.composite_ptrs(self.index, ptrs, npix, background, rgb8_ptr=self.root_frame + 3 * off,
                               rgba_ptr=(self.root_rgba + 16 * off) if keep_float else 0, ranges=ranges,
                               half=self.fdt == torch.float16)
        ep.device_barrier()  # every tile has landed in rank 0's frame
        if bands is None:
            self.last_bytes = self.px * npix * (ep.R - 1) + (3 * npix if ep.rank else 0)
        else:
            read = sum((c[1] - c[0]) * self.W for s in range(ep.R) if s != ep.rank
                       for c in [clip_rows(rows, bands[s])] if c)
            self.last_bytes = self.px * read + (3 * npix if ep.rank else 0)
        if ep.rank != 0:
            return CompositeOutput(None, None)
        frame = self.frame.tensor.view(self.H, self.W, 3)
        return CompositeOutput(frame, self.frame_rgba.tensor if keep_float else None)

    def close(self) -> None:
        self.ep.unshare_pointers(self.index, self.peer_partials)
        for buf in (self.partial, self.frame, self.frame_rgba):
            if buf is not None:
                buf.close()
