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
        self._root_frames = ep.share_pointers(self.index, self.frame.ptr if self.frame else 0)
        self.root_frame = self._root_frames[0]
        self.ok = self.ok and all(self.peer_partials) and self.root_frame != 0
        self.root_rgba = 0
        self._root_rgbas = None
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
        self._root_rgbas = self.ep.share_pointers(self.index, self.frame_rgba.ptr if self.frame_rgba else 0)
        self.root_rgba = self._root_rgbas[0]

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
        for ptrs in (self.peer_partials, self._root_frames, self._root_rgbas):
            if ptrs:
                self.ep.unshare_pointers(self.index, ptrs)
        for buf in (self.partial, self.frame, self.frame_rgba):
            if buf is not None:
                buf.close()


# ------------------------------------------------------------------------------------------------------
# Fused march + exchange ("p2p_push"): the march itself writes each row block of the partial
# into the block owner's inbox over NVLink while it runs, so the fragment exchange overlaps the march tile
# by tile; per-source epoch flags in the owner's memory replace the stream-ordered NCCL barriers.



class PushLayout:
    """Pointer arithmetic of the fused march + exchange -- pure, shared by the compositor and the
    single-GPU emulation test.  Rank j's inbox holds, per frame parity (epoch & 1) and source rank s, a
    slot of ``slot`` pixels: s's fragment of j's row block (``assign_pixels``, engine.py:216-221), pixel
    (x, y) at element (y - block_start) * W + x.  Double buffering by parity is what makes the flags
    sufficient: source s's march of frame k follows its own blend of frame k-1 on its stream, and that blend
    waited for every source's march of frame k-1, which followed every rank's blend of frame k-2 -- the
    last reader of this parity's slots."""

    def __init__(self, P: int, width: int, height: int, px_bytes: int):
        self.P, self.W, self.H, self.es = P, width, height, px_bytes
        self.blocks = assign_rows(height, P)
        self.row_start = [b[0] for b in self.blocks] + [height]
        self.slot = max(b1 - b0 for b0, b1 in self.blocks) * width  # pixels per (parity, source) slot

    def inbox_pixels(self) -> int:
        return 2 * self.P * self.slot

    # A rank's flag buffer (int32 words): [0, P) fragment arrivals (one epoch word per source), [P, 2P) frame
    # rows done (read on rank 0), then two DPRT_SIGNAL_COUNTER_WORDS counter sets (march, blend), 128-byte
    # aligned.
    def counter_offset(self, which: int) -> int:
        """Byte offset of counter set ``which`` (0 = march, 1 = blend) in a flag buffer."""
        return 4 * ((2 * self.P + 31) // 32 * 32 + which * dev._lib.SIGNAL_COUNTER_WORDS)

    def flag_words(self) -> int:
        return self.counter_offset(2) // 4

    def slot_ptr(self, inbox_base: int, epoch: int, src: int) -> int:
        return inbox_base + self.es * (((epoch & 1) * self.P + src) * self.slot)

    def march_targets(self, peer_inbox: Sequence[int], peer_flags: Sequence[int], rank: int, epoch: int):
        """(dst, flags) for source ``rank``'s march of frame ``epoch``: its slot at every block owner."""
        dst = [self.slot_ptr(peer_inbox[j], epoch, rank) for j in range(self.P)]
        return dst, [peer_flags[j] + 4 * rank for j in range(self.P)]

    def fragments(self, inbox_base: int, rank: int, epoch: int, order: Sequence[int], bands=None):
        """Blend inputs of ``rank``'s block in visibility order: (pointers, pixel ranges or None, pixels
        received from other ranks).  With ``bands`` a source's fragment covers only its footprint rows."""
        rows = self.blocks[rank]
        ptrs, ranges, recv = [], [], 0
        for s in order:
            base = self.slot_ptr(inbox_base, epoch, s)
            if bands is None:
                ptrs.append(base)
                ranges.append((0, (rows[1] - rows[0]) * self.W))
                recv += 0 if s == rank else (rows[1] - rows[0]) * self.W
                continue
            c = clip_rows(rows, bands[s])
            if c:
                ptrs.append(base + self.es * (c[0] - rows[0]) * self.W)
                ranges.append(((c[0] - rows[0]) * self.W, (c[1] - rows[0]) * self.W))
                recv += 0 if s == rank else (c[1] - c[0]) * self.W
        if not ptrs:  # no footprint meets this block: the background alone
            ptrs, ranges = [self.slot_ptr(inbox_base, epoch, rank)], [(0, 0)]
        return ptrs, (None if bands is None else ranges), recv


def _device_identity(index: int) -> str:
    import socket

    props = torch.cuda.get_device_properties(index)
    return f"{socket.gethostname()}:{getattr(props, 'uuid', index)}"


class P2PPushCompositor:
    """Fused march + exchange over peer memory (one process, or one thread, per GPU).

    Per frame (epoch e = 1, 2, ...): ``march_targets()`` -> the engine's ``dprt_march_push`` writes this
    rank's partial straight into every block owner's inbox slot and raises its epoch flag there when its
    last CTA retires; ``composite()`` waits (one spinning warp, stream-ordered) until all P sources' flags
    of this rank's block reach e, blends them from local memory into rank 0's frame over NVLink and raises
    rank 0's done flag for this block; rank 0 then waits for every block's done flag, so its frame is
    complete in stream order -- no NCCL call per frame.  Needs every rank on its own GPU (a spinning wait
    must never share a GPU with the work it waits for): ``try_create`` checks that collectively."""

    def __init__(self, ep: RankEndpoint, width: int, height: int, device: torch.device,
                 fragment_dtype: torch.dtype = torch.float32, _emulated: bool = False):
        """``_emulated`` (tests only): accept ranks that share a GPU.  Such ranks must then issue every
        rank's march before any rank's ``composite`` and rank 0's last, from ONE thread on one stream, so
        that every flag wait is satisfied when it is issued (tests/test_gpu_push.py)."""
        self.ep = ep
        self.fdt = fragment_dtype
        self.px = 8 if fragment_dtype == torch.float16 else 16
        self.W, self.H = width, height
        self.device = device
        self.index = device.index if device.index is not None else torch.cuda.current_device()
        self.layout = PushLayout(ep.R, width, height, self.px)
        self.ok = ep.R <= dev._lib.MAX_PUSH
        self.inbox = self.flags = self.frame = self.frame_rgba = None
        self.epoch = 0
        try:
            if self.ok:
                self.inbox = dev.DeviceBuffer(device, self.layout.inbox_pixels() * 4, fragment_dtype)
                self.flags = dev.DeviceBuffer(device, self.layout.flag_words(), torch.int32)
                self.flags.tensor.zero_()
                if ep.rank == 0:
                    self.frame = dev.DeviceBuffer(device, width * height * 3, torch.uint8)
                torch.cuda.synchronize(device)
        except Exception:  # noqa: BLE001 - reported through self.ok
            self.ok = False
        ids = ep.all_gather_bytes(_device_identity(self.index).encode() if device.type == "cuda" else b"cpu")
        self.distinct = len(set(ids)) == len(ids) or _emulated
        self.peer_inbox = ep.share_pointers(self.index, self.inbox.ptr if self.inbox else 0)
        self.peer_flags = ep.share_pointers(self.index, self.flags.ptr if self.flags else 0)
        self._root_frames = ep.share_pointers(self.index, self.frame.ptr if self.frame else 0)
        self.root_frame = self._root_frames[0]
        self.ok = self.ok and self.distinct and all(self.peer_inbox) and all(self.peer_flags) and self.root_frame != 0
        self.root_rgba = 0
        self._root_rgbas = None
        self.last_bytes = 0

    @classmethod
    def try_create(cls, ep: RankEndpoint, width: int, height: int, device: torch.device,
                   fragment_dtype: torch.dtype = torch.float32) -> Optional["P2PPushCompositor"]:
        """Collective: every rank gets the compositor, or every rank gets None (peers not mappable, ranks
        sharing a GPU, more than DPRT_MAX_PUSH ranks)."""
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
        self._root_rgbas = self.ep.share_pointers(self.index, self.frame_rgba.ptr if self.frame_rgba else 0)
        self.root_rgba = self._root_rgbas[0]

    def march_targets(self):
        """Start a frame: (row_start, dst pointers, flag pointers, counter pointer, epoch) for dprt_march_push."""
        self.epoch += 1
        dst, fl = self.layout.march_targets(self.peer_inbox, self.peer_flags, self.ep.rank, self.epoch)
        return self.layout.row_start, dst, fl, self.flags.ptr + self.layout.counter_offset(0), self.epoch

    def composite(self, order: Sequence[int], background, keep_float: bool = False, bands=None) -> CompositeOutput:
        ep, L, e = self.ep, self.layout, self.epoch
        if keep_float:
            self._ensure_rgba()
        r = ep.rank
        dev.wait_flags(self.index, self.flags.ptr, ep.R, e)  # every source's fragment of my block has landed
        rows = L.blocks[r]
        npix = (rows[1] - rows[0]) * self.W
        ptrs, ranges, recv = L.fragments(self.inbox.ptr, r, e, order, bands)
        off = rows[0] * self.W
        dev.composite_signal(self.index, ptrs, npix, background, self.root_frame + 3 * off,
                             (self.root_rgba + 16 * off) if keep_float else 0, ranges,
                             self.flags.ptr + L.counter_offset(1), [self.peer_flags[0] + 4 * (ep.R + r)], e,
                             half=self.fdt == torch.float16)
        # bytes this rank moved over NVLink this frame: its pushed fragments (those of the other blocks) and
        # its RGB8 rows into rank 0's frame
        sent = 0
        for j in range(ep.R):
            if j == r:
                continue
            bj = L.blocks[j]
            c = bj if bands is None else clip_rows(bj, bands[r])
            if c:
                sent += (c[1] - c[0]) * self.W
        self.last_bytes = self.px * sent + (3 * npix if r else 0)
        if r != 0:
            return CompositeOutput(None, None)
        dev.wait_flags(self.index, self.flags.ptr + 4 * ep.R, ep.R, e)  # every block's rows are in my frame
        frame = self.frame.tensor.view(self.H, self.W, 3)
        return CompositeOutput(frame, self.frame_rgba.tensor if keep_float else None)

    def close(self) -> None:
        for ptrs in (self.peer_inbox, self.peer_flags, self._root_frames, self._root_rgbas):
            if ptrs:
                self.ep.unshare_pointers(self.index, ptrs)
        for buf in (self.inbox, self.flags, self.frame, self.frame_rgba):
            if buf is not None:
                buf.close()
