"""Sort-last compositing of per-rank RGBA partials: direct-send, binary-swap and fused peer-memory.

The reference resolves cross-rank visibility by cycling every ray through every rank and reducing with
the commutative (t, gid) min (pkg/src/dprt/engine.py:282-310, bvh.py:246-248), then gathers disjoint
row tiles to rank 0 (engine.py:443-456, 485; transport.py:465-475).  Volume partials need the
non-commutative 'over' in brick visibility order instead, so this module exchanges image fragments:

* ``direct_send``: one round; rank j receives row block j (``assign_pixels``, engine.py:216-221) of every
  other rank's partial, blends the P fragments in visibility order with the fused tone map, and sends
  its RGB8 tile to rank 0.  On NVSwitch every peer is one hop at full bandwidth, so this is the default.
* ``binary_swap``: log2(P) rounds; in round k rank r trades half of its current row range with
  r XOR 2^k and blends the two group composites (front group first).  Needs P a power of two and a
  visibility order in which every aligned rank group is contiguous (true for kd decompositions).
* ``p2p``: one kernel per rank reads the P fragments of its row block straight out of the peers'
  partial buffers over NVLink (CUDA IPC mappings), blends, tone-maps and writes the RGB8 tile directly
  into rank 0's frame -- the exchange, the blend and the gather fused.
* ``p2p_push``: the march itself writes each row block of its partial into the block owner's inbox over
  NVLink as its tiles finish (the exchange overlaps the march), epoch flags in peer memory replace the
  barriers, and the blend reads local memory only (``p2p.P2PPushCompositor``).

Fragment bytes per rank per frame are (1 - 1/P)*W*H*16 in both exchange modes.  The
blend itself always runs in libdprt_cuda.so (``CudaBlender``); there is no CPU blend in the product.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import torch

from .errors import TransportError, UsageError
from .transport import RankEndpoint


def clip_rows(rows: Tuple[int, int], band: Tuple[int, int]) -> Optional[Tuple[int, int]]:
    """rows ∩ band, or None when empty."""
    lo, hi = max(rows[0], band[0]), min(rows[1], band[1])
    return (lo, hi) if hi > lo else None


def assign_rows(height: int, P: int) -> List[Tuple[int, int]]:
    """Row blocks [b*H//P, (b+1)*H//P) -- engine.py:216-221."""
    return [(b * height // P, (b + 1) * height // P) for b in range(P)]


@dataclass(frozen=True)
class DirectSendPlan:
    rank: int
    own_rows: Tuple[int, int]
    sends: Tuple[Tuple[int, Tuple[int, int]], ...]   # (peer, rows of MY partial that peer owns)
    recvs: Tuple[int, ...]                           # peers whose fragment of own_rows I receive


def direct_send_plan(height: int, P: int, rank: int) -> DirectSendPlan:
    blocks = assign_rows(height, P)
    sends = tuple((j, blocks[j]) for j in range(P) if j != rank)
    recvs = tuple(j for j in range(P) if j != rank)
    return DirectSendPlan(rank, blocks[rank], sends, recvs)


@dataclass(frozen=True)
class SwapRound:
    k: int
    partner: int
    keep: Tuple[int, int]   # block range kept after the round
    give: Tuple[int, int]   # block range sent to the partner
    my_group: Tuple[int, int]       # rank range [g0, g1) my current composite covers
    partner_group: Tuple[int, int]


def binary_swap_plan(P: int, rank: int) -> Tuple[List[SwapRound], int]:
    """Rounds for ``rank`` and the final row block it ends up owning (bit-reversed rank)."""
    if P < 1 or P & (P - 1):
        raise UsageError(f"binary-swap needs a power-of-two rank count, got {P}")
    rounds: List[SwapRound] = []
    b0, b1 = 0, P
    k = 0
    while (1 << k) < P:
        partner = rank ^ (1 << k)
        mid = (b0 + b1) // 2
        lower, upper = (b0, mid), (mid, b1)
        keep, give = (lower, upper) if not (rank >> k) & 1 else (upper, lower)
        size = 1 << k
        g0 = (rank >> k) << k
        p0 = (partner >> k) << k
        rounds.append(SwapRound(k, partner, keep, give, (g0, g0 + size), (p0, p0 + size)))
        b0, b1 = keep
        k += 1
    return rounds, b0


class CudaBlender:
    """The product blender: libdprt_cuda.so's composite kernel."""

    def over(self, frags: Sequence[torch.Tensor], out_rgba: torch.Tensor) -> None:
        from . import device as dev
        dev.composite(frags, None, rgba=out_rgba)

    def over_tonemap(self, frags: Sequence[torch.Tensor], background, out_rgb8: torch.Tensor,
                     out_rgba: Optional[torch.Tensor] = None, ranges=None, npix: Optional[int] = None) -> None:
        from . import device as dev
        dev.composite(frags, background, rgb8=out_rgb8, rgba=out_rgba, ranges=ranges, npix=npix)


@dataclass
class CompositeOutput:
    rgb8: Optional[torch.Tensor]   # rank 0: (H, W, 3) uint8
    rgba: Optional[torch.Tensor]   # rank 0 with keep_float: (H*W*4) f32 blended, no background


class Compositor:
    """Per-rank compositing state for one frame size (scratch buffers persist across frames)."""

    def __init__(self, ep: RankEndpoint, width: int, height: int, mode: str, device: torch.device,
                 blender=None, fragment_dtype: torch.dtype = torch.float32):
        self.ep = ep
        self.W = width
        self.H = height
        self.device = device
        self.mode_requested = mode
        self.mode = self.resolve_mode(mode, ep.R)
        if fragment_dtype not in (torch.float32, torch.float16):
            raise UsageError(f"fragments are float32 or float16, not {fragment_dtype}")
        if fragment_dtype == torch.float16 and self.mode in ("binary_swap", "cycle"):
            raise UsageError("fp16 fragments are exchanged by direct_send / p2p / auto only")
        self.fdt = fragment_dtype
        self.blender = blender if blender is not None else CudaBlender()
        self.last_bytes = 0
        self._frame = None
        self._frame_rgba = None
        self._scratch: Dict[str, torch.Tensor] = {}

    @staticmethod
    def resolve_mode(mode: str, P: int) -> str:
        if P == 1:
            return "single"
        if mode == "auto":
            return "auto"  # p2p if every rank can map its peers (decided collectively), else direct_send
        if mode == "binary_swap" and P & (P - 1):
            raise UsageError(f"binary_swap needs a power-of-two rank count, got {P}")
        if mode not in ("direct_send", "binary_swap", "p2p", "p2p_push", "cycle"):
            raise UsageError(f"unknown composite mode {mode!r}")
        return mode  # "cycle": the renderer moves rays, this object only gathers the tiles

    def _buf(self, name: str, numel: int, dtype=torch.float32) -> torch.Tensor:
        t = self._scratch.get(name)
        if t is None or t.numel() < numel or t.dtype != dtype:
            t = torch.empty(numel, dtype=dtype, device=self.device)
            self._scratch[name] = t
        return t[:numel]

    def _frame_buffers(self, keep_float: bool):
        if self._frame is None:
            self._frame = torch.empty((self.H, self.W, 3), dtype=torch.uint8, device=self.device)
        if keep_float and self._frame_rgba is None:
            self._frame_rgba = torch.empty(self.H * self.W * 4, dtype=torch.float32, device=self.device)
        return self._frame, (self._frame_rgba if keep_float else None)

    def _rows(self, flat: torch.Tensor, rows: Tuple[int, int], ch: int) -> torch.Tensor:
        return flat[rows[0] * self.W * ch: rows[1] * self.W * ch]

    def clips_bands(self) -> bool:
        """True when this mode reads only each rank's footprint row band (``bands`` in composite)."""
        return self.mode in ("direct_send", "p2p", "p2p_push")

    # ------------------------------------------------------------------------------------------
    def composite(self, partial: torch.Tensor, order: Sequence[int], background, keep_float: bool = False,
                  solo: bool = False, bands: Optional[Sequence[Tuple[int, int]]] = None) -> CompositeOutput:
        """``bands``: per rank, the rows [y0, y1) outside which its partial is clear (its screen footprint):
        direct-send and p2p then move and read only those rows."""
        order = list(order)
        if sorted(order) != list(range(self.ep.R)):
            raise UsageError(f"visibility order {order} is not a permutation of {self.ep.R} ranks")
        self.last_bytes = 0
        if self.mode == "auto":
            self.shared_partial()  # resolves auto collectively
        if self.mode == "single" or solo:
            return self._single(partial, background, keep_float)
        if bands is not None and len(bands) != self.ep.R:
            raise UsageError(f"need one row band per rank, got {len(bands)}")
        if self.mode == "direct_send":
            return self._direct_send(partial, order, background, keep_float, bands)
        if self.mode == "binary_swap":
            return self._binary_swap(partial, order, background, keep_float)
        if self.mode == "p2p_push":
            # the march already pushed this frame's fragments (push_targets); blend what arrived
            out = self._push().composite(order, background, keep_float, bands)
            self.last_bytes = self._push_impl.last_bytes
            return out
        return self._p2p_composite(partial, order, background, keep_float, bands)

    def _push(self):
        if getattr(self, "_push_impl", None) is None:
            from .p2p import P2PPushCompositor
            impl = P2PPushCompositor.try_create(self.ep, self.W, self.H, self.device, self.fdt)
            if impl is None:
                raise TransportError("p2p_push needs every rank on its own GPU with its peers' buffers mapped "
                                     "(CUDA IPC over NVLink); use composite='p2p' or 'direct_send'")
            self._push_impl = impl
        return self._push_impl

    def push_targets(self):
        """p2p_push: start a frame and return the march's push targets (row_start, dst, flags, counter,
        epoch); None in every other mode (the march writes the local partial)."""
        if self.mode != "p2p_push":
            return None
        return self._push().march_targets()

    def _single(self, partial, background, keep_float) -> CompositeOutput:
        if self.ep.rank != 0:
            return CompositeOutput(None, None)
        frame, rgba = self._frame_buffers(keep_float)
        self.blender.over_tonemap([partial], background, frame.view(-1), rgba)
        return CompositeOutput(frame, rgba)

    def _gather_tiles(self, rows: Tuple[int, int], tile_rgb8: torch.Tensor, tile_rgba: Optional[torch.Tensor],
                      all_rows: Sequence[Tuple[int, int]], keep_float: bool) -> CompositeOutput:
        """Final gather of RGB8 (and optionally RGBA) row tiles to rank 0 (engine.py:485-487)."""
        ep = self.ep
        if ep.rank == 0:
            frame, frame_rgba = self._frame_buffers(keep_float)
            flat = frame.view(-1)
            recvs = []
            for src in range(1, ep.R):
                r = all_rows[src]
                if r[1] > r[0]:
                    recvs.append((src, self._rows(flat, r, 3)))
                    if keep_float:
                        recvs.append((src, self._rows(frame_rgba, r, 4)))
            own = self._rows(flat, rows, 3)
            if tile_rgb8.data_ptr() != own.data_ptr():
                own.copy_(tile_rgb8)
            if keep_float:
                own_f = self._rows(frame_rgba, rows, 4)
                if tile_rgba.data_ptr() != own_f.data_ptr():
                    own_f.copy_(tile_rgba)
            ep.exchange([], recvs)
            return CompositeOutput(frame, frame_rgba)
        sends = []
        if rows[1] > rows[0]:
            sends.append((0, tile_rgb8))
            if keep_float:
                sends.append((0, tile_rgba))
        ep.exchange(sends, [])
        self.last_bytes += sum(t.numel() * t.element_size() for _, t in sends)
        return CompositeOutput(None, None)

    def _direct_send(self, partial, order, background, keep_float, bands=None) -> CompositeOutput:
        ep = self.ep
        P, r = ep.R, ep.rank
        plan = direct_send_plan(self.H, P, r)
        rows = plan.own_rows
        n_own = (rows[1] - rows[0]) * self.W
        full = (0, self.H)
        band = [full] * P if bands is None else list(bands)
        # every rank derives the same clipped row ranges from the same bands: no sizes are exchanged
        sends = []
        for j, rr in plan.sends:
            c = clip_rows(rr, band[r])
            if c:
                sends.append((j, self._rows(partial, c, 4)))
        clips = {s: clip_rows(rows, band[s]) for s in range(P)}
        inbox = {s: self._buf(f"in{s}", (clips[s][1] - clips[s][0]) * self.W * 4, self.fdt)[
                    : (clips[s][1] - clips[s][0]) * self.W * 4] for s in plan.recvs if clips[s]}
        recvs = [(s, inbox[s]) for s in plan.recvs if clips[s]]
        ep.exchange(sends, recvs)
        self.last_bytes += sum(t.numel() * t.element_size() for _, t in sends)
        frags, ranges = [], []
        for s in order:
            c = clips[s]
            if not c:
                continue  # this rank's footprint misses my rows: its fragment is clear
            frags.append(self._rows(partial, c, 4) if s == r else inbox[s])
            ranges.append(((c[0] - rows[0]) * self.W, (c[1] - rows[0]) * self.W))
        tile = self._buf("tile8", n_own * 3, torch.uint8)
        tile_f = self._buf("tilef", n_own * 4) if keep_float else None
        if n_own:
            if not frags:  # every fragment clear: the background alone
                frags, ranges = [self._buf("tilef0", 4, self.fdt)], [(0, 0)]
            if bands is None:
                self.blender.over_tonemap(frags, background, tile, tile_f)
            else:
                self.blender.over_tonemap(frags, background, tile, tile_f, ranges=ranges, npix=n_own)
        return self._gather_tiles(rows, tile, tile_f, assign_rows(self.H, P), keep_float)

    def _binary_swap(self, partial, order, background, keep_float) -> CompositeOutput:
        ep = self.ep
        P, r = ep.R, ep.rank
        pos = {s: i for i, s in enumerate(order)}
        rounds, final_block = binary_swap_plan(P, r)
        blocks = assign_rows(self.H, P)

        def rows_of(br):
            return (blocks[br[0]][0], blocks[br[1] - 1][1])

        cur = partial          # full-frame-indexed buffer holding my current group composite
        work = [self._buf("swapA", self.H * self.W * 4), self._buf("swapB", self.H * self.W * 4)]
        for i, rd in enumerate(rounds):
            keep_rows, give_rows = rows_of(rd.keep), rows_of(rd.give)
            n_keep = (keep_rows[1] - keep_rows[0]) * self.W
            inbox = self._buf("swapIn", max(n_keep, 1) * 4)[: n_keep * 4]
            send = self._rows(cur, give_rows, 4)
            ep.exchange([(rd.partner, send)] if send.numel() else [], [(rd.partner, inbox)] if n_keep else [])
            self.last_bytes += send.numel() * 4
            mine = self._rows(cur, keep_rows, 4)
            mine_front = min(pos[s] for s in range(*rd.my_group)) < min(pos[s] for s in range(*rd.partner_group))
            frags = [mine, inbox] if mine_front else [inbox, mine]
            last = i == len(rounds) - 1
            if not last:
                out = work[i % 2]
                if n_keep:
                    self.blender.over(frags, self._rows(out, keep_rows, 4))
                cur = out
            else:
                tile = self._buf("tile8", n_keep * 3, torch.uint8)
                tile_f = self._buf("tilef", n_keep * 4) if keep_float else None
                if n_keep:
                    self.blender.over_tonemap(frags, background, tile, tile_f)
                final_rows = rows_of((final_block, final_block + 1))
                assert final_rows == keep_rows
                finals = [binary_swap_plan(P, s)[1] for s in range(P)]
                all_rows = [rows_of((b, b + 1)) for b in finals]
                return self._gather_tiles(keep_rows, tile, tile_f, all_rows, keep_float)
        raise AssertionError("binary swap with P > 1 always has a last round")

    def shared_partial(self) -> Optional[torch.Tensor]:
        """The buffer the marcher should write into (peer-mapped in p2p mode), or None for any buffer.
        In ``auto`` mode this is where the fused path is chosen: every rank tries to map its peers'
        buffers and the group switches to p2p only if all succeed (collective), else to direct_send."""
        if self.mode == "auto":
            impl = None
            if self.device.type == "cuda":
                from .p2p import P2PCompositor
                impl = P2PCompositor.try_create(self.ep, self.W, self.H, self.device, self.fdt)
            self._p2p_impl = impl
            self.mode = "p2p" if impl is not None else "direct_send"
        if self.mode != "p2p":
            return None
        return self._p2p().partial.tensor

    def _p2p(self):
        if getattr(self, "_p2p_impl", None) is None:
            from .p2p import P2PCompositor
            impl = P2PCompositor.try_create(self.ep, self.W, self.H, self.device, self.fdt)
            if impl is None:
                raise TransportError("p2p compositing needs every rank to map its peers' buffers "
                                     "(CUDA IPC over NVLink); use composite='direct_send'")
            self._p2p_impl = impl
        return self._p2p_impl

    def _p2p_composite(self, partial, order, background, keep_float, bands=None) -> CompositeOutput:
        out = self._p2p().composite(partial, order, background, keep_float, bands)
        self.last_bytes = self._p2p_impl.last_bytes
        return out
