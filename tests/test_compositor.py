"""Sort-last exchange schedules (direct-send, binary-swap) on CPU ranks over gloo, world sizes 2 and 4.

The product blend is the CUDA kernel; these CPU tests inject ``TorchBlender`` (a test-only stand-in
with the kernel's f32 arithmetic) so the schedule, the fragment exchange and the final gather are
exercised without a GPU.  The result is compared with the oracle's f64 'over' of all partials.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from dist_util import run_ranks
from paper_2501_01628_b200.compositor import (Compositor, assign_rows, binary_swap_plan, clip_rows,
                                              direct_send_plan)
from paper_2501_01628_b200.volume import binary_swap_compatible, blob_field, decompose


class TorchBlender:
    """Test-only CPU blender: same f32 front-to-back over + tone map as composite.cu."""

    @staticmethod
    def _over(frags):
        acc = frags[0].view(-1, 4).float().clone()
        for f in frags[1:]:
            acc = acc + (1.0 - acc[:, 3:4]) * f.view(-1, 4).float()
        return acc

    def over(self, frags, out_rgba):
        out_rgba.view(-1, 4).copy_(self._over(frags))

    def over_tonemap(self, frags, background, out_rgb8, out_rgba=None, ranges=None, npix=None):
        if ranges is not None:  # ranged fragments: clear outside [lo, hi) of the tile
            full = []
            for f, (lo, hi) in zip(frags, ranges):
                t = torch.zeros(npix * 4, dtype=torch.float32)
                t[lo * 4: hi * 4] = f.view(-1)[: (hi - lo) * 4].float()
                full.append(t)
            frags = full
        acc = self._over(frags)
        bg = torch.tensor(background, dtype=torch.float32)
        rgb = acc[:, :3] + (1.0 - acc[:, 3:4]) * bg
        q = torch.floor(torch.clamp(rgb, 0.0, 1.0) * 255.0 + 0.5).to(torch.uint8)
        out_rgb8.view(-1, 3).copy_(q)
        if out_rgba is not None:
            out_rgba.view(-1, 4).copy_(acc)


def _partials(P, W, H, seed=5):
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.0, 0.5, (P, H, W, 1))
    rgb = rng.uniform(0.0, 1.0, (P, H, W, 3)) * a
    return np.concatenate([rgb, a], axis=3).astype(np.float32)


def _rank_body(ep, mode, W, H, order, bg):
    parts = _partials(ep.R, W, H)
    mine = torch.from_numpy(parts[ep.rank].reshape(-1).copy())
    comp = Compositor(ep, W, H, mode, torch.device("cpu"), blender=TorchBlender())
    outs = []
    for _ in range(2):  # scratch reuse across frames
        out = comp.composite(mine, order, bg, keep_float=True)
        if ep.rank == 0:
            outs.append((out.rgb8.numpy().copy(), out.rgba.numpy().copy()))
    return outs, comp.last_bytes


@pytest.mark.parametrize("mode,P", [("direct_send", 2), ("direct_send", 3), ("direct_send", 4),
                                    ("binary_swap", 2), ("binary_swap", 4)])
def test_exchange_matches_oracle(mode, P):
    W, H = 24, 19  # H not divisible by P: uneven row blocks
    f = blob_field((33, 17, 17))
    dec = decompose(f, P)
    order = dec.visibility_order((-5.0, 40.0, 9.0))
    assert mode != "binary_swap" or binary_swap_compatible(order)
    bg = (0.1, 0.2, 0.3)
    res = run_ranks(P, _rank_body, mode, W, H, order, bg)
    parts = _partials(P, W, H).astype(np.float64)
    ref = oracle.composite(list(parts), order, bg)
    ref8 = oracle.tone_map_rgb8(ref)
    outs, _ = res[0]
    for rgb8, rgba in outs:
        rgba = rgba.reshape(H, W, 4).astype(np.float64)
        img = rgba[..., :3] + (1 - rgba[..., 3:4]) * np.asarray(bg)
        assert np.abs(img - ref).max() < 1e-5
        assert np.abs(rgb8.astype(np.int16) - ref8.astype(np.int16)).max() <= 1
    # fragment bytes per non-root rank: (1 - 1/P) of the frame in RGBA f32 + its RGB8 (+RGBA) tile to root
    for r in range(1, P):
        assert res[r][1] > 0


def _banded_body(ep, W, H, order, bg, bands):
    parts = _partials(ep.R, W, H)
    for s, (y0, y1) in enumerate(bands):  # each rank's partial is clear outside its footprint rows
        parts[s, :y0] = 0.0
        parts[s, y1:] = 0.0
    mine = torch.from_numpy(parts[ep.rank].reshape(-1).copy())
    comp = Compositor(ep, W, H, "direct_send", torch.device("cpu"), blender=TorchBlender())
    out = comp.composite(mine, order, bg, keep_float=True, bands=bands)
    clipped = comp.last_bytes
    full = comp.composite(mine, order, bg, keep_float=True)
    if ep.rank == 0:
        return out.rgb8.numpy().copy(), out.rgba.numpy().copy(), full.rgba.numpy().copy(), clipped, comp.last_bytes
    return None, None, None, clipped, comp.last_bytes


@pytest.mark.parametrize("P", [2, 3, 4])
def test_band_clipped_direct_send_equals_full_exchange(P):
    """Band-clipped direct-send (only footprint rows move) gives the same frame as the full exchange and
    sends fewer bytes; bands may be empty, cover everything, or miss whole row blocks."""
    W, H = 20, 23
    bands = [(3, 11), (0, 23), (9, 9), (15, 23)][:P]
    order = list(reversed(range(P)))
    bg = (0.1, 0.2, 0.3)
    res = run_ranks(P, _banded_body, W, H, order, bg, bands)
    rgb8, rgba, rgba_full, _, _ = res[0]
    assert np.array_equal(rgba, rgba_full)
    parts = _partials(P, W, H).astype(np.float64)
    for s, (y0, y1) in enumerate(bands):
        parts[s, :y0] = 0.0
        parts[s, y1:] = 0.0
    ref = oracle.composite(list(parts), order, bg)
    img = rgba.reshape(H, W, 4).astype(np.float64)
    assert np.abs(img[..., :3] + (1 - img[..., 3:4]) * np.asarray(bg) - ref).max() < 1e-5
    assert sum(r[3] for r in res) < sum(r[4] for r in res)


def _half_body(ep, W, H, order, bg):
    parts = _partials(ep.R, W, H)
    mine = torch.from_numpy(parts[ep.rank].reshape(-1).copy()).half()
    comp = Compositor(ep, W, H, "direct_send", torch.device("cpu"), blender=TorchBlender(),
                      fragment_dtype=torch.float16)
    out = comp.composite(mine, order, bg, keep_float=True)
    return (out.rgba.numpy().copy() if ep.rank == 0 else None), comp.last_bytes


def test_fp16_fragments_direct_send():
    """fp16 fragments move half the bytes; the blend of the rounded fragments matches the oracle composite
    of the same rounded data."""
    P, W, H = 3, 16, 11
    order = [2, 0, 1]
    bg = (0.1, 0.2, 0.3)
    res = run_ranks(P, _half_body, W, H, order, bg)
    parts = _partials(P, W, H).astype(np.float16).astype(np.float64)
    ref = oracle.composite(list(parts), order, bg)
    rgba = res[0][0].reshape(H, W, 4).astype(np.float64)
    assert np.abs(rgba[..., :3] + (1 - rgba[..., 3:4]) * np.asarray(bg) - ref).max() < 1e-5
    with pytest.raises(Exception, match="fp16"):
        fake_ep = type("Ep", (), {"R": 2, "rank": 0})()
        Compositor(fake_ep, W, H, "binary_swap", torch.device("cpu"), fragment_dtype=torch.float16)


def test_direct_send_plan_covers_every_block_once():
    for P in (1, 2, 3, 8):
        H = 37
        seen = {}
        for r in range(P):
            plan = direct_send_plan(H, P, r)
            assert plan.own_rows == assign_rows(H, P)[r]
            for peer, rows in plan.sends:
                seen.setdefault(peer, []).append(r)
                assert rows == assign_rows(H, P)[peer]
        for j in range(P):
            assert sorted(seen.get(j, [])) == [r for r in range(P) if r != j]


def test_binary_swap_plan_partners_and_final_blocks():
    for P in (2, 4, 8, 16):
        finals = []
        for r in range(P):
            rounds, final = binary_swap_plan(P, r)
            assert len(rounds) == P.bit_length() - 1
            for rd in rounds:
                prounds, _ = binary_swap_plan(P, rd.partner)
                prd = prounds[rd.k]
                assert prd.partner == r and prd.keep == rd.give and prd.give == rd.keep
            finals.append(final)
        assert sorted(finals) == list(range(P))  # every row block ends on exactly one rank
    with pytest.raises(Exception):
        binary_swap_plan(6, 0)


def test_kd_orders_are_binary_swap_compatible():
    rng = np.random.default_rng(3)
    for P in (2, 4, 8):
        f = blob_field((65, 49, 33), spacing=(1.0, 1.3, 2.0))
        dec = decompose(f, P)
        for _ in range(20):
            eye = tuple(rng.uniform(-100, 200, 3))
            assert binary_swap_compatible(dec.visibility_order(eye))


@pytest.mark.parametrize("P,W,H", [(2, 64, 48), (3, 157, 113), (8, 3840, 2160), (5, 33, 7)])
def test_push_layout_slots_are_disjoint_and_consistent(P, W, H):
    """p2p_push pointer arithmetic (p2p.PushLayout): per (parity, source) slots tile the inbox without
    overlap; the slot a source pushes into at owner j is the one owner j blends for that source; the
    band-clipped ranges are the pull compositor's (clip of the owner's block by the source's band)."""
    from paper_2501_01628_b200.p2p import PushLayout

    L = PushLayout(P, W, H, 16)
    assert L.row_start[0] == 0 and L.row_start[-1] == H and len(L.row_start) == P + 1
    spans = sorted((L.slot_ptr(0, e, s), L.slot_ptr(0, e, s) + 16 * L.slot) for e in (1, 2) for s in range(P))
    for (a0, a1), (b0, _) in zip(spans, spans[1:]):
        assert a1 <= b0
    assert spans[-1][1] <= 16 * L.inbox_pixels()
    bases = [1 << 40 | (j << 32) for j in range(P)]
    flags = [1 << 44 | (j << 32) for j in range(P)]
    rng = np.random.default_rng(P)
    for epoch in (1, 2, 3):
        order = list(rng.permutation(P))
        bands = [tuple(sorted(rng.integers(0, H + 1, 2))) for _ in range(P)]
        for src in range(P):
            dst, fl = L.march_targets(bases, flags, src, epoch)
            assert fl == [flags[j] + 4 * src for j in range(P)]
            for j in range(P):
                assert dst[j] == L.slot_ptr(bases[j], epoch, src)
        for j in range(P):
            ptrs, ranges, recv = L.fragments(bases[j], j, epoch, order, bands)
            rows = L.blocks[j]
            want = [(s, clip_rows(rows, bands[s])) for s in order if clip_rows(rows, bands[s])]
            if not want:
                assert ranges == [(0, 0)]
                continue
            assert len(ptrs) == len(want)
            for p, (lo, hi), (s, c) in zip(ptrs, ranges, want):
                assert p == L.slot_ptr(bases[j], epoch, s) + 16 * (c[0] - rows[0]) * W
                assert (lo, hi) == ((c[0] - rows[0]) * W, (c[1] - rows[0]) * W)
            assert recv == sum((c[1] - c[0]) * W for s, c in want if s != j)
