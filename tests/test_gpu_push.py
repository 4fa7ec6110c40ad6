"""Fused march + exchange ("p2p_push") on ONE GPU by sequential emulation.

The production path needs every rank on its own GPU: a rank's blend waits (one spinning warp) for the
epoch flags its peers' marches raise, and such a wait must never share a GPU with the work it waits for.
Here the R ranks' buffers all live on cuda:0 and one thread issues, on one stream, every rank's
``dprt_march_push`` first and only then every rank's flag wait + ``dprt_composite_signal`` -- so each
wait is already satisfied when it is issued and no kernel ever waits on a kernel that is not complete
(the emulation B200_PROFILING.md prescribes for fewer GPUs than ranks).  The pointer arithmetic is the
production one (``p2p.PushLayout``); every frame must be byte-identical to marching into local partials
and compositing them with ``dprt_composite`` (same kernels, same fragment values, other destinations),
and every epoch flag must carry the frame's epoch afterwards."""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.compositor import clip_rows
from paper_2501_01628_b200.geom import orbit_camera
from paper_2501_01628_b200.p2p import PushLayout
from scenes import c1

pytestmark = pytest.mark.gpu


def _bands(dec, cam, W, H):
    return [tuple(dev.desc_footprint(dec.brick(s), cam, W, H)[1::2]) for s in range(dec.P)]


@pytest.mark.parametrize("P,W,H,clip,half", [(2, 160, 122, True, False), (3, 157, 113, True, False),
                                            (4, 176, 130, False, False), (4, 176, 130, True, True),
                                            (8, 128, 96, True, False)])
def test_push_frames_equal_local_march_and_composite(cuda_device, P, W, H, clip, half):
    s = c1(P=P, W=W, H=H)
    bb = s.field.bounds()
    cams = [s.cam] + [orbit_camera(bb.center(), 1.3 * bb.diagonal(), math.radians(35.0 * k), math.radians(15.0),
                                   45.0, W / H) for k in range(1, 4)]
    _push_vs_local(cuda_device, s, cams, P, W, H, clip, half)


@pytest.mark.parametrize("P", [4, 8])
def test_push_frames_with_offscreen_bricks_and_an_eye_inside(cuda_device, P):
    """Cameras for which some bricks have no footprint at all (narrow view of one corner: their pushes are
    background-only and whole row blocks blend nothing but the background) and one inside a brick."""
    from paper_2501_01628_b200.geom import CameraSpec

    W, H = 150, 110
    s = c1(P=P, W=W, H=H)
    lo, hi = s.field.bounds().lo, s.field.bounds().hi

    def at(fx, fy, fz):  # a point in field-relative coordinates
        return tuple(lo[i] + f * (hi[i] - lo[i]) for i, f in enumerate((fx, fy, fz)))

    inside = at(0.3, 0.3, 0.3)
    centre = s.field.bounds().center()

    def look(pos, tgt, fov):
        v = tuple(t - p for t, p in zip(tgt, pos))
        n = math.sqrt(sum(c * c for c in v))
        return CameraSpec(pos, tuple(c / n for c in v), (0.0, 1.0, 0.0), fov, W / H)

    # axis-parallel narrow views down one corner column of the field: bricks away from it project nowhere
    cams = [look(at(0.1, 0.1, -1.5), at(0.1, 0.1, 0.5), 10.0), look(at(-1.5, 0.9, 0.85), at(0.5, 0.9, 0.85), 6.0),
            look(inside, centre, 60.0), look(inside, tuple(2 * p - c for p, c in zip(inside, centre)), 75.0)]
    bands = [[tuple(dev.desc_footprint(s.dec.brick(r), c, W, H)[1::2]) for r in range(P)] for c in cams[:2]]
    assert any(b[1] <= b[0] for bl in bands for b in bl), "the narrow views should leave some brick off-screen"
    _push_vs_local(cuda_device, s, cams, P, W, H, True, False)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("DPRT_PUSH_FUZZ_CASES", "12"))))
def test_push_fuzz(cuda_device, seed):
    """Seeded random push scenes: P in 2..8, odd frame sizes (row blocks of unequal height), random orbit
    cameras incl. close-ups, band clipping on / off, fp16 fragments; byte-identical to march + composite."""
    rng = np.random.default_rng(5000 + seed)
    P = int(rng.integers(2, 9))
    W, H = int(rng.integers(24, 200)), int(rng.integers(P, 160))
    s = c1(P=P, W=W, H=H)
    bb = s.field.bounds()
    cams = [orbit_camera(bb.center(), float(rng.uniform(0.4, 1.6)) * bb.diagonal(),
                         math.radians(float(rng.uniform(0, 360))), math.radians(float(rng.uniform(-60, 60))),
                         float(rng.uniform(20, 80)), W / H) for _ in range(3)]
    _push_vs_local(cuda_device, s, cams, P, W, H, bool(rng.integers(0, 2)), bool(rng.integers(0, 4) == 0))


def _push_vs_local(cuda_device, s, cams, P, W, H, clip, half):
    d = cuda_device
    fdt = torch.float16 if half else torch.float32
    L = PushLayout(P, W, H, 8 if half else 16)
    bricks = [dev.DeviceBrick(s.dec.brick(r), d).generate(s.field) for r in range(P)]
    dtf = dev.DeviceTF(s.tf, d)
    inbox = [torch.full((L.inbox_pixels() * 4,), float("nan"), dtype=fdt, device=d) for _ in range(P)]
    flags = [torch.zeros(L.flag_words(), dtype=torch.int32, device=d) for _ in range(P)]
    frame = torch.zeros((H, W, 3), dtype=torch.uint8, device=d)
    ib = [t.data_ptr() for t in inbox]
    fb = [t.data_ptr() for t in flags]
    for epoch, cam in enumerate(cams, start=1):
        order = s.dec.visibility_order(cam.position)
        bands = _bands(s.dec, cam, W, H) if clip else None
        # every rank's march first (pushing into every owner's inbox slot, raising its flags) ...
        for r in range(P):
            dst, fl = L.march_targets(ib, fb, r, epoch)
            dev.march_push(bricks[r], cam, dtf, s.dt, s.ert, W, H, L.row_start, dst, fl, fb[r] + L.counter_offset(0),
                           epoch, band_clear=clip, half=half)
        # ... then every rank's wait + blend into rank 0's frame (+ rank 0's done flag), then rank 0's wait
        for r in range(P):
            dev.wait_flags(d.index, fb[r], P, epoch)
            rows = L.blocks[r]
            ptrs, ranges, _ = L.fragments(ib[r], r, epoch, order, bands)
            dev.composite_signal(d.index, ptrs, (rows[1] - rows[0]) * W, s.background,
                                 frame.data_ptr() + 3 * rows[0] * W, 0, ranges, fb[r] + L.counter_offset(1),
                                 [fb[0] + 4 * (P + r)], epoch, half=half)
        dev.wait_flags(d.index, fb[0] + 4 * P, P, epoch)
        got = frame.cpu().numpy().copy()
        # reference: local partials + one composite of the whole frame in visibility order
        parts = []
        for r in range(P):
            part = torch.empty(H * W * 4, dtype=fdt, device=d)
            dev.march(bricks[r], cam, dtf, s.dt, s.ert, part, W, H)
            parts.append(part)
        ref = torch.empty(H * W * 3, dtype=torch.uint8, device=d)
        dev.composite([parts[o] for o in order], s.background, rgb8=ref)
        assert np.array_equal(got, ref.view(H, W, 3).cpu().numpy()), f"frame {epoch} differs"
        for r in range(P):
            f = flags[r].cpu().numpy()
            assert (f[:P] == epoch).all(), f"rank {r} arrival flags {f[:P]} at epoch {epoch}"
            assert not f[L.counter_offset(0) // 4:].any()  # the CTA counters reset themselves
        assert (flags[0].cpu().numpy()[P:2 * P] == epoch).all()
        if clip:  # the pushed rows of each source are exactly its footprint band within each block
            for r in range(P):
                for src in range(P):
                    rows = L.blocks[r]
                    c = clip_rows(rows, bands[src])
                    slot = inbox[r][(L.slot_ptr(0, epoch, src) // L.es) * 4:][: (rows[1] - rows[0]) * W * 4]
                    written = ~torch.isnan(slot.view(-1, 4)[:, 0].float())
                    if c:
                        lo, hi = (c[0] - rows[0]) * W, (c[1] - rows[0]) * W
                        assert bool(written[lo:hi].all())
    for b in bricks:
        b.close()


def test_push_targets_reject_bad_layouts(cuda_device):
    s = c1(P=2, W=64, H=48)
    d = cuda_device
    b = dev.DeviceBrick(s.dec.brick(0), d).generate(s.field)
    dtf = dev.DeviceTF(s.tf, d)
    buf = torch.zeros(64 * 48 * 4, device=d)
    fl = torch.zeros(4 + 2 * 1056, dtype=torch.int32, device=d)
    ok = dict(row_start=[0, 24, 48], dst=[buf.data_ptr(), buf.data_ptr()], flag_ptrs=[fl.data_ptr(), fl.data_ptr() + 4],
              counter_ptr=fl.data_ptr() + 128, epoch=1)
    dev.march_push(b, s.cam, dtf, s.dt, s.ert, 64, 48, **ok)
    from paper_2501_01628_b200.errors import UsageError
    for bad in (dict(row_start=[0, 24, 40]), dict(epoch=0), dict(dst=[buf.data_ptr() + 4, buf.data_ptr()]),
                dict(flag_ptrs=[fl.data_ptr(), 0])):
        with pytest.raises(UsageError):
            dev.march_push(b, s.cam, dtf, s.dt, s.ert, 64, 48, **{**ok, **bad})
    torch.cuda.synchronize()
    b.close()


def test_push_compositor_class_sequential_emulation(cuda_device):
    """P2PPushCompositor itself (collective set-up over the in-process endpoint, march_targets, composite
    with its flag waits and the signal into rank 0's frame), driven for R ranks sharing cuda:0 in the only
    safe order: every rank's push march, then ranks R-1 .. 1's blends, then rank 0's (whose wait for every
    block's done flag is then satisfied).  Frames must equal local marches + one composite, byte for byte."""
    from paper_2501_01628_b200.p2p import P2PPushCompositor
    from paper_2501_01628_b200.transport import run_collective

    P, W, H = 4, 144, 104
    s = c1(P=P, W=W, H=H)
    d = cuda_device
    def make(ep):
        c = P2PPushCompositor(ep, W, H, d, _emulated=True)
        c._ensure_rgba()  # collective: the float RGBA gather target (keep_float frames)
        return c

    comps = run_collective(P, make, device=d)
    assert all(c.ok for c in comps)
    bricks = [dev.DeviceBrick(s.dec.brick(r), d).generate(s.field) for r in range(P)]
    dtf = dev.DeviceTF(s.tf, d)
    bb = s.field.bounds()
    cams = [s.cam] + [orbit_camera(bb.center(), 1.25 * bb.diagonal(), math.radians(50.0 * k), math.radians(-10.0),
                                   45.0, W / H) for k in range(1, 4)]
    for cam in cams:
        order = s.dec.visibility_order(cam.position)
        bands = _bands(s.dec, cam, W, H)
        for r in range(P):
            row_start, dst, fl, counter, epoch = comps[r].march_targets()
            dev.march_push(bricks[r], cam, dtf, s.dt, s.ert, W, H, row_start, dst, fl, counter, epoch, band_clear=True)
        kf = cam is cams[-1]  # the last frame also gathers the float RGBA (keep_float) into rank 0
        outs = {r: comps[r].composite(order, s.background, keep_float=kf, bands=bands) for r in list(range(1, P)) + [0]}
        assert all(outs[r].rgb8 is None for r in range(1, P))
        got = outs[0].rgb8.cpu().numpy().copy()
        got_rgba = outs[0].rgba.cpu().numpy().copy() if kf else None
        parts = []
        for r in range(P):
            part = torch.empty(H * W * 4, dtype=torch.float32, device=d)
            dev.march(bricks[r], cam, dtf, s.dt, s.ert, part, W, H)
            parts.append(part)
        ref = torch.empty(H * W * 3, dtype=torch.uint8, device=d)
        ref_rgba = torch.empty(H * W * 4, dtype=torch.float32, device=d)
        dev.composite([parts[o] for o in order], s.background, rgb8=ref, rgba=ref_rgba)
        assert np.array_equal(got, ref.view(H, W, 3).cpu().numpy())
        if kf:
            assert np.array_equal(got_rgba, ref_rgba.cpu().numpy())
        assert comps[1].last_bytes > 0
    torch.cuda.synchronize()
    for c in comps:
        c.close()
    for b in bricks:
        b.close()
