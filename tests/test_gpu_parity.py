"""GPU parity: the sm_100a data path through the C ABI against the CPU oracle on the same inputs.

Integer / byte work is compared exactly (field voxels, per-pixel owned sample counts, brick ownership,
visibility order); float RGBA within RGBA_ATOL (tests/scenes.py); RGB8 within 1 LSB.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.engine import RenderOptions, VolumeRenderer
from paper_2501_01628_b200.geom import CameraSpec, auto_camera, orbit_camera
from paper_2501_01628_b200.transport import SoloEndpoint
from paper_2501_01628_b200.volume import BrickDesc, blob_field, decompose, default_tf
from scenes import (RGB8_MAX_LSB, RGBA_ATOL, RGBA_MEAN_ATOL, c1, cam_array, dense_tf, oracle_brick,
                    oracle_partials)

pytestmark = pytest.mark.gpu


def _gpu_partials(dec, cam, tf, dt, ert, W, H, device, skip=True, ghost=1):
    dtf = dev.DeviceTF(tf, device)
    parts, samples = [], []
    for r in range(dec.P):
        b = dev.DeviceBrick(dec.brick(r, ghost), device).generate(dec.field)
        p = torch.empty(H * W * 4, dtype=torch.float32, device=device)
        s = torch.empty(H * W, dtype=torch.int32, device=device)
        dev.march(b, cam, dtf, dt, ert, p, W, H, samples=s, skip=skip)
        torch.cuda.synchronize()
        parts.append(p)
        samples.append(s)
        b.close()
    return parts, samples


def _check_rgba(gpu: np.ndarray, ref: np.ndarray, what: str):
    err = np.abs(gpu.astype(np.float64) - ref)
    assert err.max() <= RGBA_ATOL, f"{what}: max |dRGBA| {err.max():.3e} > {RGBA_ATOL}"
    assert err.mean() <= RGBA_MEAN_ATOL, f"{what}: mean |dRGBA| {err.mean():.3e}"


def test_field_generation_bit_exact(cuda_device, oracle_lib):
    f = blob_field((37, 29, 23), seed=5, n_blobs=16)
    for lo, hi, g in [((0, 0, 0), (36, 28, 22), 0), ((5, 3, 7), (20, 28, 15), 1), ((0, 10, 0), (36, 20, 22), 2)]:
        desc = BrickDesc(f.dims, lo, hi, g)
        b = dev.DeviceBrick(desc, cuda_device).generate(f)
        got = b.download()
        ref = oracle.generate_field(f.dims, f.blobs, desc.stored_lo, desc.stored_dims)
        assert np.array_equal(got, ref)
        b.close()


def test_upload_roundtrip(cuda_device):
    desc = BrickDesc((9, 8, 7), (0, 0, 0), (8, 7, 6), 0)
    vox = np.random.default_rng(0).random((7, 8, 9)).astype(np.float32)
    b = dev.DeviceBrick(desc, cuda_device).upload(vox)
    assert np.array_equal(b.download(), vox)
    b.close()


@pytest.mark.parametrize("skip", [False, True])
def test_single_brick_matches_oracle(cuda_device, oracle_lib, skip):
    f = blob_field((48, 40, 44), seed=7)
    vox = oracle.generate_field(f.dims, f.blobs)
    dec = decompose(f, 1)
    W, H = 96, 80
    for cam, tf, dt, ert in [(auto_camera(f.bounds(), W, H), default_tf(), 1.0, 0.99),
                             (auto_camera(f.bounds(), W, H), dense_tf(), 0.6, 0.95),
                             (CameraSpec((24.0, 20.0, 22.0), (0.2, 0.1, -1.0), (0, 1, 0), 80.0, W / H), dense_tf(),
                              0.8, 0.99)]:
        ref, rs = oracle_partials(vox, dec, cam, tf, dt, ert, W, H)
        parts, samples = _gpu_partials(dec, cam, tf, dt, ert, W, H, cuda_device, skip=skip)
        got = parts[0].view(H, W, 4).cpu().numpy()
        assert np.array_equal(samples[0].view(H, W).cpu().numpy().astype(np.uint32), rs[0])
        _check_rgba(got, ref[0], f"single brick skip={skip}")


@pytest.mark.parametrize("P", [2, 3, 8])
def test_bricks_and_composite_match_oracle(cuda_device, oracle_lib, P):
    """C1 (64^3, 256^2) at P bricks: per-brick partials, integer-exact sample ownership, exact
    visibility order, composite kernel vs oracle 'over' (float) and RGB8 within 1 LSB."""
    s = c1(P=P)
    vox = oracle.generate_field(s.field.dims, s.field.blobs)
    ref, rs = oracle_partials(vox, s.dec, s.cam, s.tf, s.dt, s.ert, s.W, s.H)
    parts, samples = _gpu_partials(s.dec, s.cam, s.tf, s.dt, s.ert, s.W, s.H, cuda_device)
    for r in range(P):
        assert np.array_equal(samples[r].view(s.H, s.W).cpu().numpy().astype(np.uint32), rs[r])
        _check_rgba(parts[r].view(s.H, s.W, 4).cpu().numpy(), ref[r], f"brick {r}")
    order = s.dec.visibility_order(s.cam.position)
    from scenes import oracle_order
    assert order == oracle_order(s.dec, s.cam.position)
    rgb8 = torch.empty(s.H * s.W * 3, dtype=torch.uint8, device=cuda_device)
    rgba = torch.empty(s.H * s.W * 4, dtype=torch.float32, device=cuda_device)
    dev.composite([parts[r] for r in order], s.background, rgb8=rgb8, rgba=rgba)
    torch.cuda.synchronize()
    img_ref = oracle.composite(ref, order, s.background)
    blended = rgba.view(s.H, s.W, 4).double().cpu().numpy()
    img = blended[..., :3] + (1.0 - blended[..., 3:4]) * np.asarray(s.background)
    assert np.abs(img - img_ref).max() <= RGBA_ATOL
    q = rgb8.view(s.H, s.W, 3).cpu().numpy().astype(np.int16)
    assert np.abs(q - oracle.tone_map_rgb8(img_ref).astype(np.int16)).max() <= RGB8_MAX_LSB


def test_composite_kernel_random_partials(cuda_device, oracle_lib):
    """Compositing-only (config 5 style): seeded premultiplied RGBA with alpha <= 0.5, odd pixel count."""
    rng = np.random.default_rng(11)
    P, npix = 5, 1000 * 37 + 3
    a = rng.uniform(0, 0.5, (P, npix, 1))
    parts = np.concatenate([rng.uniform(0, 1, (P, npix, 3)) * a, a], axis=2).astype(np.float32)
    order = [3, 0, 4, 1, 2]
    bg = (0.2, 0.3, 0.4)
    ts = [torch.from_numpy(parts[i].reshape(-1)).to(cuda_device) for i in range(P)]
    rgb8 = torch.empty(npix * 3, dtype=torch.uint8, device=cuda_device)
    rgba = torch.empty(npix * 4, dtype=torch.float32, device=cuda_device)
    dev.composite([ts[r] for r in order], bg, rgb8=rgb8, rgba=rgba)
    ref = oracle.composite([parts[i].astype(np.float64) for i in range(P)], order, bg)
    out = rgba.view(npix, 4).double().cpu().numpy()
    img = out[:, :3] + (1 - out[:, 3:4]) * np.asarray(bg)
    assert np.abs(img - ref).max() < 1e-5
    q = rgb8.view(npix, 3).cpu().numpy().astype(np.int16)
    assert np.abs(q - oracle.tone_map_rgb8(ref).astype(np.int16)).max() <= 1


def test_ranged_composite_kernel(cuda_device, oracle_lib):
    """dprt_composite_ranged: fragments clear outside [lo, hi) (edges not multiples of 4, empty and full
    ranges) equal the full-size composite of the zero-padded fragments, bit for bit."""
    rng = np.random.default_rng(12)
    P, npix = 6, 4097 * 3 + 2
    a = rng.uniform(0, 0.5, (P, npix, 1))
    parts = np.concatenate([rng.uniform(0, 1, (P, npix, 3)) * a, a], axis=2).astype(np.float32)
    ranges = [(0, npix), (5, 4001), (4001, 4001), (1234, npix), (0, 7), (333, 9998)]
    padded = np.zeros_like(parts)
    for i, (lo, hi) in enumerate(ranges):
        padded[i, lo:hi] = parts[i, lo:hi]
    bg = (0.2, 0.3, 0.4)
    full = [torch.from_numpy(padded[i].reshape(-1)).to(cuda_device) for i in range(P)]
    clip = [torch.from_numpy(parts[i, lo:hi].reshape(-1).copy() if hi > lo else np.zeros(4, np.float32)).to(cuda_device)
            for i, (lo, hi) in enumerate(ranges)]
    out = []
    for frags, rg in ((full, None), (clip, ranges)):
        rgb8 = torch.empty(npix * 3, dtype=torch.uint8, device=cuda_device)
        rgba = torch.empty(npix * 4, dtype=torch.float32, device=cuda_device)
        dev.composite(frags, bg, rgb8=rgb8, rgba=rgba, ranges=rg, npix=npix)
        torch.cuda.synchronize()
        out.append((rgb8.cpu().numpy(), rgba.cpu().numpy()))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    from paper_2501_01628_b200.errors import UsageError

    with pytest.raises(UsageError, match="range"):
        dev.composite(clip, bg, rgb8=torch.empty(npix * 3, dtype=torch.uint8, device=cuda_device),
                      ranges=[(0, npix + 1)] + ranges[1:], npix=npix)


def test_engine_single_rank_frame(cuda_device, oracle_lib):
    """The public per-rank driver at R=1 (render_with slot): RGB8 frame + float image vs oracle."""
    s = c1(P=1, W=160, H=120)
    vox = oracle.generate_field(s.field.dims, s.field.blobs)
    ref, _ = oracle_partials(vox, s.dec, s.cam, s.tf, s.dt, s.ert, s.W, s.H)
    img_ref = oracle.composite(ref, [0], s.background)
    brick = dev.DeviceBrick(s.dec.brick(0), cuda_device).generate(s.field)
    r = VolumeRenderer(SoloEndpoint(cuda_device), brick, s.dec, s.tf, s.background)
    res = r.render(s.cam, s.W, s.H, RenderOptions(keep_float=True))
    torch.cuda.synchronize()
    assert np.abs(res.image - img_ref).max() <= RGBA_ATOL
    q = res.rgb8.cpu().numpy().astype(np.int16)
    assert np.abs(q - oracle.tone_map_rgb8(img_ref).astype(np.int16)).max() <= RGB8_MAX_LSB
    brick.close()


def test_orbit_frames_order_and_ownership(cuda_device, oracle_lib):
    """Config-4 style: uneven anisotropic bricks, orbiting camera; order exact every frame, samples exact."""
    f = blob_field((72, 40, 24), seed=3, spacing=(1.0, 1.0, 2.0), lopsided=True)
    vox = oracle.generate_field(f.dims, f.blobs)

    def mass(axis, lo, hi):
        sub = vox[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] >= np.float32(0.1)
        return sub.sum(axis=tuple(a for a in range(3) if a != 2 - axis)).astype(np.int64)

    dec = decompose(f, 8, "mass", mass)
    leaves, nodes = oracle.kd_leaves(f.dims, f.spacing, 8, "mass", field=vox)
    assert [tuple(map(tuple, l)) for l in leaves] == dec.boxes
    W, H = 64, 48
    b = f.bounds()
    target = b.center()
    for i in range(6):
        cam = orbit_camera(target, 1.6 * b.diagonal(), np.radians(60.0 * i), np.radians(20.0), 45.0, W / H)
        order = dec.visibility_order(cam.position)
        assert order == oracle.kd_order(nodes, 8, cam.position, f.origin, f.spacing)
        ref, rs = oracle_partials(vox, dec, cam, dense_tf(), 1.0, 0.99, W, H)
        parts, samples = _gpu_partials(dec, cam, dense_tf(), 1.0, 0.99, W, H, cuda_device)
        for r in range(8):
            assert np.array_equal(samples[r].view(H, W).cpu().numpy().astype(np.uint32), rs[r])
            _check_rgba(parts[r].view(H, W, 4).cpu().numpy(), ref[r], f"frame {i} brick {r}")


def test_skip_cache_follows_tf_updates(cuda_device, oracle_lib):
    """The TF-dependent skip distances are cached per DeviceTF version; updating the TF (different
    empty range) must rebuild them so the frame still matches the oracle for the new TF."""
    from paper_2501_01628_b200.volume import TransferFunction1D

    f = blob_field((40, 36, 32), seed=8)
    vox = oracle.generate_field(f.dims, f.blobs)
    dec = decompose(f, 1)
    W, H = 64, 48
    cam = auto_camera(f.bounds(), W, H)
    b = dev.DeviceBrick(dec.brick(0), cuda_device).generate(f)
    tf_a = default_tf(threshold=0.6)
    t = dense_tf().as_f32().copy()
    t[:, 3] = np.where(np.arange(256) < 20, 0.0, 0.05)
    tf_b = TransferFunction1D(t, 0.0, 1.0)
    dtf = dev.DeviceTF(tf_a, cuda_device)
    p = torch.empty(H * W * 4, dtype=torch.float32, device=cuda_device)
    for tf in (tf_a, tf_b, tf_a):
        dtf.update(tf)
        dev.march(b, cam, dtf, 1.0, 0.99, p, W, H)
        torch.cuda.synchronize()
        ref, _ = oracle_partials(vox, dec, cam, tf, 1.0, 0.99, W, H)
        _check_rgba(p.view(H, W, 4).cpu().numpy(), ref[0], "after TF update")
    b.close()


def test_fused_single_rank_frame_equals_composited(cuda_device, oracle_lib, monkeypatch):
    """R == 1: dprt_march_rgb8 (over-background + tone map fused into the march) gives the same bytes as
    dprt_march + dprt_composite(P=1), and matches the oracle within 1 LSB."""
    s = c1(P=1, W=200, H=150)
    vox = oracle.generate_field(s.field.dims, s.field.blobs)
    ref, _ = oracle_partials(vox, s.dec, s.cam, s.tf, s.dt, s.ert, s.W, s.H)
    want = oracle.tone_map_rgb8(oracle.composite(ref, [0], s.background)).astype(np.int16)
    brick = dev.DeviceBrick(s.dec.brick(0), cuda_device).generate(s.field)
    r = VolumeRenderer(SoloEndpoint(cuda_device), brick, s.dec, s.tf, s.background)
    fused = r.render(s.cam, s.W, s.H).rgb8.cpu().numpy().copy()
    monkeypatch.setenv("DPRT_FUSED_SINGLE", "0")
    plain = r.render(s.cam, s.W, s.H).rgb8.cpu().numpy().copy()
    assert np.array_equal(fused, plain)
    assert np.abs(fused.astype(np.int16) - want).max() <= RGB8_MAX_LSB
    brick.close()


# ---- Marschner-Lobb field: high-frequency stress for trilinear + TF -------------

def _peak_tf(n: int = 256, centre: float = 0.5, width: float = 0.06):
    """An iso-surface-like TF: a narrow opacity peak around ``centre`` on a colour ramp."""
    from paper_2501_01628_b200.volume import TransferFunction1D

    x = np.linspace(0.0, 1.0, n)
    a = 0.35 * np.exp(-(((x - centre) / width) ** 2))
    t = np.column_stack([0.2 + 0.8 * x, 1.0 - 0.7 * x, 0.3 + 0.4 * np.sin(3 * x), a]).astype(np.float32)
    return TransferFunction1D(t, 0.0, 1.0)


def test_marschner_lobb_generation_bit_exact(cuda_device, oracle_lib):
    from paper_2501_01628_b200.volume import marschner_lobb_field

    for f in (marschner_lobb_field((41, 37, 33)), marschner_lobb_field((129, 129, 129), f_m=9.0, alpha=0.1)):
        hi = tuple(d - 1 for d in f.dims)
        for lo, hi_, g in [((0, 0, 0), hi, 0), ((5, 3, 7), (20, hi[1], 15), 1), ((0, 10, 0), (hi[0], 20, hi[2]), 2)]:
            desc = BrickDesc(f.dims, lo, hi_, g)
            b = dev.DeviceBrick(desc, cuda_device).generate(f)
            got = b.download()
            ref = oracle.generate_ml(f.dims, f.ml, desc.stored_lo, desc.stored_dims)
            assert np.array_equal(got, ref), f"{f.dims} brick {lo}-{hi_}"
            b.close()


@pytest.mark.parametrize("P", [1, 2, 4])
def test_marschner_lobb_frame_matches_oracle(cuda_device, oracle_lib, P):
    from paper_2501_01628_b200.volume import marschner_lobb_field

    f = marschner_lobb_field((65, 65, 65))
    vox = oracle.generate_ml(f.dims, f.ml)
    dec = decompose(f, P)
    W, H = 128, 112
    for cam, tf in [(auto_camera(f.bounds(), W, H), _peak_tf()),
                    (orbit_camera(f.bounds().center(), 110.0, 0.7, 0.4, 40.0, W / H), _peak_tf(centre=0.3)),
                    (auto_camera(f.bounds(), W, H), dense_tf())]:
        ref, rs = oracle_partials(vox, dec, cam, tf, 1.0, 0.99, W, H)
        parts, samples = _gpu_partials(dec, cam, tf, 1.0, 0.99, W, H, cuda_device)
        for r in range(P):
            assert np.array_equal(samples[r].view(H, W).cpu().numpy().astype(np.uint32), rs[r]), f"rank {r}"
            _check_rgba(parts[r].view(H, W, 4).cpu().numpy(), ref[r], f"ML P={P} rank {r}")
        order = dec.visibility_order(cam.position)
        img = oracle.composite(ref, order, (0.1, 0.1, 0.1))
        assert img.max() > 0.15, "the peak TF must make the field visible"


def test_stage_input_from_pinned_memory(cuda_device):
    """dprt_stage_input: SM-driven copy from mapped pinned memory (any size, byte tail), usage errors."""
    import ctypes

    from paper_2501_01628_b200 import _lib
    from paper_2501_01628_b200.errors import UsageError

    for n in (16, 4096, 4099, 65536 + 5):
        src = torch.randint(0, 256, (n,), dtype=torch.uint8).pin_memory()
        dst = torch.zeros(n + 16, dtype=torch.uint8, device=cuda_device)
        _lib.check(_lib.lib().dprt_stage_input(cuda_device.index or 0, ctypes.c_void_p(dst.data_ptr()),
                                               ctypes.c_void_p(src.data_ptr()), n, None), "stage")
        torch.cuda.synchronize()
        assert torch.equal(dst[:n].cpu(), src) and int(dst[n:].sum()) == 0
    plain = torch.zeros(64, dtype=torch.uint8)  # pageable: refused
    with pytest.raises(UsageError, match="page-locked"):
        _lib.check(_lib.lib().dprt_stage_input(0, ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(plain.data_ptr()),
                                               64, None), "stage")


def test_tf_update_through_pinned_staging_matches_oracle(cuda_device, oracle_lib):
    """DeviceTF.update(staging=pinned) (the e2e path) re-renders with the new table, frame after frame."""
    f = blob_field((40, 36, 32), seed=3)
    vox = oracle.generate_field(f.dims, f.blobs)
    dec = decompose(f, 1)
    W, H = 64, 56
    cam = auto_camera(f.bounds(), W, H)
    b = dev.DeviceBrick(dec.brick(0), cuda_device).generate(f)
    dtf = dev.DeviceTF(default_tf(), cuda_device)
    p = torch.empty(H * W * 4, dtype=torch.float32, device=cuda_device)
    for tf in (dense_tf(), default_tf(), dense_tf(64)):
        staging = torch.from_numpy(tf.as_f32().reshape(-1).copy()).pin_memory()
        dtf.update(tf, staging=staging)
        dev.march(b, cam, dtf, 1.0, 0.99, p, W, H)
        torch.cuda.synchronize()
        ref, _ = oracle_partials(vox, dec, cam, tf, 1.0, 0.99, W, H)
        _check_rgba(p.view(H, W, 4).cpu().numpy(), ref[0], f"staged TF n={tf.n}")
    b.close()


def test_render_stats_device_times_and_samples(cuda_device, oracle_lib):
    """RenderOptions(timing=True) / collect_samples fill RankStats' device timings and the owned sample
    total (the reference's per-rank counters, engine.py:177-193, extended for DVR)."""
    s = c1(P=1, W=96, H=80)
    vox = oracle.generate_field(s.field.dims, s.field.blobs)
    _, rs = oracle_partials(vox, s.dec, s.cam, s.tf, s.dt, s.ert, s.W, s.H)
    b = dev.DeviceBrick(s.dec.brick(0), cuda_device).generate(s.field)
    vr = VolumeRenderer(SoloEndpoint(cuda_device), b, s.dec, s.tf, s.background)
    for keep in (False, True):  # fused single-rank path and march + composite path
        res = vr.render(s.cam, s.W, s.H, RenderOptions(timing=True, collect_samples=True, keep_float=keep))
        t = res.stats.device_times()
        assert t["march_ms"] > 0 and t["composite_ms"] >= 0 and t["brick_GBps"] > 0
        assert res.stats.owned_samples() == int(rs[0].sum())
    from paper_2501_01628_b200.errors import UsageError

    with pytest.raises(UsageError, match="timing"):
        vr.render(s.cam, s.W, s.H, RenderOptions()).stats.device_times()
    b.close()


def test_fp16_fragments_march_and_composite(cuda_device, oracle_lib):
    """fp16 fragments: the march's fp16 partial is its f32 partial rounded to nearest (bit for bit), and
    the composite of fp16 fragments equals the f32 composite of the same rounded values (bit for bit)."""
    s = c1(P=2, W=101, H=77)
    dtf = dev.DeviceTF(s.tf, cuda_device)
    n = s.W * s.H
    f32, f16 = [], []
    for r in range(2):
        b = dev.DeviceBrick(s.dec.brick(r), cuda_device).generate(s.field)
        p32 = torch.empty(n * 4, dtype=torch.float32, device=cuda_device)
        p16 = torch.empty(n * 4, dtype=torch.float16, device=cuda_device)
        dev.march(b, s.cam, dtf, s.dt, s.ert, p32, s.W, s.H)
        dev.march(b, s.cam, dtf, s.dt, s.ert, p16, s.W, s.H)
        torch.cuda.synchronize()
        assert torch.equal(p16, p32.half())
        f32.append(p32)
        f16.append(p16)
        b.close()
    bg = (0.2, 0.1, 0.3)
    outs = []
    for frags in ([f.half().float() for f in f32], f16):
        rgb8 = torch.empty(n * 3, dtype=torch.uint8, device=cuda_device)
        rgba = torch.empty(n * 4, dtype=torch.float32, device=cuda_device)
        dev.composite(frags, bg, rgb8=rgb8, rgba=rgba)
        outs.append((rgb8, rgba))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    # ranged fp16 (odd offsets: 8-byte loads) == ranged f32 of the same values
    ranges = [(3, n - 5), (0, n)]
    r32 = [f32[0].half().float()[12: (n - 5) * 4], f32[1].half().float()]
    r16 = [f16[0][12: (n - 5) * 4], f16[1]]
    res = []
    for frags in (r32, r16):
        rgba = torch.empty(n * 4, dtype=torch.float32, device=cuda_device)
        dev.composite(frags, None, rgba=rgba, ranges=ranges, npix=n)
        res.append(rgba)
    assert torch.equal(res[0], res[1])


def test_fused_frame_writes_every_pixel(cuda_device, oracle_lib):
    """dprt_march_rgb8 owns the whole frame: pixels outside the footprint, beams that miss the brick and
    misses inside it all get the tone-mapped background (the buffer starts as garbage)."""
    s = c1(P=1, W=203, H=151)
    b = dev.DeviceBrick(s.dec.brick(0), cuda_device).generate(s.field)
    dtf = dev.DeviceTF(s.tf, cuda_device)
    n = s.W * s.H
    for cam in (s.cam, orbit_camera(s.field.bounds().center(), 300.0, 0.4, 0.2, 20.0, s.W / s.H)):
        guarded = torch.full((n * 3 + 256,), 0xAB, dtype=torch.uint8, device=cuda_device)
        frame = guarded[:n * 3]
        dev.march_rgb8(b, cam, dtf, s.dt, s.ert, s.background, frame, s.W, s.H)
        p = torch.empty(n * 4, dtype=torch.float32, device=cuda_device)
        dev.march(b, cam, dtf, s.dt, s.ert, p, s.W, s.H)
        ref = torch.empty(n * 3, dtype=torch.uint8, device=cuda_device)
        dev.composite([p], s.background, rgb8=ref)
        torch.cuda.synchronize()
        assert torch.equal(frame, ref)
        assert bool((guarded[n * 3:] == 0xAB).all()), "write past the frame"
    b.close()


def test_partial_writes_stay_in_bounds(cuda_device, oracle_lib):
    """Band-cleared, windowed and fp16 partial marches write only their buffers (sentinel guard after the
    end) and define every pixel they promise: the band rows (band clear) / the window rows."""
    s = c1(P=2, W=131, H=97)
    dtf = dev.DeviceTF(s.tf, cuda_device)
    n = s.W * s.H
    b = dev.DeviceBrick(s.dec.brick(1), cuda_device).generate(s.field)
    full = torch.empty(n * 4, dtype=torch.float32, device=cuda_device)
    dev.march(b, s.cam, dtf, s.dt, s.ert, full, s.W, s.H)
    rect = b.footprint(s.cam, s.W, s.H)
    cases = [("band", torch.float32, None), ("window", torch.float32, (20, 71)), ("half", torch.float16, None)]
    for name, dt, rows in cases:
        npx = n if rows is None else (rows[1] - rows[0]) * s.W
        guarded = torch.full((npx * 4 + 64,), 7.0, dtype=dt, device=cuda_device)
        buf = guarded[:npx * 4]
        dev.march(b, s.cam, dtf, s.dt, s.ert, buf, s.W, s.H, band_clear=name == "band", rows=rows)
        torch.cuda.synchronize()
        assert bool((guarded[npx * 4:] == 7.0).all()), f"{name}: write past the buffer"
        ref = full.view(s.H, s.W, 4)
        got = buf.view(-1, s.W, 4).float()
        if name == "band":
            assert torch.equal(got[rect[1]:rect[3]], ref[rect[1]:rect[3]])
        elif name == "window":
            assert torch.equal(got, ref[rows[0]:rows[1]])
        else:
            assert torch.equal(got, ref.half().float())
    b.close()


@pytest.mark.parametrize("half", [False, True])
def test_wide_quad_offsets_are_bit_identical(cuda_device, oracle_lib, half):
    """Bricks of >= 2^31 apron quads march with unsigned offsets from the apron base (kWide), bricks of
    >= 2^28 voxels with 6-sample batches at 2 CTAs/SM (deep); forced onto a small brick, every
    combination writes exactly the bytes of the default kernel (padded slots and ERT-masked slots add
    exact zeros whatever the batch length).  The same holds among the four fp16-quad kernels (``half``),
    including half+deep (the even config-3 bricks) and half+deep+wide (the mass-balanced ones)."""
    f = blob_field((70, 61, 53), seed=12)
    dec = decompose(f, 2)
    W, H = 150, 110
    cam = auto_camera(f.bounds(), W, H)
    dtf = dev.DeviceTF(dense_tf(), cuda_device)
    for r in range(2):
        b = dev.DeviceBrick(dec.brick(r), cuda_device, half_quads=half).generate(f)
        out = []
        for wide, deep in ((False, False), (True, False), (False, True), (True, True)):
            p = torch.empty(H * W * 4, dtype=torch.float32, device=cuda_device)
            s = torch.empty(H * W, dtype=torch.int32, device=cuda_device)
            dev.march(b, cam, dtf, 0.8, 0.97, p, W, H, samples=s, force_wide=wide, force_deep=deep)
            out.append((p, s))
        torch.cuda.synchronize()
        for p, s in out[1:]:
            assert torch.equal(out[0][0], p) and torch.equal(out[0][1], s)
        b.close()
