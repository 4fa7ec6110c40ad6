"""Seeded randomized parity sweep: the GPU path against the CPU oracle on random fields, decompositions,
cameras (outside, grazing, inside the volume), transfer functions, step sizes and frame sizes.

Per case: every brick's per-pixel owned sample counts are integer-exact, every RGBA partial is within
RGBA_ATOL of the oracle's, the visibility order equals the oracle's independent kd order, and the
composited RGB8 frame is within RGB8_MAX_LSB; single-brick cases also check the fused
single-rank frame byte for byte against march + composite, and brick 0 of every case is re-marched with the
large-brick kernel configurations (wide addressing, deep batches), which must write identical bytes.  Sizes stay small so the oracle finishes
each case in well under a second.
"""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch

import oracle
from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.geom import CameraSpec, orbit_camera
from paper_2501_01628_b200.volume import TransferFunction1D, blob_field, decompose
from scenes import RGB8_MAX_LSB, RGBA_ATOL, RGBA_MEAN_ATOL, ert_edge_pixels, oracle_order, oracle_partials

pytestmark = pytest.mark.gpu

N_CASES = int(os.environ.get("DPRT_FUZZ_CASES", "64"))  # the committed sweep; a stress run sets more


def _random_tf(rng) -> TransferFunction1D:
    n = int(rng.choice([2, 3, 17, 64, 256, 1024]))
    x = np.linspace(0.0, 1.0, n)
    thr = rng.uniform(0.0, 0.6)
    ramp = np.clip((x - thr) / max(1e-9, 1 - thr), 0.0, None) ** rng.uniform(0.5, 2.0)
    a = np.where(x < thr, 0.0, rng.uniform(0.01, 0.35) * ramp)
    if rng.random() < 0.3:  # a narrow opacity spike
        c = rng.uniform(0.2, 0.9)
        a = np.maximum(a, 0.6 * np.exp(-((x - c) / 0.03) ** 2))
    # colour: a piecewise-linear ramp through 2..5 random stops (smooth, like an editor's TF; a table of
    # independent random entries would make the f32-vs-f64 comparison ill-conditioned, not the code wrong)
    k = int(rng.integers(2, 6))
    stops = rng.uniform(0.0, 1.0, size=(k, 3))
    rgb = np.column_stack([np.interp(x, np.linspace(0, 1, k), stops[:, c]) for c in range(3)])
    t = np.column_stack([rgb, np.clip(a, 0.0, 1.0)]).astype(np.float32)
    vmin = float(rng.uniform(-0.2, 0.1))
    return TransferFunction1D(t, vmin, float(vmin + rng.uniform(0.6, 1.3)))


def _random_case(seed: int):
    rng = np.random.default_rng(1000 + seed)
    dims = tuple(int(v) for v in rng.integers(17, 66, size=3))
    spacing = tuple(float(v) for v in rng.choice([0.5, 1.0, 1.5, 2.0], size=3))
    origin = tuple(float(v) for v in rng.uniform(-20, 20, size=3))
    f = blob_field(dims, seed=int(rng.integers(1, 1 << 30)), n_blobs=int(rng.integers(1, 17)), spacing=spacing,
                   origin=origin, lopsided=bool(rng.random() < 0.5))
    P = int(rng.choice([1, 2, 3, 4, 5, 8]))
    dec = decompose(f, P)
    W, H = int(rng.integers(16, 97)), int(rng.integers(16, 97))
    b = f.bounds()
    centre = b.center()
    radius = 0.5 * b.diagonal()
    kind = rng.random()
    if kind < 0.15:  # eye inside the volume
        eye = tuple(float(centre[a] + rng.uniform(-0.3, 0.3) * (b.hi[a] - b.lo[a])) for a in range(3))
        d = rng.normal(size=3)
        cam = CameraSpec(eye, tuple(float(v) for v in d / np.linalg.norm(d)), (0.0, 1.0, 0.0),
                         float(rng.uniform(30, 90)), W / H)
    else:
        cam = orbit_camera(centre, radius * rng.uniform(1.2, 4.0), rng.uniform(0, 2 * np.pi),
                           rng.uniform(-1.2, 1.2), float(rng.uniform(20, 70)), W / H)
    tf = _random_tf(rng)
    dt = float(rng.uniform(0.3, 1.5) * min(spacing))
    ert = float(rng.choice([0.9, 0.95, 0.99, 1.0]))
    bg = tuple(float(v) for v in rng.uniform(0, 1, size=3))
    return f, dec, cam, tf, dt, ert, W, H, bg


@pytest.mark.parametrize("seed", range(N_CASES))
def test_random_scene_matches_oracle(cuda_device, oracle_lib, seed):
    f, dec, cam, tf, dt, ert, W, H, bg = _random_case(seed)
    vox = oracle.generate_field(f.dims, f.blobs)
    ref, ref_s = oracle_partials(vox, dec, cam, tf, dt, ert, W, H)
    dtf = dev.DeviceTF(tf, cuda_device)
    parts = []
    ert_edge = np.zeros((H, W), bool)
    for r in range(dec.P):
        b = dev.DeviceBrick(dec.brick(r), cuda_device).generate(f)
        p = torch.empty(H * W * 4, dtype=torch.float32, device=cuda_device)
        s = torch.empty(H * W, dtype=torch.int32, device=cuda_device)
        dev.march(b, cam, dtf, dt, ert, p, W, H, samples=s)
        if r == 0:  # the large-brick configurations write the same bytes
            for wide, deep in ((True, False), (False, True)):
                p2 = torch.empty_like(p)
                dev.march(b, cam, dtf, dt, ert, p2, W, H, force_wide=wide, force_deep=deep)
                torch.cuda.synchronize()
                assert torch.equal(p, p2), f"case {seed}: wide={wide} deep={deep} kernel differs"
        torch.cuda.synchronize()
        b.close()
        got_s = s.view(H, W).cpu().numpy().astype(np.uint32)
        assert np.array_equal(got_s, ref_s[r]), f"case {seed}: brick {r} owned sample counts differ"
        got = p.view(H, W, 4).cpu().numpy().astype(np.float64)
        err = np.abs(got - ref[r])
        assert err.mean() <= RGBA_MEAN_ATOL, f"case {seed}: brick {r} mean |dRGBA| {err.mean():.3e}"
        # early ray termination is a threshold: where one side's opacity reaches ert within rounding and the
        # other's stops a hair below, the latter takes one more sample, worth <= (1 - ert) * alpha_max
        # (DESIGN.md §3.3); every other pixel is held to RGBA_ATOL
        edge = ert_edge_pixels(got[..., 3], ref[r][..., 3], ert)
        bad = (err.max(axis=2) > RGBA_ATOL) & ~edge
        assert not bad.any(), f"case {seed}: brick {r} max |dRGBA| {err.max(axis=2)[bad].max():.3e} off the ERT edge"
        amax = float(tf.as_f32()[:, 3].max())
        assert err.max() <= RGBA_ATOL + (1.0 - ert) * amax + 1e-6, f"case {seed}: brick {r} ERT-edge error"
        ert_edge |= edge
        parts.append(p)
    order = dec.visibility_order(cam.position)
    assert order == oracle_order(dec, cam.position), f"case {seed}: visibility order"
    rgb8 = torch.empty(H * W * 3, dtype=torch.uint8, device=cuda_device)
    dev.composite([parts[r] for r in order], bg, rgb8=rgb8)
    want = oracle.tone_map_rgb8(oracle.composite(ref, order, bg)).astype(np.int16)
    diff = np.abs(rgb8.view(H, W, 3).cpu().numpy().astype(np.int16) - want).max(axis=2)
    assert diff[~ert_edge].max(initial=0) <= RGB8_MAX_LSB, f"case {seed}: RGB8 differs by {diff.max()} LSB"
    if dec.P == 1:  # the fused single-rank frame (march + over-background + tone map) gives the same bytes
        b = dev.DeviceBrick(dec.brick(0), cuda_device).generate(f)
        fused = torch.empty(H * W * 3, dtype=torch.uint8, device=cuda_device)
        dev.march_rgb8(b, cam, dtf, dt, ert, bg, fused, W, H)
        torch.cuda.synchronize()
        b.close()
        assert torch.equal(fused, rgb8), f"case {seed}: fused single-rank frame differs from march + composite"


MODES = ["direct_send", "binary_swap", "p2p", "cycle"]


@pytest.mark.parametrize("seed", range(int(os.environ.get("DPRT_FUZZ_MULTIRANK_CASES", "16"))))
def test_random_multirank_frame_matches_oracle(cuda_device, oracle_lib, seed):
    """R rank threads on one GPU through the real exchange schedules (transport.run_collective): the RGB8
    frame at rank 0 within 1 LSB of the oracle's sort-last composite (ray cycling: of its own oracle
    restatement, oracle.cycle_frame), and every rank's sample ownership exact."""
    from paper_2501_01628_b200.compositor import assign_rows
    from paper_2501_01628_b200.engine import RenderOptions, VolumeRenderer
    from paper_2501_01628_b200.transport import run_collective
    from scenes import cam_array, oracle_brick

    rng = np.random.default_rng(5000 + seed)
    mode = MODES[seed % len(MODES)]
    R = int(rng.choice([2, 4, 8])) if mode == "binary_swap" else int(rng.integers(2, 9))
    f, _, cam, tf, dt, ert, W, H, bg = _random_case(seed + 100)
    dec = decompose(f, R)
    vox = oracle.generate_field(f.dims, f.blobs)
    ref, ref_s = oracle_partials(vox, dec, cam, tf, dt, ert, W, H)
    order = dec.visibility_order(cam.position)
    if mode == "cycle":
        obs = [oracle_brick(dec, r) for r in range(R)]
        img = oracle.cycle_frame([ob.extract(vox) for ob in obs], obs, order, assign_rows(H, R), cam_array(cam),
                                 tf.as_f32(), tf.vmin, tf.vmax, dt, ert, W, H, bg)
    else:
        img = oracle.composite(ref, order, bg)
    want = oracle.tone_map_rgb8(img).astype(np.int16)

    def body(ep):
        b = dev.DeviceBrick(dec.brick(ep.rank), cuda_device).generate(f)
        vr = VolumeRenderer(ep, b, dec, tf, bg)
        res = vr.render(cam, W, H, RenderOptions(composite=mode, dt=dt, ert=ert, collect_samples=True))
        torch.cuda.synchronize()
        out = (res.samples.cpu().numpy().astype(np.uint32), None if res.rgb8 is None else res.rgb8.cpu().numpy())
        b.close()
        return out

    results = run_collective(R, body, device=cuda_device)
    for r in range(R):
        assert np.array_equal(results[r][0], ref_s[r]), f"case {seed} ({mode}, R={R}): rank {r} ownership"
    diff = np.abs(results[0][1].astype(np.int16) - want)
    assert diff.max() <= RGB8_MAX_LSB, f"case {seed} ({mode}, R={R}): RGB8 differs by {diff.max()} LSB"


def half_quad_bound(tf) -> float:
    """Stated per-pixel RGBA bound of the opt-in fp16 quads: each coefficient of the face
    value a + B fx + C fy + D fx fy rounds once to fp16 (relative 2^-11), so for field values in [0, 1] the
    sampled value moves by <= 5 * 2^-11; through the TF's steepest channel slope L that moves a sample's
    colour / opacity by <= 5 * 2^-11 * L, and the front-to-back weights sum to <= 1."""
    t = tf.as_f32().astype(np.float64)
    slope = np.abs(np.diff(t, axis=0)).max() * (tf.n - 1) / (tf.vmax - tf.vmin)
    return RGBA_ATOL + 5 * 2.0 ** -11 * slope


@pytest.mark.parametrize("seed", range(16))
def test_half_quads_within_stated_bound(cuda_device, oracle_lib, seed):
    """Opt-in fp16 coefficient quads (DPRT_BRICK_HALF_QUADS): ownership still exact (the ray setup is f64),
    RGBA within half_quad_bound of the oracle (ERT-edge pixels as in the f32 sweep)."""
    f, dec, cam, tf, dt, ert, W, H, bg = _random_case(seed)
    vox = oracle.generate_field(f.dims, f.blobs)
    ref, ref_s = oracle_partials(vox, dec, cam, tf, dt, ert, W, H)
    dtf = dev.DeviceTF(tf, cuda_device)
    bound = half_quad_bound(tf)
    amax = float(tf.as_f32()[:, 3].max())
    for r in range(dec.P):
        b = dev.DeviceBrick(dec.brick(r), cuda_device, half_quads=True).generate(f)
        p = torch.empty(H * W * 4, dtype=torch.float32, device=cuda_device)
        s = torch.empty(H * W, dtype=torch.int32, device=cuda_device)
        dev.march(b, cam, dtf, dt, ert, p, W, H, samples=s)
        torch.cuda.synchronize()
        b.close()
        assert np.array_equal(s.view(H, W).cpu().numpy().astype(np.uint32), ref_s[r])
        got = p.view(H, W, 4).cpu().numpy().astype(np.float64)
        err = np.abs(got - ref[r]).max(axis=2)
        edge = ert_edge_pixels(got[..., 3], ref[r][..., 3], ert, eps=5 * 2.0 ** -11 * amax * 4)
        assert err[~edge].max(initial=0) <= bound, f"case {seed}: brick {r} {err.max():.3e} > {bound:.3e}"
        assert err.max() <= bound + (1.0 - ert) * amax
