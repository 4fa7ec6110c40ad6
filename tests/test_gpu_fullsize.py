"""Parity at BASELINE's full sizes through size-independent properties (the oracle cannot march whole
frames of these volumes in test time):

* owned lattice sample counts, full frame, integer-exact against the oracle's ownership-only pass;
* partition invariance at full size: the 8 ranks' counts sum to the whole field's count per pixel;
* RGBA on a strided subset of rows against the oracle marching exactly those rows (RGBA_ATOL);
* the bench workload (config 2) and the heaviest / lightest config-3 bricks.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.geom import auto_camera
from paper_2501_01628_b200.volume import blob_field, decompose, default_tf
from scenes import RGBA_ATOL, cam_array, ert_edge_pixels, oracle_brick

pytestmark = pytest.mark.gpu


def _march(dec, r, cam, tf, W, H, device):
    b = dev.DeviceBrick(dec.brick(r), device).generate(dec.field)
    p = torch.empty(W * H * 4, dtype=torch.float32, device=device)
    s = torch.empty(W * H, dtype=torch.int32, device=device)
    dev.march(b, cam, dev.DeviceTF(tf, device), 1.0, 0.99, p, W, H, samples=s)
    torch.cuda.synchronize()
    return b, p.view(H, W, 4).cpu().numpy(), s.view(H, W).cpu().numpy().astype(np.uint32)


def _strided_rows_check(b, dec, r, cam, tf, W, H, got, stride):
    vox = b.download()
    ob = oracle_brick(dec, r)
    ref, _ = oracle.render_brick(vox, ob, cam_array(cam), tf.as_f32(), tf.vmin, tf.vmax, 1.0, 0.99, W, H,
                                 rows=(stride // 2, H, stride))
    rows = list(range(stride // 2, H, stride))
    err = np.abs(got[rows].astype(np.float64) - ref[rows])
    assert err.max() <= RGBA_ATOL, f"max |dRGBA| {err.max():.3e}"
    return err.max()


def test_config2_full_frame(cuda_device, oracle_lib):
    """BASELINE config 2 (the bench workload): 512^3 brick at 1920x1080."""
    W, H = 1920, 1080
    f = blob_field((513, 513, 513), seed=1)
    dec = decompose(f, 1)
    cam = auto_camera(f.bounds(), W, H)
    tf = default_tf()
    b, rgba, samples = _march(dec, 0, cam, tf, W, H, cuda_device)
    assert np.array_equal(samples, oracle.sample_counts(oracle_brick(dec, 0), cam_array(cam), 1.0, W, H))
    _strided_rows_check(b, dec, 0, cam, tf, W, H, rgba, 24)
    b.close()


@pytest.mark.parametrize("rank", [5, 6])
def test_config3_brick_full_frame(cuda_device, oracle_lib, rank):
    """One 1024^3 brick of BASELINE config 3 (2048^3 field, 8 bricks) at 3840x2160."""
    W, H = 3840, 2160
    f = blob_field((2049, 2049, 2049), seed=1)
    dec = decompose(f, 8)
    cam = auto_camera(f.bounds(), W, H)
    tf = default_tf()
    b, rgba, samples = _march(dec, rank, cam, tf, W, H, cuda_device)
    assert np.array_equal(samples, oracle.sample_counts(oracle_brick(dec, rank), cam_array(cam), 1.0, W, H))
    _strided_rows_check(b, dec, rank, cam, tf, W, H, rgba, 96)
    b.close()
    del b
    torch.cuda.empty_cache()


def test_config3_mass_balanced_wide_brick(cuda_device, oracle_lib):
    """Config 3's field split by non-empty voxel count (the GPU mass function): its largest brick holds
    more than 2^31 apron quads, so it marches with 64-bit quad offsets.  Full-frame ownership exact,
    strided rows within tolerance."""
    W, H = 3840, 2160
    f = blob_field((2049, 2049, 2049), seed=1)
    dec = decompose(f, 8, "mass", dev.field_mass_function(f, cuda_device, 0.1))
    torch.cuda.empty_cache()
    sizes = [np.prod([d + 2 for d in dec.brick(r).stored_dims]) for r in range(8)]
    r = int(np.argmax(sizes))
    assert sizes[r] >= 2 ** 31, "expected one brick beyond the 32-bit quad range"
    cam = auto_camera(f.bounds(), W, H)
    tf = default_tf()
    b, rgba, samples = _march(dec, r, cam, tf, W, H, cuda_device)
    assert np.array_equal(samples, oracle.sample_counts(oracle_brick(dec, r), cam_array(cam), 1.0, W, H))
    _strided_rows_check(b, dec, r, cam, tf, W, H, rgba, 96)
    b.close()
    del b
    torch.cuda.empty_cache()


@pytest.mark.parametrize("strategy", ["even", "mass"])
def test_config3_composited_frame_on_pixel_lattice(cuda_device, oracle_lib, strategy):
    """BASELINE config 3 as a whole frame: all 8 bricks of the 2048^3 field marched on this GPU (rank by
    rank), their partials over-composited in visibility order and tone mapped by the compositor kernel;
    against the oracle's 8 bricks (its own host generator) on the strided 1/64 pixel lattice (every 8th
    pixel in x and y): per-brick RGBA within RGBA_ATOL, composited RGB8 within 1 LSB (ERT-edge pixels as
    in the other parity tests), visibility order equal to the oracle's kd order."""
    W, H, S = 3840, 2160, 8
    f = blob_field((2049, 2049, 2049), seed=1)
    mass = dev.field_mass_function(f, cuda_device, 0.1) if strategy == "mass" else None
    dec = decompose(f, 8, strategy, mass)
    torch.cuda.empty_cache()
    cam = auto_camera(f.bounds(), W, H)
    tf = default_tf()
    dtf = dev.DeviceTF(tf, cuda_device)
    order = dec.visibility_order(cam.position)
    parts, lat = [], []
    for r in range(8):
        b = dev.DeviceBrick(dec.brick(r), cuda_device).generate(f)
        p = torch.empty(W * H * 4, dtype=torch.float32, device=cuda_device)
        dev.march(b, cam, dtf, 1.0, 0.99, p, W, H)
        torch.cuda.synchronize()
        b.close()
        del b
        torch.cuda.empty_cache()
        parts.append(p)
        lat.append(p.view(H, W, 4)[::S, ::S].double().cpu().numpy())
    rgb8 = torch.empty(W * H * 3, dtype=torch.uint8, device=cuda_device)
    dev.composite([parts[r] for r in order], (0.05, 0.06, 0.08), rgb8=rgb8)
    got8 = rgb8.view(H, W, 3)[::S, ::S].cpu().numpy().astype(np.int16)
    del parts
    torch.cuda.empty_cache()
    ca = cam_array(cam)
    refs, edge = [], np.zeros(lat[0].shape[:2], bool)
    for r in range(8):
        ob = oracle_brick(dec, r)
        vox = oracle.generate_field(f.dims, f.blobs, ob.stored_lo, ob.stored_dims, fast=True)
        ref = oracle.render_lattice(vox, ob, ca, tf.as_f32(), tf.vmin, tf.vmax, 1.0, 0.99, W, H, S, S)
        del vox
        e = ert_edge_pixels(lat[r][..., 3], ref[..., 3], 0.99)
        edge |= e
        err = np.abs(lat[r] - ref)[~e]
        assert err.max() <= RGBA_ATOL, f"brick {r}: max |dRGBA| {err.max():.3e}"
        refs.append(ref)
    want8 = oracle.tone_map_rgb8(oracle.composite(refs, order, (0.05, 0.06, 0.08))).astype(np.int16)
    d8 = np.abs(got8 - want8).max(axis=-1)
    assert d8[~edge].max() <= 1, f"composited RGB8 differs by {d8[~edge].max()} LSB"
    nodes = oracle.kd_leaves(f.dims, f.spacing, 8, strategy, field=None)[1] if strategy == "even" else None
    if nodes is not None:
        assert order == oracle.kd_order(nodes, 8, cam.position, f.origin, f.spacing)
