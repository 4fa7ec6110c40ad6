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
from scenes import RGBA_ATOL, cam_array, oracle_brick

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
