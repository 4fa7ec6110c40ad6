"""Brick ownership and visibility order: product vs the oracle's independent restatement, exactly."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2501_01628_b200.errors import UsageError
from paper_2501_01628_b200.geom import CameraSpec
from paper_2501_01628_b200.volume import (BrickDesc, TransferFunction1D, blob_field, blob_mixture, decompose,
                                          default_tf, visibility_order)
from scenes import cam_array


@pytest.mark.parametrize("dims,spacing,P", [((64, 64, 64), (1, 1, 1), 2), ((64, 64, 64), (1, 1, 1), 8),
                                            ((101, 37, 55), (1, 1, 1), 5), ((1537, 769, 385), (1, 1, 2), 8),
                                            ((2049, 2049, 2049), (1, 1, 1), 8), ((40, 40, 9), (0.5, 0.5, 3.0), 7)])
def test_even_decomposition_matches_oracle_and_tiles_the_grid(dims, spacing, P):
    f = blob_field(dims, spacing=spacing)
    dec = decompose(f, P)
    leaves, _ = oracle.kd_leaves(dims, spacing, P)
    assert [tuple(map(tuple, l)) for l in leaves] == dec.boxes
    cells = np.prod([d - 1 for d in dims])
    assert sum(np.prod([hi[a] - lo[a] for a in range(3)]) for lo, hi in dec.boxes) == cells
    # disjoint: no two boxes overlap
    for i in range(P):
        for j in range(i + 1, P):
            (a0, a1), (b0, b1) = dec.boxes[i], dec.boxes[j]
            assert any(a1[k] <= b0[k] or b1[k] <= a0[k] for k in range(3))


def test_c3_bricks_are_1024_cubed():
    dec = decompose(blob_field((2049, 2049, 2049)), 8)
    for lo, hi in dec.boxes:
        assert tuple(h - l for l, h in zip(lo, hi)) == (1024, 1024, 1024)


def test_mass_decomposition_matches_oracle_and_is_uneven():
    f = blob_field((96, 48, 40), seed=3, spacing=(1.0, 1.0, 2.0), lopsided=True)
    vox = oracle.generate_field(f.dims, f.blobs)

    def mass(axis, lo, hi):
        sub = vox[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] >= np.float32(0.1)
        return sub.sum(axis=tuple(a for a in range(3) if a != 2 - axis)).astype(np.int64)

    dec = decompose(f, 8, "mass", mass)
    leaves, _ = oracle.kd_leaves(f.dims, f.spacing, 8, "mass", field=vox)
    assert [tuple(map(tuple, l)) for l in leaves] == dec.boxes
    sizes = {np.prod([hi[a] - lo[a] for a in range(3)]) for lo, hi in dec.boxes}
    assert len(sizes) > 1  # uneven bricks (config 4)


def test_visibility_order_matches_oracle_for_random_eyes():
    rng = np.random.default_rng(1)
    for P in (2, 3, 5, 8):
        f = blob_field((70, 50, 30), spacing=(1.0, 1.0, 2.0))
        dec = decompose(f, P)
        _, nodes = oracle.kd_leaves(f.dims, f.spacing, P)
        for _ in range(50):
            eye = tuple(rng.uniform(-100, 200, 3))
            assert visibility_order(dec, eye) == oracle.kd_order(nodes, P, eye, f.origin, f.spacing)


def test_visibility_order_is_front_to_back_for_every_ray():
    """Per pixel, the bricks a ray enters appear in the kd order sorted by entry distance."""
    f = blob_field((41, 33, 29))
    dec = decompose(f, 6)
    W = H = 24
    rng = np.random.default_rng(2)
    for _ in range(6):
        eye = tuple(rng.uniform(-40, 80, 3))
        center = f.bounds().center()
        cam = CameraSpec(eye, tuple(np.subtract(center, eye)), (0.0, 1.0, 0.0) if abs(eye[1] - center[1]) < 30 else (1, 0, 0),
                         70.0, 1.0)
        order = dec.visibility_order(cam.position)
        dirs = oracle.primary_dirs(cam_array(cam), W, H)
        for d in dirs.reshape(-1, 3):
            enter = []
            for r in order:
                b = dec.brick(r).box_world()
                iv = oracle.slab(cam.position, d, b.lo, b.hi)
                if iv is not None and iv[1] >= max(iv[0], 0.0):
                    enter.append(max(iv[0], 0.0))
            assert enter == sorted(enter)


def test_brick_descriptor_ghost_and_storage():
    b = BrickDesc((65, 65, 65), (0, 0, 32), (32, 64, 64), ghost=1)
    assert b.stored_lo == (0, 0, 31)
    assert b.stored_dims == (34, 65, 34)
    assert b.stored_bytes == 4 * 34 * 65 * 34
    with pytest.raises(UsageError):
        BrickDesc((10, 10, 10), (0, 0, 0), (10, 9, 9))


def test_blob_mixture_is_seeded_and_bounded():
    a = blob_mixture(7, 16)
    assert np.array_equal(a, blob_mixture(7, 16))
    assert not np.array_equal(a, blob_mixture(8, 16))
    assert a.shape == (16, 5) and a[:, 4].max() == 1.0
    vox = oracle.generate_field((20, 20, 20), a)
    assert 0.0 <= vox.min() and vox.max() <= 1.0


def test_default_tf_shape():
    tf = default_tf()
    t = tf.as_f32()
    assert t.shape == (256, 4)
    x = np.arange(256) / 255
    assert np.all(t[x < 0.1, 3] == 0) and abs(t[-1, 3] - 0.05) < 1e-7
    with pytest.raises(UsageError):
        TransferFunction1D(np.zeros((1, 4), np.float32))


def test_centre_out_tile_order_is_a_permutation():
    """The marcher's tile-queue order (march.cu center_out: m, m-1, m+1, m-2, ... with m = n / 2) visits
    every row index exactly once and ends at the edges -- restated here for the CPU suite."""
    def center_out(k, n):
        m, d = n >> 1, (k + 1) >> 1
        return m - d if k & 1 else m + d

    for n in range(1, 70):
        seq = [center_out(k, n) for k in range(n)]
        assert sorted(seq) == list(range(n))
        assert seq[0] == n // 2 and set(seq[-2:]) <= {0, n - 1} | ({n - 2, 1} if n < 4 else set())
