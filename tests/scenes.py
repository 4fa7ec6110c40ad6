"""Shared test scenarios: the SURVEY §8(d) configurations at oracle-friendly sizes, and helpers that
run the CPU oracle on exactly the decomposition the GPU path uses."""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

import oracle
from paper_2501_01628_b200.geom import CameraSpec, auto_camera
from paper_2501_01628_b200.volume import (Decomposition, FieldSpec, TransferFunction1D, blob_field, decompose,
                                          default_tf)

# Per-pixel RGBA tolerance of the f32 GPU marcher against the f64 oracle.  Sources:
# f32 sample positions (<= ~2e-4 voxel), f32 trilinear/TF/blend rounding over <= ~2k samples, and a
# possibly different ERT stopping sample (<= (1 - ert) * alpha_max).  Measured maxima are far below.
RGBA_ATOL = 2e-3
RGBA_MEAN_ATOL = 5e-5
RGB8_MAX_LSB = 1
RGBA_ATOL_F16 = 4e-3  # fp16 fragments: <= P * 2^-11 per channel before blending (P <= 8)


def ert_edge_pixels(a_gpu: np.ndarray, a_ref: np.ndarray, ert: float, eps: float = 1e-5) -> np.ndarray:
    """Pixels where early ray termination can legitimately differ between the f32 GPU path and the f64
    oracle: one side's accumulated opacity reached ``ert`` (within rounding) at a sample where the other's
    stayed a hair below it, so the latter takes (at most) one more sample.  Elsewhere both stop -- or run
    out -- at the same sample and the strict RGBA_ATOL applies."""
    if ert >= 1.0:
        return np.zeros(a_gpu.shape, bool)
    # the side that stopped first ends within rounding of the threshold; the other may hold one more sample
    return np.abs(np.minimum(a_gpu, a_ref) - ert) <= eps


def cam_array(cam: CameraSpec) -> np.ndarray:
    return oracle.camera_array(cam.position, cam.view_dir, cam.up, cam.fov_y, cam.aspect)


def oracle_brick(dec: Decomposition, rank: int, ghost: int = 1) -> oracle.OracleBrick:
    lo, hi = dec.boxes[rank]
    f = dec.field
    return oracle.OracleBrick(tuple(f.dims), tuple(lo), tuple(hi), ghost, tuple(f.origin), tuple(f.spacing))


def oracle_partials(field_vox: np.ndarray, dec: Decomposition, cam: CameraSpec, tf: TransferFunction1D,
                    dt: float, ert: float, W: int, H: int, ghost: int = 1, rows=None):
    """Every rank's f64 partial and sample counts, rendered by the C oracle."""
    parts, samples = [], []
    ca = cam_array(cam)
    for r in range(dec.P):
        ob = oracle_brick(dec, r, ghost)
        rgba, s = oracle.render_brick(ob.extract(field_vox), ob, ca, tf.as_f32(), tf.vmin, tf.vmax, dt, ert, W, H,
                                      rows=rows)
        parts.append(rgba)
        samples.append(s)
    return parts, samples


def oracle_order(dec: Decomposition, eye) -> List[int]:
    f = dec.field
    _, nodes = oracle.kd_leaves(f.dims, f.spacing, dec.P, dec.strategy,
                                field=None if dec.strategy == "even" else _FIELD_CACHE.get(id(f)))
    return oracle.kd_order(nodes, dec.P, eye, f.origin, f.spacing)


_FIELD_CACHE = {}


@dataclass
class Scenario:
    field: FieldSpec
    dec: Decomposition
    cam: CameraSpec
    tf: TransferFunction1D
    W: int
    H: int
    dt: float = 1.0
    ert: float = 0.99
    background: Tuple[float, float, float] = (0.05, 0.06, 0.08)


def c1(P: int = 2, W: int = 256, H: int = 256) -> Scenario:
    """SURVEY config 1: 64^3 blob field split in 2 along x (the longest-axis tie goes to x), 256^2."""
    f = blob_field((64, 64, 64), seed=1, n_blobs=16)
    dec = decompose(f, P)
    cam = auto_camera(f.bounds(), W, H)
    return Scenario(f, dec, cam, default_tf(), W, H)


def dense_tf(n: int = 256) -> TransferFunction1D:
    """A TF with strong opacity so ERT triggers often (exercises the termination path)."""
    x = np.arange(n) / (n - 1)
    a = np.where(x < 0.05, 0.0, np.minimum(1.0, 0.4 * (x - 0.05) / 0.95 + 0.02))
    rgb = np.column_stack([x, 1 - x, 0.5 + 0.5 * np.sin(6 * x)])
    return TransferFunction1D(np.column_stack([rgb, a]).astype(np.float32), 0.0, 1.0)
