"""The reference's own golden vectors, checked on the GPU marcher's device functions (bit-exact):
camera rays from engine.gen_primary_batch (engine.py:224-251) and slab intervals from
geom.ray_aabb_intersect (geom.py:171-200), incl. zero-direction components, on-face origins and
empty boxes (tests/golden/make_golden.py)."""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np
import pytest

from paper_2501_01628_b200 import _lib
from paper_2501_01628_b200.device import camera_struct
from paper_2501_01628_b200.geom import CameraSpec

pytestmark = pytest.mark.gpu
GOLD = np.load(Path(__file__).parent / "golden" / "reference_vectors.npz")


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def test_gpu_primary_rays_match_reference(cuda_device):
    for i, p in enumerate(GOLD["cam_params"]):
        cam = CameraSpec(tuple(p[0:3]), tuple(p[3:6]), tuple(p[6:9]), float(p[9]), float(p[10]))
        w, h = int(p[11]), int(p[12])
        out = np.zeros((h * w, 3), np.float64)
        c = camera_struct(cam)
        _lib.check(_lib.lib().dprt_kat_primary_dirs(0, ctypes.byref(c), w, h, _p(out)), "kat")
        assert np.array_equal(out, GOLD[f"cam_dirs_{i}"]), f"camera {i}"


def test_gpu_slab_intervals_match_reference(cuda_device):
    o, d = np.ascontiguousarray(GOLD["slab_o"]), np.ascontiguousarray(GOLD["slab_d"])
    lo, hi = np.ascontiguousarray(GOLD["slab_lo"]), np.ascontiguousarray(GOLD["slab_hi"])
    n = len(o)
    t01 = np.zeros((n, 2), np.float64)
    hit = np.zeros(n, np.int32)
    _lib.check(_lib.lib().dprt_kat_slab(0, n, _p(o), _p(d), _p(lo), _p(hi), _p(t01), _p(hit)), "kat")
    assert np.array_equal(hit.astype(np.uint8), GOLD["slab_hit"])
    m = hit.astype(bool)
    assert np.array_equal(t01[m], GOLD["slab_t"][m])
