"""Pure-Python scalar restatement of the brick march (TEST INFRASTRUCTURE ONLY, small cases only).

A second, independent statement of DESIGN.md §2.4-2.7 written in the style of the reference's own
brute-force oracle (pkg/tests/util.py:95-148: per-pixel scalar loops over Python floats).  Python floats
are IEEE f64 with one rounding per operation, so on the same inputs this must agree with dvr_oracle.c
bit for bit; tests/test_oracle.py checks that, which pins the C oracle to a readable statement.
"""

from __future__ import annotations

import math
from typing import Tuple

import numpy as np


def primary_dir(cam, px: int, py: int, width: int, height: int):
    """pkg/src/dprt/geom.py:240-259, operation for operation."""
    f, r, u = cam[3:6], cam[6:9], cam[9:12]
    half_w, half_h = cam[12], cam[13]
    sx = ((px + 0.5) / width * 2.0 - 1.0) * half_w
    sy = (1.0 - (py + 0.5) / height * 2.0) * half_h
    d = (f[0] + sx * r[0] + sy * u[0], f[1] + sx * r[1] + sy * u[1], f[2] + sx * r[2] + sy * u[2])
    n = math.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
    return (d[0] / n, d[1] / n, d[2] / n)


def slab(o, d, lo, hi):
    """pkg/src/dprt/geom.py:171-200."""
    if lo[0] > hi[0] or lo[1] > hi[1] or lo[2] > hi[2]:
        return None
    t0, t1 = -math.inf, math.inf
    for i in range(3):
        if d[i] == 0.0:
            if o[i] < lo[i] or o[i] > hi[i]:
                return None
            continue
        inv = 1.0 / d[i]
        ta = (lo[i] - o[i]) * inv
        tb = (hi[i] - o[i]) * inv
        if ta > tb:
            ta, tb = tb, ta
        if ta > t0:
            t0 = ta
        if tb < t1:
            t1 = tb
        if t1 < t0:
            return None
    return (t0, t1)


def _lerp(a, b, f):
    return a + (b - a) * f


def march_pixel(vox: np.ndarray, brick, cam, px, py, width, height, tf: np.ndarray, vmin, vmax, dt,
                ert) -> Tuple[Tuple[float, float, float, float], int]:
    """One pixel of one brick; returns ((C_r, C_g, C_b, A), owned sample count)."""
    o = (float(cam[0]), float(cam[1]), float(cam[2]))
    d = primary_dir([float(c) for c in cam], px, py, width, height)
    lo_w, hi_w = brick.box_world()
    iv = slab(o, d, lo_w, hi_w)
    if iv is None:
        return (0.0, 0.0, 0.0, 0.0), 0
    t0, t1 = iv
    t0 = max(t0, 0.0)
    if t1 < t0:
        return (0.0, 0.0, 0.0, 0.0), 0
    k0 = math.ceil(t0 / dt)
    k1 = math.ceil(t1 / dt)
    n = max(k1 - k0, 0)
    s_lo = brick.stored_lo
    sd = brick.stored_dims
    clo = [max(s_lo[a], 0) for a in range(3)]
    chi = [min(s_lo[a] + sd[a] - 2, brick.dims[a] - 2) for a in range(3)]
    n_tf = tf.shape[0]
    tf_scale = (n_tf - 1) / (float(vmax) - float(vmin))
    C = [0.0, 0.0, 0.0]
    A = 0.0
    for k in range(k0, k0 + n):
        t = float(k) * dt
        u = [((o[a] + t * d[a]) - brick.origin[a]) / brick.spacing[a] for a in range(3)]
        c = []
        fr = []
        for a in range(3):
            ci = min(max(int(math.floor(u[a])), clo[a]), chi[a])
            f = min(max(u[a] - ci, 0.0), 1.0)
            c.append(ci - s_lo[a])
            fr.append(f)
        x, y, z = c

        def v(dx, dy, dz):
            return float(vox[z + dz, y + dy, x + dx])

        c00 = _lerp(v(0, 0, 0), v(1, 0, 0), fr[0])
        c10 = _lerp(v(0, 1, 0), v(1, 1, 0), fr[0])
        c01 = _lerp(v(0, 0, 1), v(1, 0, 1), fr[0])
        c11 = _lerp(v(0, 1, 1), v(1, 1, 1), fr[0])
        val = _lerp(_lerp(c00, c10, fr[1]), _lerp(c01, c11, fr[1]), fr[2])
        xq = min(max((val - vmin) * tf_scale, 0.0), float(n_tf - 1))
        i = min(int(math.floor(xq)), n_tf - 2)
        f = xq - i
        e = [_lerp(float(tf[i, ch]), float(tf[i + 1, ch]), f) for ch in range(4)]
        w = (1.0 - A) * e[3]
        C = [C[0] + w * e[0], C[1] + w * e[1], C[2] + w * e[2]]
        A = A + w
        if A >= ert:
            break
    return (C[0], C[1], C[2], A), n
