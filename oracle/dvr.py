"""ctypes binding of oracle/dvr_oracle.c plus the oracle's numpy/Python pieces (TEST INFRASTRUCTURE ONLY).

Every function cites the reference code it restates (``pkg/src/dprt/...`` under the reference root) or
the DESIGN.md section that fixes semantics the reference does not have.
"""

from __future__ import annotations

import ctypes
import math
import os
import shutil
import subprocess
from dataclasses import dataclass
from pathlib import Path
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libdvr_oracle.so"
_ABI = 7

_lib = None


def build_oracle(force: bool = False) -> Path:
    """Compile dvr_oracle.c with strict IEEE f64 (no contraction).  Uses the PATH gcc, not $CC."""
    src = HERE / "dvr_oracle.c"
    if LIB_PATH.exists() and not force and LIB_PATH.stat().st_mtime >= src.stat().st_mtime:
        return LIB_PATH
    LIB_PATH.parent.mkdir(parents=True, exist_ok=True)
    cc = os.environ.get("ORACLE_CC") or shutil.which("gcc") or "cc"
    base = [cc, "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-std=c11", "-shared",
            "-o", str(LIB_PATH), str(src), "-lm"]
    try:
        subprocess.run(base[:1] + ["-fopenmp"] + base[1:], check=True, capture_output=True)
    except subprocess.CalledProcessError:
        subprocess.run(base, check=True, capture_output=True)  # single-threaded oracle
    return LIB_PATH


def load_oracle():
    global _lib
    if _lib is not None:
        return _lib
    if (HERE / "dvr_oracle.c").exists():
        build_oracle()  # rebuilds when the source is newer (before the first dlopen of this path)
    lib = ctypes.CDLL(str(LIB_PATH))
    if lib.dvr_oracle_version() != _ABI:
        raise RuntimeError(f"{LIB_PATH} has oracle ABI {lib.dvr_oracle_version()}, expected {_ABI}: rebuild it")
    P = ctypes.c_void_p
    lib.dvr_oracle_primary_dirs.argtypes = [P, ctypes.c_int, ctypes.c_int, P]
    lib.dvr_oracle_slab.argtypes = [P, P, P, P, P]
    lib.dvr_oracle_slab.restype = ctypes.c_int
    lib.dvr_oracle_lattice.argtypes = [P, P, P, P, ctypes.c_double, P]
    lib.dvr_oracle_lattice.restype = ctypes.c_int64
    lib.dvr_oracle_generate.argtypes = [P, P, P, ctypes.c_int, P, P, ctypes.c_int]
    lib.dvr_oracle_generate_fast.argtypes = [P, P, P, ctypes.c_int, P, P, ctypes.c_int]
    lib.dvr_oracle_render_lattice.argtypes = [
        P, P, P, P, P, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
        ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
        ctypes.c_int, P, ctypes.c_int]
    lib.dvr_oracle_render_lattice.restype = ctypes.c_int
    lib.dvr_oracle_generate_ml.argtypes = [P, P, P, P, P, ctypes.c_int]
    lib.dvr_oracle_det_cos.argtypes = [ctypes.c_double]
    lib.dvr_oracle_det_cos.restype = ctypes.c_double
    lib.dvr_oracle_render_brick.argtypes = [
        P, P, P, P, P, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
        ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P,
        ctypes.c_int]
    lib.dvr_oracle_render_brick.restype = ctypes.c_int
    lib.dvr_oracle_render_brick_accum.argtypes = [
        P, P, P, P, P, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
        ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, ctypes.c_int]
    lib.dvr_oracle_render_brick_accum.restype = ctypes.c_int
    lib.dvr_oracle_max_threads.restype = ctypes.c_int
    lib.dvr_oracle_sample_counts.argtypes = [P, P, P, ctypes.c_double, ctypes.c_int, ctypes.c_int, P, ctypes.c_int]
    _lib = lib
    return lib


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    assert a.flags["C_CONTIGUOUS"]
    return ctypes.c_void_p(a.ctypes.data)


def max_threads() -> int:
    return int(load_oracle().dvr_oracle_max_threads())


# ---------------------------------------------------------------------------------------------
# camera: pkg/src/dprt/geom.py:147-168 (CameraSpec.basis) and :240-259 (camera_primary_ray)

def _normalize(v):
    n = math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])  # geom.py:47-48
    if n == 0.0 or not math.isfinite(n):
        raise ValueError(f"cannot normalize degenerate vector {v!r}")
    return (v[0] / n, v[1] / n, v[2] / n)  # geom.py:51-55


def _cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def camera_array(position, view_dir, up, fov_y: float, aspect: float) -> np.ndarray:
    """14 f64: pos, forward, right, up, half_w, half_h -- geom.py:163-168 and :249-251 verbatim."""
    forward = _normalize(tuple(float(c) for c in view_dir))
    right = _normalize(_cross(forward, tuple(float(c) for c in up)))
    cam_up = _cross(right, forward)
    half_h = math.tan(math.radians(fov_y) * 0.5)
    half_w = half_h * aspect
    return np.array([*map(float, position), *forward, *right, *cam_up, half_w, half_h], np.float64)


def primary_dirs(cam: np.ndarray, width: int, height: int) -> np.ndarray:
    """(H, W, 3) unit directions, row-major pixels (engine.py:224-251 order)."""
    out = np.empty((height, width, 3), np.float64)
    load_oracle().dvr_oracle_primary_dirs(_ptr(np.ascontiguousarray(cam, np.float64)), width, height, _ptr(out))
    return out


def slab(origin, direction, lo, hi) -> Optional[Tuple[float, float]]:
    """geom.py:171-200 restated in C; None on a miss."""
    o = np.asarray(origin, np.float64)
    d = np.asarray(direction, np.float64)
    lo_ = np.asarray(lo, np.float64)
    hi_ = np.asarray(hi, np.float64)
    t = np.zeros(2, np.float64)
    hit = load_oracle().dvr_oracle_slab(_ptr(o), _ptr(d), _ptr(lo_), _ptr(hi_), _ptr(t))
    return (float(t[0]), float(t[1])) if hit else None


def lattice(origin, direction, lo, hi, dt: float) -> Tuple[int, int]:
    """(k0, n): owned lattice samples k0 .. k0+n-1."""
    o = np.asarray(origin, np.float64)
    d = np.asarray(direction, np.float64)
    lo_ = np.asarray(lo, np.float64)
    hi_ = np.asarray(hi, np.float64)
    k0 = np.zeros(1, np.int64)
    n = load_oracle().dvr_oracle_lattice(_ptr(o), _ptr(d), _ptr(lo_), _ptr(hi_), float(dt), _ptr(k0))
    return int(k0[0]), int(n)


# ---------------------------------------------------------------------------------------------
# field + bricks

def generate_field(dims, blobs, stored_lo=(0, 0, 0), stored_dims=None,
                   nthreads: int = 0, fast: bool = False) -> np.ndarray:
    """f32 voxels of the blob field over a stored region; array shape (sd_z, sd_y, sd_x).  ``blobs`` may
    also be a FieldSpec-like object with ``kind`` / ``blobs`` / ``ml`` (Marschner-Lobb fields)."""
    if hasattr(blobs, "kind"):
        spec = blobs
        if spec.kind == "marschnerLobb":
            return generate_ml(dims, spec.ml, stored_lo, stored_dims, nthreads)
        blobs = spec.blobs
    N = np.asarray(dims, np.int64)
    s_lo = np.asarray(stored_lo, np.int64)
    sd = np.asarray(stored_dims if stored_dims is not None else dims, np.int64)
    b = np.ascontiguousarray(blobs, np.float64).reshape(-1, 5)
    out = np.empty((int(sd[2]), int(sd[1]), int(sd[0])), np.float32)
    gen = load_oracle().dvr_oracle_generate_fast if fast else load_oracle().dvr_oracle_generate
    gen(_ptr(N), _ptr(s_lo), _ptr(sd), len(b), _ptr(b), _ptr(out), nthreads)
    return out


def generate_ml(dims, params=(6.0, 0.25), stored_lo=(0, 0, 0), stored_dims=None,
                nthreads: int = 0) -> np.ndarray:
    """f32 voxels of the Marschner-Lobb field (params = (f_M, alpha)), DESIGN.md §2.2b."""
    N = np.asarray(dims, np.int64)
    s_lo = np.asarray(stored_lo, np.int64)
    sd = np.asarray(stored_dims if stored_dims is not None else dims, np.int64)
    prm = np.ascontiguousarray(params, np.float64)
    out = np.empty((int(sd[2]), int(sd[1]), int(sd[0])), np.float32)
    load_oracle().dvr_oracle_generate_ml(_ptr(N), _ptr(s_lo), _ptr(sd), _ptr(prm), _ptr(out), nthreads)
    return out


def det_cos(a: float) -> float:
    """The oracle's reproducible cosine (range reduction + Taylor polynomial) used by generate_ml."""
    return float(load_oracle().dvr_oracle_det_cos(float(a)))


@dataclass
class OracleBrick:
    """The oracle's own view of a brick: owned cells [lo, hi), ghost g."""

    dims: Tuple[int, int, int]
    lo: Tuple[int, int, int]
    hi: Tuple[int, int, int]
    ghost: int = 1
    origin: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    spacing: Tuple[float, float, float] = (1.0, 1.0, 1.0)

    @property
    def stored_lo(self) -> Tuple[int, int, int]:
        return tuple(max(self.lo[a] - self.ghost, 0) for a in range(3))

    @property
    def stored_dims(self) -> Tuple[int, int, int]:
        return tuple(min(self.hi[a] + self.ghost, self.dims[a] - 1) - self.stored_lo[a] + 1 for a in range(3))

    def box_world(self):
        lo = tuple(self.origin[a] + float(self.lo[a]) * self.spacing[a] for a in range(3))
        hi = tuple(self.origin[a] + float(self.hi[a]) * self.spacing[a] for a in range(3))
        return lo, hi

    def extract(self, field: np.ndarray) -> np.ndarray:
        """Stored voxels of this brick out of a whole-field array (z, y, x)."""
        s = self.stored_lo
        d = self.stored_dims
        return np.ascontiguousarray(field[s[2]:s[2] + d[2], s[1]:s[1] + d[1], s[0]:s[0] + d[0]])


def sample_counts(brick: "OracleBrick", cam: np.ndarray, dt: float, width: int, height: int,
                  nthreads: int = 0) -> np.ndarray:
    """(H, W) owned lattice sample counts of the brick's owned box, no marching."""
    lo, hi = brick.box_world()
    lo_ = np.asarray(lo, np.float64)
    hi_ = np.asarray(hi, np.float64)
    out = np.zeros((height, width), np.uint32)
    load_oracle().dvr_oracle_sample_counts(_ptr(lo_), _ptr(hi_), _ptr(np.ascontiguousarray(cam, np.float64)),
                                           float(dt), width, height, _ptr(out), nthreads)
    return out


def render_brick(vox: np.ndarray, brick: OracleBrick, cam: np.ndarray, tf: np.ndarray, vmin: float,
                 vmax: float, dt: float, ert: float, width: int, height: int,
                 rows: Optional[Tuple[int, int, int]] = None, nthreads: int = 0):
    """One brick's RGBA partial (H, W, 4) f64 premultiplied + owned sample counts (H, W) u32."""
    vox = np.ascontiguousarray(vox, np.float32)
    if tuple(vox.shape) != tuple(reversed(brick.stored_dims)):
        raise ValueError(f"voxel array {vox.shape} does not match stored dims {brick.stored_dims}")
    geo = np.array([*brick.stored_lo, *brick.stored_dims, *brick.dims, *brick.lo, *brick.hi], np.int64)
    wgeo = np.array([*brick.origin, *brick.spacing], np.float64)
    tf = np.ascontiguousarray(tf, np.float32).reshape(-1, 4)
    n_tf = tf.shape[0]
    tf_scale = (n_tf - 1) / (float(vmax) - float(vmin))
    out = np.zeros((height, width, 4), np.float64)
    samples = np.zeros((height, width), np.uint32)
    r0, r1, rs = rows if rows is not None else (0, height, 1)
    rc = load_oracle().dvr_oracle_render_brick(
        _ptr(vox), _ptr(geo), _ptr(wgeo), _ptr(np.ascontiguousarray(cam, np.float64)), _ptr(tf), n_tf,
        float(vmin), float(tf_scale), float(dt), float(ert), width, height, r0, r1, rs, _ptr(out),
        _ptr(samples), nthreads)
    if rc != 0:
        raise ValueError(f"oracle render_brick failed with code {rc}")
    return out, samples


def render_lattice(vox: np.ndarray, brick: OracleBrick, cam: np.ndarray, tf: np.ndarray, vmin: float,
                   vmax: float, dt: float, ert: float, width: int, height: int, xs: int, ys: int,
                   x0: int = 0, y0: int = 0, nthreads: int = 0) -> np.ndarray:
    """One brick's RGBA partial (f64 premultiplied) on the pixel lattice (x0 + i xs, y0 + j ys): an
    (ny, nx, 4) array, ny = ceil((H - y0) / ys), nx = ceil((W - x0) / xs)."""
    vox = np.ascontiguousarray(vox, np.float32)
    if tuple(vox.shape) != tuple(reversed(brick.stored_dims)):
        raise ValueError(f"voxel array {vox.shape} does not match stored dims {brick.stored_dims}")
    geo = np.array([*brick.stored_lo, *brick.stored_dims, *brick.dims, *brick.lo, *brick.hi], np.int64)
    wgeo = np.array([*brick.origin, *brick.spacing], np.float64)
    tf = np.ascontiguousarray(tf, np.float32).reshape(-1, 4)
    tf_scale = (tf.shape[0] - 1) / (float(vmax) - float(vmin))
    nx = -(-(width - x0) // xs)
    ny = -(-(height - y0) // ys)
    out = np.zeros((ny, nx, 4), np.float64)
    rc = load_oracle().dvr_oracle_render_lattice(
        _ptr(vox), _ptr(geo), _ptr(wgeo), _ptr(np.ascontiguousarray(cam, np.float64)), _ptr(tf), tf.shape[0],
        float(vmin), float(tf_scale), float(dt), float(ert), width, height, x0, xs, nx, y0, ys, ny, _ptr(out),
        nthreads)
    if rc != 0:
        raise ValueError(f"oracle render_lattice failed with code {rc}")
    return out


def render_brick_accum(vox: np.ndarray, brick: OracleBrick, cam: np.ndarray, tf: np.ndarray, vmin: float,
                       vmax: float, dt: float, ert: float, width: int, height: int, state: np.ndarray,
                       rows: Tuple[int, int], nthreads: int = 0) -> None:
    """Ray cycling: continue the accumulated state (H, W, 4) f64 of rows [r0, r1) through
    one brick, in place (ERT on the accumulated alpha)."""
    vox = np.ascontiguousarray(vox, np.float32)
    if tuple(vox.shape) != tuple(reversed(brick.stored_dims)):
        raise ValueError(f"voxel array {vox.shape} does not match stored dims {brick.stored_dims}")
    if state.dtype != np.float64 or state.shape != (height, width, 4) or not state.flags["C_CONTIGUOUS"]:
        raise ValueError("state must be a C-contiguous (H, W, 4) float64 array")
    geo = np.array([*brick.stored_lo, *brick.stored_dims, *brick.dims, *brick.lo, *brick.hi], np.int64)
    wgeo = np.array([*brick.origin, *brick.spacing], np.float64)
    tf = np.ascontiguousarray(tf, np.float32).reshape(-1, 4)
    tf_scale = (tf.shape[0] - 1) / (float(vmax) - float(vmin))
    rc = load_oracle().dvr_oracle_render_brick_accum(
        _ptr(vox), _ptr(geo), _ptr(wgeo), _ptr(np.ascontiguousarray(cam, np.float64)), _ptr(tf), tf.shape[0],
        float(vmin), float(tf_scale), float(dt), float(ert), width, height, int(rows[0]), int(rows[1]), _ptr(state),
        nthreads)
    if rc != 0:
        raise ValueError(f"oracle render_brick_accum failed with code {rc}")


def cycle_frame(bricks_vox: Sequence[np.ndarray], bricks: Sequence[OracleBrick], order: Sequence[int],
                row_blocks: Sequence[Tuple[int, int]], cam: np.ndarray, tf: np.ndarray, vmin: float, vmax: float,
                dt: float, ert: float, width: int, height: int, background) -> np.ndarray:
    """The ray-cycling frame, restated serially: the batch of rank b's rows starts at b's
    position p0 in the visibility order and visits positions p0, p0+1, ..., R-1 (back segment, state B)
    then 0, ..., p0-1 (front segment, state F); the frame is F over B over the background."""
    R = len(bricks)
    pos = {s: i for i, s in enumerate(order)}
    out = np.zeros((height, width, 3), np.float64)
    for b in range(R):
        r0, r1 = row_blocks[b]
        if r1 <= r0:
            continue
        B = np.zeros((height, width, 4), np.float64)
        F = np.zeros((height, width, 4), np.float64)
        p0 = pos[b]
        for k in range(R):
            q = (p0 + k) % R
            s = order[q]
            render_brick_accum(bricks_vox[s], bricks[s], cam, tf, vmin, vmax, dt, ert, width, height,
                               B if q >= p0 else F, (r0, r1))
        acc = F.copy()
        acc[..., :3] += (1.0 - F[..., 3:4]) * B[..., :3]
        acc[..., 3:4] += (1.0 - F[..., 3:4]) * B[..., 3:4]
        img = acc[..., :3] + (1.0 - acc[..., 3:4]) * np.asarray(background, np.float64)
        out[r0:r1] = img[r0:r1]
    return out


# ---------------------------------------------------------------------------------------------
# compositing and output (engine.py:500-502)

def composite(partials: Sequence[np.ndarray], order: Sequence[int], background) -> np.ndarray:
    """Front-to-back 'over' of premultiplied partials in visibility order, then background."""
    shape = partials[0].shape[:-1]
    C = np.zeros(shape + (3,), np.float64)
    A = np.zeros(shape + (1,), np.float64)
    for r in order:
        p = np.asarray(partials[r], np.float64)
        one = 1.0 - A
        C = C + one * p[..., 0:3]
        A = A + one * p[..., 3:4]
    return C + (1.0 - A) * np.asarray(background, np.float64)


def tone_map_rgb8(image: np.ndarray) -> np.ndarray:
    """engine.py:500-502: clamp to [0, 1], quantize rounding half up."""
    return np.floor(np.clip(image, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)


# ---------------------------------------------------------------------------------------------
# brick decomposition and visibility order, restated independently of the product:
# iterative work list here, recursion in the product.  Axis choice follows geom.py:107-116
# (strict '>' so ties go to the lowest axis); integer cuts follow scene.py:234-238 (r*n//R).

def _slab_masses(field: np.ndarray, axis: int, lo, hi, tau: float) -> np.ndarray:
    """Per cell-slab count of voxels >= tau (voxel plane c, other axes over cells [lo, hi))."""
    sub = field[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] >= np.float32(tau)
    np_axis = 2 - axis
    other = tuple(a for a in range(3) if a != np_axis)
    return sub.sum(axis=other).astype(np.int64)


def kd_leaves(dims, spacing, P: int, strategy: str = "even", field: Optional[np.ndarray] = None,
              tau: float = 0.1):
    """Returns (leaves, nodes): leaves[rank] = (lo, hi) cell boxes; nodes = [(axis, cut, lrange, rrange)]."""
    if P < 1:
        raise ValueError("P must be >= 1")
    leaves: Dict[int, Tuple[Tuple[int, ...], Tuple[int, ...]]] = {}
    nodes = []
    work = [((0, 0, 0), tuple(int(d) - 1 for d in dims), P, 0)]
    while work:
        lo, hi, p, r0 = work.pop()
        if p == 1:
            leaves[r0] = (lo, hi)
            continue
        pl = p // 2
        ext = [(hi[a] - lo[a]) * float(spacing[a]) for a in range(3)]
        axis = 0
        if ext[1] > ext[axis]:
            axis = 1
        if ext[2] > ext[axis]:
            axis = 2
        n = hi[axis] - lo[axis]
        if n < 2:
            raise ValueError(f"cannot split {n} cells along axis {axis} into {p} bricks")
        cut = None
        if strategy == "mass":
            m = _slab_masses(field, axis, lo, hi, tau)
            total = int(m.sum())
            if total > 0:
                acc = 0
                for i in range(n - 1):
                    acc += int(m[i])
                    c = lo[axis] + i + 1
                    if p * acc >= total * pl:
                        cut = c
                        break
                if cut is None:
                    cut = hi[axis] - 1
        elif strategy != "even":
            raise ValueError(f"unknown strategy {strategy!r}")
        if cut is None:
            cut = lo[axis] + (n * pl) // p
        cut = min(max(cut, lo[axis] + 1), hi[axis] - 1)
        lhi = list(hi)
        lhi[axis] = cut
        rlo = list(lo)
        rlo[axis] = cut
        nodes.append((axis, cut, (r0, r0 + pl), (r0 + pl, r0 + p)))
        work.append((tuple(rlo), hi, p - pl, r0 + pl))
        work.append((lo, tuple(lhi), pl, r0))
    return [leaves[r] for r in range(P)], nodes


def kd_order(nodes, P: int, eye, origin, spacing) -> List[int]:
    """Front-to-back rank order: a rank range is split by each node; eye side first, ties lower first."""
    by_range = {(n[2][0], n[3][1]): n for n in nodes}
    out: List[int] = []
    stack = [(0, P)]
    while stack:
        a, b = stack.pop()
        if b - a == 1:
            out.append(a)
            continue
        axis, cut, lr, rr = by_range[(a, b)]
        s = float(origin[axis]) + float(cut) * float(spacing[axis])
        first, second = (lr, rr) if float(eye[axis]) <= s else (rr, lr)
        stack.append(second)
        stack.append(first)
    return out
