"""Volume-side scene description: synthetic field, transfer function, bricks, kd decomposition and
visibility order.

These take the place of the reference's scene layer for triangles (pkg/src/dprt/scene.py): the seeded
generator ``generate_uneven_cloud`` (scene.py:250-289) becomes a seeded blob-mixture field, and the
deterministic object-space partition ``partition_scene`` (scene.py:217-247, spatialSlab = cuts along the
longest axis at r*n//R) becomes a kd split of the cell grid into one brick per rank.  Because 'over' is
not commutative (unlike the reference's (t, gid) min, bvh.py:246-248), the kd tree also yields the
front-to-back brick order for any eye position.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple, Union

import numpy as np

from .errors import UsageError
from .geom import Aabb, Vec3

# ------------------------------------------------------------------------------------------------
# field


FIELD_KINDS = ("blobs", "marschnerLobb")


@dataclass(frozen=True)
class FieldSpec:
    """Vertex-centred scalar field: dims voxels, voxel (i,j,k) at origin + (i,j,k)*spacing.
    ``kind`` "blobs": ``blobs`` (K x 5: cx, cy, cz, inv_rho2, amp in unit-cube coordinates) defines the
    synthetic blob-mixture values.  ``kind`` "marschnerLobb": the Marschner-Lobb test
    signal over [-1, 1]^3 with ``ml`` = (f_M, alpha) (``blobs`` unused)."""

    dims: Tuple[int, int, int]
    blobs: np.ndarray = field(repr=False)
    origin: Vec3 = (0.0, 0.0, 0.0)
    spacing: Vec3 = (1.0, 1.0, 1.0)
    kind: str = "blobs"
    ml: Tuple[float, float] = (6.0, 0.25)

    def __post_init__(self) -> None:
        if len(self.dims) != 3 or any(int(d) < 2 for d in self.dims):
            raise UsageError(f"field dims must be three integers >= 2, got {self.dims}")
        if self.kind not in FIELD_KINDS:
            raise UsageError(f"unknown field kind {self.kind!r}; choose from {FIELD_KINDS}")
        b = np.asarray(self.blobs, np.float64)
        if b.ndim != 2 or b.shape[1] != 5 or b.shape[0] > 64:
            raise UsageError(f"blobs must be a (K <= 64, 5) array, got {b.shape}")
        if self.kind == "marschnerLobb" and not (float(self.ml[0]) > 0.0 and float(self.ml[1]) >= 0.0):
            raise UsageError(f"Marschner-Lobb needs f_M > 0 and alpha >= 0, got {self.ml}")

    def bounds(self) -> Aabb:
        hi = tuple(self.origin[a] + float(self.dims[a] - 1) * self.spacing[a] for a in range(3))
        return Aabb(tuple(float(c) for c in self.origin), hi)

    @property
    def cells(self) -> Tuple[int, int, int]:
        return tuple(int(d) - 1 for d in self.dims)

    @property
    def nbytes(self) -> int:
        return 4 * int(np.prod(np.asarray(self.dims, np.int64)))


def blob_mixture(seed: int, n_blobs: int = 16, lopsided: bool = False) -> np.ndarray:
    """Seeded blob parameters, drawn like generate_uneven_cloud's mixture (scene.py:258-262):
    PCG64(seed), centres U[0,1)^3, sigma U(.02,.08), weights U(.5,2) (times 3^k when ``lopsided``).
    Each blob is the polynomial bump amp*(1 - r^2/rho^2)^3 for r < rho = 3 sigma (no exp, so CPU and
    GPU agree bit for bit); amplitudes are scaled so the largest is 1."""
    if not (1 <= n_blobs <= 64):
        raise UsageError(f"need 1..64 blobs, got {n_blobs}")
    rng = np.random.Generator(np.random.PCG64(seed))
    centers = rng.random((n_blobs, 3))
    sigma = rng.uniform(0.02, 0.08, n_blobs)
    weights = rng.uniform(0.5, 2.0, n_blobs)
    if lopsided:
        weights = weights * (3.0 ** np.arange(n_blobs))
    amp = weights / weights.max()
    rho = 3.0 * sigma
    return np.column_stack([centers, 1.0 / (rho * rho), amp]).astype(np.float64)


def blob_field(dims, seed: int = 1, n_blobs: int = 16, spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0),
               lopsided: bool = False) -> FieldSpec:
    return FieldSpec(tuple(int(d) for d in dims), blob_mixture(seed, n_blobs, lopsided),
                     tuple(float(o) for o in origin), tuple(float(s) for s in spacing))


def marschner_lobb_field(dims, f_m: float = 6.0, alpha: float = 0.25, spacing=(1.0, 1.0, 1.0),
                         origin=(0.0, 0.0, 0.0)) -> FieldSpec:
    """The Marschner-Lobb signal (smooth, high-frequency stress for trilinear + TF)."""
    return FieldSpec(tuple(int(d) for d in dims), np.zeros((0, 5)), tuple(float(o) for o in origin),
                     tuple(float(s) for s in spacing), "marschnerLobb", (float(f_m), float(alpha)))


# ------------------------------------------------------------------------------------------------
# transfer function


@dataclass(frozen=True)
class TransferFunction1D:
    """RGBA table (n x 4 f32: non-premultiplied colour, opacity per sample at the fixed dt) over
    [vmin, vmax]; lookup interpolates linearly between entries and clamps."""

    table: np.ndarray = field(repr=False)
    vmin: float = 0.0
    vmax: float = 1.0

    def __post_init__(self) -> None:
        t = np.asarray(self.table)
        if t.ndim != 2 or t.shape[1] != 4 or not (2 <= t.shape[0] <= 1024):
            raise UsageError(f"transfer function table must be (2..1024, 4), got {t.shape}")
        if not (float(self.vmax) > float(self.vmin)):
            raise UsageError("transfer function needs vmax > vmin")

    @property
    def n(self) -> int:
        return int(np.asarray(self.table).shape[0])

    def as_f32(self) -> np.ndarray:
        return np.ascontiguousarray(self.table, np.float32)


_RAMP_STOPS = np.array([(0.10, 0.20, 0.90), (0.10, 0.80, 0.80), (0.95, 0.90, 0.20), (0.90, 0.20, 0.10)],
                       np.float64)


def default_tf(n: int = 256, threshold: float = 0.1, alpha_max: float = 0.05) -> TransferFunction1D:
    """SURVEY §8(d) TF: alpha 0 below ``threshold``, rising linearly to ``alpha_max`` at 1; colour from a
    fixed 4-stop ramp; no RNG."""
    x = np.arange(n, dtype=np.float64) / (n - 1)
    alpha = np.where(x < threshold, 0.0, alpha_max * (x - threshold) / (1.0 - threshold))
    seg = np.minimum((x * 3.0).astype(np.int64), 2)
    f = x * 3.0 - seg
    rgb = _RAMP_STOPS[seg] * (1.0 - f)[:, None] + _RAMP_STOPS[seg + 1] * f[:, None]
    return TransferFunction1D(np.column_stack([rgb, alpha]).astype(np.float32), 0.0, 1.0)


def opaque_tf(n: int = 256, threshold: float = 0.1) -> TransferFunction1D:
    """alpha = 1 at or above ``threshold`` (first non-empty sample terminates the ray); white."""
    x = np.arange(n, dtype=np.float64) / (n - 1)
    a = np.where(x >= threshold, 1.0, 0.0)
    return TransferFunction1D(np.column_stack([a, a, a, a]).astype(np.float32), 0.0, 1.0)


# ------------------------------------------------------------------------------------------------
# bricks


@dataclass(frozen=True)
class BrickDesc:
    """One rank's brick: owns cells [lo, hi) of ``dims`` voxels, stores voxels [lo-ghost, hi+ghost]
    clipped to the grid."""

    dims: Tuple[int, int, int]
    lo: Tuple[int, int, int]
    hi: Tuple[int, int, int]
    ghost: int = 1
    origin: Vec3 = (0.0, 0.0, 0.0)
    spacing: Vec3 = (1.0, 1.0, 1.0)

    def __post_init__(self) -> None:
        for a in range(3):
            if not (0 <= self.lo[a] < self.hi[a] <= self.dims[a] - 1):
                raise UsageError(f"brick cells [{self.lo[a]}, {self.hi[a]}) invalid on axis {a} for {self.dims[a]} voxels")
        if self.ghost < 0:
            raise UsageError("ghost must be >= 0")

    @property
    def stored_lo(self) -> Tuple[int, int, int]:
        return tuple(max(self.lo[a] - self.ghost, 0) for a in range(3))

    @property
    def stored_dims(self) -> Tuple[int, int, int]:
        s = self.stored_lo
        return tuple(min(self.hi[a] + self.ghost, self.dims[a] - 1) - s[a] + 1 for a in range(3))

    @property
    def stored_bytes(self) -> int:
        d = self.stored_dims
        return 4 * d[0] * d[1] * d[2]

    def box_world(self) -> Aabb:
        return Aabb(tuple(self.origin[a] + float(self.lo[a]) * self.spacing[a] for a in range(3)),
                    tuple(self.origin[a] + float(self.hi[a]) * self.spacing[a] for a in range(3)))

    @staticmethod
    def whole(f: FieldSpec, ghost: int = 1) -> "BrickDesc":
        return BrickDesc(f.dims, (0, 0, 0), f.cells, ghost, f.origin, f.spacing)


# ------------------------------------------------------------------------------------------------
# kd decomposition and visibility order


@dataclass
class KdNode:
    """Split of the rank range [r0, r1) at cell plane ``cut`` on ``axis``; children are KdNode or a rank."""

    axis: int
    cut: int
    r0: int
    r1: int
    left: Union["KdNode", int]
    right: Union["KdNode", int]


@dataclass
class Decomposition:
    """rank -> owned cell box, plus the kd tree that produced it."""

    field: FieldSpec
    boxes: List[Tuple[Tuple[int, int, int], Tuple[int, int, int]]]
    root: Union[KdNode, int]
    strategy: str

    @property
    def P(self) -> int:
        return len(self.boxes)

    def brick(self, rank: int, ghost: int = 1) -> BrickDesc:
        lo, hi = self.boxes[rank]
        return BrickDesc(self.field.dims, lo, hi, ghost, self.field.origin, self.field.spacing)

    def visibility_order(self, eye: Vec3) -> List[int]:
        return visibility_order(self, eye)


MassFn = Callable[[int, Tuple[int, int, int], Tuple[int, int, int]], np.ndarray]


def decompose(f: FieldSpec, P: int, strategy: str = "even", mass: Optional[MassFn] = None) -> Decomposition:
    """Split the cell grid into P bricks, one per rank, by recursive bisection of the rank range.

    Each node splits along the longest world extent of its box (ties -> lowest axis, geom.py:107-116);
    ``even`` cuts at lo + n*P_left//P (the integer rule of scene.py:234-238); ``mass`` cuts at the first
    cell plane where the running integer mass reaches P_left/P of the node's total, using
    ``mass(axis, lo, hi)`` = per-cell-slab counts of non-empty voxels.  Leaves are ranks in order, so
    ranks that differ only in bit k are kd siblings at depth log2(P)-1-k (binary-swap partners).
    """
    if P < 1:
        raise UsageError(f"need at least one brick, got {P}")
    if strategy not in ("even", "mass"):
        raise UsageError(f"unknown decomposition strategy {strategy!r}; choose 'even' or 'mass'")
    if strategy == "mass" and mass is None:
        raise UsageError("mass decomposition needs a mass function")
    boxes: List = [None] * P

    def split(lo, hi, r0, r1):
        p = r1 - r0
        if p == 1:
            boxes[r0] = (tuple(lo), tuple(hi))
            return r0
        ext = [float(hi[a] - lo[a]) * f.spacing[a] for a in range(3)]
        axis = 0
        for a in (1, 2):  # strict '>' -> ties go to the lowest axis (geom.py:112-116)
            if ext[a] > ext[axis]:
                axis = a
        n = hi[axis] - lo[axis]
        if n < 2:
            raise UsageError(f"cannot split {n} cells along axis {axis} between {p} ranks")
        pl = p // 2
        cut = lo[axis] + (n * pl) // p
        if strategy == "mass":
            m = np.asarray(mass(axis, tuple(lo), tuple(hi)), np.int64)
            total = int(m.sum())
            if total > 0:
                run = np.cumsum(m[:-1])
                hit = np.nonzero(run * p >= total * pl)[0]
                cut = lo[axis] + 1 + int(hit[0]) if hit.size else hi[axis] - 1
        cut = min(max(cut, lo[axis] + 1), hi[axis] - 1)
        lhi = list(hi)
        lhi[axis] = cut
        rlo = list(lo)
        rlo[axis] = cut
        left = split(lo, lhi, r0, r0 + pl)
        right = split(rlo, hi, r0 + pl, r1)
        return KdNode(axis, cut, r0, r1, left, right)

    root = split([0, 0, 0], list(f.cells), 0, P)
    return Decomposition(f, boxes, root, strategy)


def visibility_order(d: Decomposition, eye: Vec3) -> List[int]:
    """Front-to-back rank order for an eye point: at every split, the side containing the eye first
    (eye exactly on the plane -> lower side first).  Valid for every ray of a perspective camera because
    kd leaves are convex and separated by the split planes."""
    out: List[int] = []

    def walk(node):
        if isinstance(node, int):
            out.append(node)
            return
        plane = d.field.origin[node.axis] + float(node.cut) * d.field.spacing[node.axis]
        if float(eye[node.axis]) <= plane:
            walk(node.left)
            walk(node.right)
        else:
            walk(node.right)
            walk(node.left)

    walk(d.root)
    return out


def binary_swap_compatible(order: Sequence[int]) -> bool:
    """True when every aligned rank group {g*2^k .. (g+1)*2^k - 1} is contiguous in ``order`` -- the
    condition for merging XOR partners round by round (always true for power-of-2 kd decompositions)."""
    P = len(order)
    if P & (P - 1):
        return False
    pos = {r: i for i, r in enumerate(order)}
    size = 2
    while size <= P:
        for g in range(0, P, size):
            idx = sorted(pos[r] for r in range(g, g + size))
            if idx[-1] - idx[0] != size - 1:
                return False
        size *= 2
    return True
