"""Host-side camera and box math (float64), the part of the reference's geom layer the DVR path keeps.

Semantics follow pkg/src/dprt/geom.py: ``CameraSpec`` validation and orthonormal ``basis()``
(geom.py:147-168), pixel-centre film mapping (geom.py:240-259), ``Aabb`` with the empty sentinel and
``longest_axis`` tie-break (geom.py:71-116).  Only what the host needs is here: per-pixel rays are
generated on the device (march.cu) with the identical operation order.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Tuple

Vec3 = Tuple[float, float, float]
INF = float("inf")


def _vdot(a: Vec3, b: Vec3) -> float:
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def _vcross(a: Vec3, b: Vec3) -> Vec3:
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def vlen(v: Vec3) -> float:
    return math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])


def unit(v: Vec3) -> Vec3:
    """v / |v| by three divisions (the rounding the reference's normalize uses, geom.py:51-55)."""
    n = vlen(v)
    if n == 0.0 or not math.isfinite(n):
        raise ValueError(f"cannot normalize degenerate vector {v!r}")
    return (v[0] / n, v[1] / n, v[2] / n)


def vsub(a: Vec3, b: Vec3) -> Vec3:
    return (a[0] - b[0], a[1] - b[1], a[2] - b[2])


def vadd(a: Vec3, b: Vec3) -> Vec3:
    return (a[0] + b[0], a[1] + b[1], a[2] + b[2])


def vscale(v: Vec3, s: float) -> Vec3:
    return (v[0] * s, v[1] * s, v[2] * s)


@dataclass(frozen=True)
class CameraSpec:
    """Pinhole camera; fov_y in degrees, aspect = width / height (geom.py:147-161)."""

    position: Vec3
    view_dir: Vec3
    up: Vec3
    fov_y: float
    aspect: float

    def __post_init__(self) -> None:
        if not (0.0 < self.fov_y < 180.0):
            raise ValueError(f"fov_y must be in (0, 180), got {self.fov_y}")
        if vlen(_vcross(tuple(self.view_dir), tuple(self.up))) == 0.0:
            raise ValueError("view_dir and up must not be parallel")

    def basis(self) -> Tuple[Vec3, Vec3, Vec3]:
        """(forward, right, up) orthonormal frame (geom.py:163-168)."""
        fwd = unit(tuple(float(c) for c in self.view_dir))
        right = unit(_vcross(fwd, tuple(float(c) for c in self.up)))
        return fwd, right, _vcross(right, fwd)

    def film_half_extents(self) -> Tuple[float, float]:
        """(half_w, half_h) of the film at distance 1 (geom.py:250-251)."""
        half_h = math.tan(math.radians(self.fov_y) * 0.5)
        return half_h * self.aspect, half_h


@dataclass(frozen=True)
class Aabb:
    """Axis-aligned box; empty when lo > hi on any axis (geom.py:71-83)."""

    lo: Vec3
    hi: Vec3

    @staticmethod
    def empty() -> "Aabb":
        return Aabb((INF, INF, INF), (-INF, -INF, -INF))

    def is_empty(self) -> bool:
        return any(self.lo[i] > self.hi[i] for i in range(3))

    def union(self, other: "Aabb") -> "Aabb":
        return Aabb(tuple(min(self.lo[i], other.lo[i]) for i in range(3)),
                    tuple(max(self.hi[i], other.hi[i]) for i in range(3)))

    def center(self) -> Vec3:
        return vscale(vadd(self.lo, self.hi), 0.5)

    def diagonal(self) -> float:
        return 0.0 if self.is_empty() else vlen(vsub(self.hi, self.lo))

    def longest_axis(self) -> int:
        """Index of the largest extent; ties resolve to the lowest axis (geom.py:107-116)."""
        if self.is_empty():
            return 0
        ext = vsub(self.hi, self.lo)
        best = 0
        for axis in (1, 2):
            if ext[axis] > ext[best]:
                best = axis
        return best


def auto_camera(box: Aabb, width: int, height: int, fov_y: float = 45.0) -> CameraSpec:
    """Deterministic framing: back off from the box centre along a fixed diagonal by 2.2 radii
    (the reference's default_camera, pkg/src/dprt/cli.py:23-34)."""
    if box.is_empty():
        center, radius = (0.0, 0.0, 0.0), 1.0
    else:
        center = box.center()
        radius = max(box.diagonal() * 0.5, 1e-6)
    position = vadd(center, vscale(unit((0.75, 0.55, 1.0)), 2.2 * radius))
    return CameraSpec(position, unit(vsub(center, position)), (0.0, 1.0, 0.0), fov_y, width / height)


def orbit_camera(target: Vec3, radius: float, yaw: float, pitch: float, fov_y: float, aspect: float) -> CameraSpec:
    """Orbit parametrisation of the (unshipped) viewer's orbit_update: position =
    target + radius * (cos p sin y, sin p, cos p cos y), view_dir = normalize(target - position)."""
    cp = math.cos(pitch)
    offset = (cp * math.sin(yaw), math.sin(pitch), cp * math.cos(yaw))
    position = vadd(target, vscale(offset, radius))
    return CameraSpec(position, unit(vsub(target, position)), (0.0, 1.0, 0.0), fov_y, aspect)
