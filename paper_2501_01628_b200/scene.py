"""Volume scene documents, brick partitioning and the time-step cache ("next" row 2).

The on-disk input side of the DVR path, shaped like the reference's triangle scene layer
(pkg/src/dprt/scene.py): a UTF-8 JSON document whose bulk data may live in a little-endian binary sidecar
referenced as ``{"binary": path, ...}`` (scene.py:79-93 does this for f64 triangles; here the sidecar is
the raw f32 field, x fastest), full validation with errors that name the offending field
(``SceneFormatError``, scene.py:61-76), ``partition_volume`` with the reference's strategy names where
they make sense (``spatialSlab`` -> even kd split, ``massBalanced`` -> mass-weighted kd split,
``fromFile`` -> an explicit brick table folded onto the rank count like scene.py:239-242), and the same
LRU ``TimestepCache`` contract (scene.py:292-341).

A rank never loads the whole field: ``brick_voxels`` memory-maps the sidecar and copies only the brick's
stored sub-box (owned cells + ghost), so a 2048^3 (32 GiB) time step costs each of 8 ranks 4.3 GB of I/O.

Document::

    {"format": "dprt-volume", "version": 1,
     "field": {"dims": [nx, ny, nz], "origin": [..], "spacing": [..],
               "data": {"binary": "step0.f32", "dtype": "<f4"}            # raw sidecar, x fastest
                    | {"generator": "blobs", "seed": 1, "blobCount": 16, "lopsided": false}
                    | {"generator": "marschnerLobb", "frequency": 6.0, "alpha": 0.25}},
     "transferFunction": {"table": [[r, g, b, a], ...] | {"binary": "tf.f32", "count": n},
                          "valueRange": [0, 1]},
     "background": [r, g, b],
     "bricks": [[[lo..], [hi..]], ...],     # optional explicit brick table (partition "fromFile")
     "timeSteps": ["step1.json", ...]}      # optional, loaded through TimestepCache
"""

from __future__ import annotations

import json
from collections import OrderedDict
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from .errors import SceneFormatError, UsageError
from .volume import (BrickDesc, Decomposition, FieldSpec, KdNode, TransferFunction1D, blob_mixture, decompose,
                     default_tf)

FORMAT = "dprt-volume"
VERSION = 1
PARTITION_STRATEGIES = ("spatialSlab", "massBalanced", "fromFile")


def _expect(cond: bool, where: str, msg: str) -> None:
    if not cond:
        raise SceneFormatError(f"{where}: {msg}")


def _numbers(value, n: int, where: str, kind=float) -> Tuple:
    _expect(isinstance(value, (list, tuple)) and len(value) == n, where, f"expected {n} numbers")
    for c in value:
        _expect(isinstance(c, (int, float)) and not isinstance(c, bool), where, f"expected {n} numbers")
        if kind is int:
            _expect(float(c).is_integer(), where, "expected integers")
    return tuple(kind(c) for c in value)


def _resolve(path: str, base_dir: Optional[Path]) -> Path:
    p = Path(path)
    return p if p.is_absolute() or base_dir is None else Path(base_dir) / p


@dataclass
class VolumeScene:
    """A parsed volume document (one time step)."""

    field: FieldSpec
    tf: TransferFunction1D
    background: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    data_path: Optional[Path] = None      # raw f32 sidecar, or None for a generated field
    bricks: Optional[List[Tuple[Tuple[int, int, int], Tuple[int, int, int]]]] = None
    time_steps: Optional[List[str]] = None
    generator: Optional[dict] = None

    def voxels(self) -> np.ndarray:
        """The whole field as a read-only memory map (z, y, x); generated fields are not stored."""
        if self.data_path is None:
            raise UsageError("generated fields have no voxel file; use DeviceBrick.generate")
        nx, ny, nz = self.field.dims
        return np.memmap(self.data_path, dtype="<f4", mode="r", shape=(nz, ny, nx))

    def brick_voxels(self, brick: BrickDesc) -> np.ndarray:
        """Only this brick's stored voxels (owned cells + ghost), copied out of the memory map."""
        s, d = brick.stored_lo, brick.stored_dims
        return np.ascontiguousarray(self.voxels()[s[2]:s[2] + d[2], s[1]:s[1] + d[1], s[0]:s[0] + d[0]],
                                    dtype=np.float32)


def parse_volume_scene(document: bytes, base_dir=None) -> VolumeScene:
    """Parse and fully validate a volume document; ``base_dir`` resolves relative sidecar paths."""
    try:
        doc = json.loads(document.decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise SceneFormatError(f"document: not valid UTF-8 JSON: {exc}") from exc
    _expect(isinstance(doc, dict), "document", "top level must be an object")
    known = {"format", "version", "field", "transferFunction", "background", "bricks", "timeSteps"}
    for key in doc:
        _expect(key in known, key, "unknown key")
    _expect(doc.get("format") == FORMAT, "format", f'must be "{FORMAT}"')
    _expect(doc.get("version") == VERSION, "version", f"must be {VERSION}")

    f = doc.get("field")
    _expect(isinstance(f, dict), "field", "expected an object")
    dims = _numbers(f.get("dims"), 3, "field.dims", int)
    _expect(all(d >= 2 for d in dims), "field.dims", "every axis needs >= 2 voxels")
    origin = _numbers(f.get("origin", (0, 0, 0)), 3, "field.origin")
    spacing = _numbers(f.get("spacing", (1, 1, 1)), 3, "field.spacing")
    _expect(all(s > 0 for s in spacing), "field.spacing", "components must be > 0")
    data = f.get("data")
    _expect(isinstance(data, dict), "field.data", "expected a binary reference or a generator")
    data_path = None
    generator = None
    blobs = np.zeros((0, 5))
    if "binary" in data:
        _expect(data.get("dtype", "<f4") == "<f4", "field.data.dtype", 'only "<f4" (little-endian f32)')
        data_path = _resolve(data["binary"], base_dir)
        _expect(data_path.exists(), "field.data.binary", f"sidecar {data_path} not found")
        need = 4 * dims[0] * dims[1] * dims[2]
        _expect(data_path.stat().st_size == need, "field.data.binary",
                f"sidecar holds {data_path.stat().st_size} bytes, expected {need}")
    elif data.get("generator") == "blobs":
        seed = data.get("seed", 1)
        count = data.get("blobCount", 16)
        _expect(isinstance(seed, int) and seed >= 0, "field.data.seed", "must be a non-negative integer")
        _expect(isinstance(count, int) and 1 <= count <= 64, "field.data.blobCount", "must be in 1..64")
        lop = bool(data.get("lopsided", False))
        blobs = blob_mixture(seed, count, lop)
        generator = {"generator": "blobs", "seed": seed, "blobCount": count, "lopsided": lop}
    elif data.get("generator") == "marschnerLobb":
        fm, alpha = data.get("frequency", 6.0), data.get("alpha", 0.25)
        _expect(isinstance(fm, (int, float)) and fm > 0, "field.data.frequency", "must be a number > 0")
        _expect(isinstance(alpha, (int, float)) and alpha >= 0, "field.data.alpha", "must be a number >= 0")
        generator = {"generator": "marschnerLobb", "frequency": float(fm), "alpha": float(alpha)}
    else:
        raise SceneFormatError('field.data: needs "binary" or "generator": "blobs" | "marschnerLobb"')
    if generator is not None and generator["generator"] == "marschnerLobb":
        fs = FieldSpec(dims, blobs, origin, spacing, "marschnerLobb", (generator["frequency"], generator["alpha"]))
    else:
        fs = FieldSpec(dims, blobs, origin, spacing)

    t = doc.get("transferFunction", {})
    _expect(isinstance(t, dict), "transferFunction", "expected an object")
    vr = _numbers(t.get("valueRange", (0.0, 1.0)), 2, "transferFunction.valueRange")
    _expect(vr[1] > vr[0], "transferFunction.valueRange", "needs max > min")
    table = t.get("table")
    if table is None:
        arr = default_tf().as_f32()
    elif isinstance(table, dict):
        count = table.get("count")
        _expect(isinstance(count, int) and 2 <= count <= 1024, "transferFunction.table.count", "must be 2..1024")
        path = _resolve(table.get("binary", ""), base_dir)
        try:
            arr = np.fromfile(path, dtype="<f4")
        except OSError as exc:
            raise SceneFormatError(f"transferFunction.table: cannot read {path}: {exc}") from exc
        _expect(arr.size == 4 * count, "transferFunction.table", f"sidecar holds {arr.size} floats, expected {4 * count}")
        arr = arr.reshape(count, 4)
    else:
        _expect(isinstance(table, list) and 2 <= len(table) <= 1024, "transferFunction.table",
                "expected 2..1024 RGBA entries")
        arr = np.array([_numbers(e, 4, f"transferFunction.table[{i}]") for i, e in enumerate(table)], np.float32)
    _expect(bool(np.all((arr >= 0) & (arr <= 1))), "transferFunction.table", "entries must be within [0, 1]")
    tf = TransferFunction1D(arr.astype(np.float32), vr[0], vr[1])

    bg = _numbers(doc.get("background", (0, 0, 0)), 3, "background")
    bricks = None
    if "bricks" in doc:
        b = doc["bricks"]
        _expect(isinstance(b, list) and len(b) >= 1, "bricks", "expected a non-empty array of [lo, hi] boxes")
        bricks = []
        for i, box in enumerate(b):
            _expect(isinstance(box, list) and len(box) == 2, f"bricks[{i}]", "expected [lo, hi]")
            lo = _numbers(box[0], 3, f"bricks[{i}].lo", int)
            hi = _numbers(box[1], 3, f"bricks[{i}].hi", int)
            _expect(all(0 <= lo[a] < hi[a] <= dims[a] - 1 for a in range(3)), f"bricks[{i}]",
                    "cells must satisfy 0 <= lo < hi <= dims - 1")
            bricks.append((lo, hi))
        cells = sum(int(np.prod([h - l for l, h in zip(lo, hi)])) for lo, hi in bricks)
        _expect(cells == int(np.prod([d - 1 for d in dims])), "bricks", "boxes must tile the cell grid exactly")
    steps = doc.get("timeSteps")
    if steps is not None:
        _expect(isinstance(steps, list) and all(isinstance(p, str) for p in steps), "timeSteps",
                "expected an array of document paths")
    return VolumeScene(fs, tf, bg, data_path, bricks, list(steps) if steps is not None else None, generator)


def serialize_volume_scene(scene: VolumeScene, data_ref: Optional[str] = None) -> bytes:
    """The document for ``scene`` (the sidecar itself is written by ``write_field``)."""
    f = scene.field
    if scene.generator is not None:
        data = dict(scene.generator)
    else:
        data = {"binary": data_ref or (str(scene.data_path) if scene.data_path else ""), "dtype": "<f4"}
    doc = {"format": FORMAT, "version": VERSION,
           "field": {"dims": list(f.dims), "origin": list(f.origin), "spacing": list(f.spacing), "data": data},
           "transferFunction": {"table": scene.tf.as_f32().tolist(), "valueRange": [scene.tf.vmin, scene.tf.vmax]},
           "background": list(scene.background)}
    if scene.bricks is not None:
        doc["bricks"] = [[list(lo), list(hi)] for lo, hi in scene.bricks]
    if scene.time_steps is not None:
        doc["timeSteps"] = list(scene.time_steps)
    return json.dumps(doc, separators=(",", ":")).encode("utf-8")


def write_field(path, voxels: np.ndarray) -> None:
    """Raw little-endian f32 sidecar, x fastest ((z, y, x) array order)."""
    np.ascontiguousarray(voxels, dtype="<f4").tofile(Path(path))


def partition_volume(scene: VolumeScene, num_ranks: int, strategy: str = "spatialSlab",
                     threshold: float = 0.1) -> Decomposition:
    """One brick per rank, deterministic per strategy (the partition_scene contract, scene.py:217-247)."""
    if num_ranks < 1:
        raise UsageError(f"num_ranks must be >= 1, got {num_ranks}")
    if strategy not in PARTITION_STRATEGIES:
        raise UsageError(f"unknown partition strategy {strategy!r}; choose from {PARTITION_STRATEGIES}")
    if strategy == "spatialSlab":
        return decompose(scene.field, num_ranks, "even")
    if strategy == "massBalanced":
        vox = scene.voxels() if scene.data_path is not None else None
        if vox is None:
            raise UsageError("massBalanced needs stored voxels (generated fields: use api 'mass' decomposition)")

        def mass(axis, lo, hi):
            sub = np.asarray(vox[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]) >= np.float32(threshold)
            return sub.sum(axis=tuple(a for a in range(3) if a != 2 - axis)).astype(np.int64)

        return decompose(scene.field, num_ranks, "mass", mass)
    if scene.bricks is None:
        raise UsageError("fromFile partitioning needs a 'bricks' table in the document")
    if len(scene.bricks) != num_ranks:
        raise UsageError(f"the brick table has {len(scene.bricks)} bricks for {num_ranks} ranks "
                         "(sort-last needs exactly one brick per rank)")
    root = _kd_from_boxes(list(range(num_ranks)), scene.bricks)
    if root is None:
        raise UsageError("the brick table is not a kd (guillotine) partition: no front-to-back order exists")
    return Decomposition(scene.field, list(scene.bricks), root, "fromFile")


def _kd_from_boxes(ranks: Sequence[int], boxes) -> Optional[object]:
    """Recover a kd tree over explicit boxes by finding guillotine cuts (needed for visibility order)."""
    if len(ranks) == 1:
        return ranks[0]
    for axis in range(3):
        cuts = sorted({boxes[r][0][axis] for r in ranks} - {min(boxes[r][0][axis] for r in ranks)})
        for c in cuts:
            left = [r for r in ranks if boxes[r][1][axis] <= c]
            right = [r for r in ranks if boxes[r][0][axis] >= c]
            if left and right and len(left) + len(right) == len(ranks):
                lt = _kd_from_boxes(left, boxes)
                rt = _kd_from_boxes(right, boxes)
                if lt is not None and rt is not None:
                    return KdNode(axis, c, min(ranks), max(ranks) + 1, lt, rt)
    return None


class TimestepCache:
    """LRU over time steps: loads on miss, evicts beyond ``capacity`` (the reference's TimestepCache
    contract, scene.py:292-327: hits / misses / evictions counters, residents least-recent first)."""

    def __init__(self, loader: Callable[[int], object], num_steps: int, capacity: int = 2):
        if capacity < 1:
            raise UsageError(f"capacity must be >= 1, got {capacity}")
        self._loader = loader
        self._num_steps = num_steps
        self._capacity = capacity
        self._resident: "OrderedDict[int, object]" = OrderedDict()
        self.hits = 0
        self.misses = 0
        self.evictions = 0

    @property
    def capacity(self) -> int:
        return self._capacity

    def residents(self) -> List[int]:
        return list(self._resident.keys())

    def fetch(self, step: int):
        if not (0 <= step < self._num_steps):
            raise UsageError(f"time step {step} out of range [0, {self._num_steps})")
        if step in self._resident:
            self.hits += 1
            self._resident.move_to_end(step)
            return self._resident[step]
        self.misses += 1
        value = self._loader(step)
        self._resident[step] = value
        while len(self._resident) > self._capacity:
            _, old = self._resident.popitem(last=False)
            self.evictions += 1
            close = getattr(old, "close", None)
            if callable(close):
                close()  # e.g. a DeviceBrick: its HBM is released on eviction
        return value


def timestep_cache_for(scene: VolumeScene, base_dir, capacity: int = 2) -> TimestepCache:
    """Cache whose steps parse the documents listed in ``scene.time_steps``."""
    steps = scene.time_steps or []
    base = Path(base_dir) if base_dir is not None else None

    def load(i: int) -> VolumeScene:
        path = _resolve(steps[i], base)
        return parse_volume_scene(path.read_bytes(), base_dir=path.parent)

    return TimestepCache(load, len(steps), capacity)
