"""Volume documents, sidecars, partition strategies and the time-step cache (CPU)."""

from __future__ import annotations

import json

import numpy as np
import pytest

import oracle
from paper_2501_01628_b200.errors import SceneFormatError, UsageError
from paper_2501_01628_b200.scene import (TimestepCache, VolumeScene, parse_volume_scene, partition_volume,
                                         serialize_volume_scene, timestep_cache_for, write_field)
from paper_2501_01628_b200.volume import blob_field, decompose, default_tf


def _doc(**over):
    d = {"format": "dprt-volume", "version": 1,
         "field": {"dims": [9, 8, 7], "data": {"generator": "blobs", "seed": 3, "blobCount": 4}}}
    d.update(over)
    return json.dumps(d).encode()


def test_generated_document_round_trip():
    s = parse_volume_scene(_doc(background=[0.1, 0.2, 0.3]))
    assert s.field.dims == (9, 8, 7) and s.background == (0.1, 0.2, 0.3)
    again = parse_volume_scene(serialize_volume_scene(s))
    assert again.field.dims == s.field.dims and np.array_equal(again.field.blobs, s.field.blobs)
    assert np.array_equal(again.tf.as_f32(), s.tf.as_f32())


def test_marschner_lobb_document_round_trip():
    s = parse_volume_scene(_doc(field={"dims": [9, 8, 7], "data": {"generator": "marschnerLobb", "frequency": 3}}))
    assert s.field.kind == "marschnerLobb" and s.field.ml == (3.0, 0.25)
    again = parse_volume_scene(serialize_volume_scene(s))
    assert again.field.kind == "marschnerLobb" and again.field.ml == (3.0, 0.25)
    with pytest.raises(SceneFormatError, match="frequency"):
        parse_volume_scene(_doc(field={"dims": [9, 8, 7], "data": {"generator": "marschnerLobb", "frequency": 0}}))


def test_binary_sidecar_and_brick_extraction(tmp_path):
    f = blob_field((21, 17, 13), seed=2)
    vox = oracle.generate_field(f.dims, f.blobs)
    write_field(tmp_path / "step0.f32", vox)
    doc = json.dumps({"format": "dprt-volume", "version": 1,
                      "field": {"dims": list(f.dims), "data": {"binary": "step0.f32"}}}).encode()
    s = parse_volume_scene(doc, base_dir=tmp_path)
    assert np.array_equal(np.asarray(s.voxels()), vox)
    dec = partition_volume(s, 4)
    for r in range(4):
        b = dec.brick(r)
        lo, d = b.stored_lo, b.stored_dims
        assert np.array_equal(s.brick_voxels(b), vox[lo[2]:lo[2] + d[2], lo[1]:lo[1] + d[1], lo[0]:lo[0] + d[0]])
    # the document written back references the same sidecar
    again = parse_volume_scene(serialize_volume_scene(s, data_ref="step0.f32"), base_dir=tmp_path)
    assert np.array_equal(np.asarray(again.voxels()), vox)


@pytest.mark.parametrize("bad,where", [
    ({"format": "x"}, "format"),
    ({"field": {"dims": [1, 8, 7], "data": {"generator": "blobs"}}}, "field.dims"),
    ({"field": {"dims": [9, 8, 7], "spacing": [1, 0, 1], "data": {"generator": "blobs"}}}, "field.spacing"),
    ({"field": {"dims": [9, 8, 7], "data": {}}}, "field.data"),
    ({"field": {"dims": [9, 8, 7], "data": {"binary": "missing.f32"}}}, "field.data.binary"),
    ({"transferFunction": {"table": [[0, 0, 0, 2], [1, 1, 1, 1]]}}, "transferFunction.table"),
    ({"transferFunction": {"valueRange": [1, 1]}}, "transferFunction.valueRange"),
    ({"bricks": [[[0, 0, 0], [8, 7, 6]], [[0, 0, 0], [1, 1, 1]]]}, "bricks"),
    ({"surprise": 1}, "surprise"),
])
def test_validation_names_the_field(bad, where):
    with pytest.raises(SceneFormatError, match=where.replace(".", r"\.")):
        parse_volume_scene(_doc(**bad))


def test_wrong_sidecar_size(tmp_path):
    (tmp_path / "v.f32").write_bytes(b"\0" * 12)
    doc = json.dumps({"format": "dprt-volume", "version": 1,
                      "field": {"dims": [9, 8, 7], "data": {"binary": "v.f32"}}}).encode()
    with pytest.raises(SceneFormatError, match="expected 2016"):
        parse_volume_scene(doc, base_dir=tmp_path)


def test_partition_strategies(tmp_path):
    f = blob_field((33, 25, 17), seed=3, lopsided=True)
    vox = oracle.generate_field(f.dims, f.blobs)
    write_field(tmp_path / "v.f32", vox)
    doc = {"format": "dprt-volume", "version": 1, "field": {"dims": list(f.dims), "data": {"binary": "v.f32"}}}
    s = parse_volume_scene(json.dumps(doc).encode(), base_dir=tmp_path)
    assert partition_volume(s, 4, "spatialSlab").boxes == decompose(f, 4).boxes
    mb = partition_volume(s, 4, "massBalanced")
    leaves, _ = oracle.kd_leaves(f.dims, f.spacing, 4, "mass", field=vox)
    assert [tuple(map(tuple, l)) for l in leaves] == mb.boxes
    # fromFile: an explicit kd table is accepted and its visibility order recovered
    doc["bricks"] = [[list(lo), list(hi)] for lo, hi in mb.boxes]
    s2 = parse_volume_scene(json.dumps(doc).encode(), base_dir=tmp_path)
    ff = partition_volume(s2, 4, "fromFile")
    assert ff.boxes == mb.boxes
    for eye in [(-5.0, 3.0, 2.0), (40.0, 30.0, -9.0), (16.0, 12.0, 8.0)]:
        assert ff.visibility_order(eye) == mb.visibility_order(eye)
    with pytest.raises(UsageError, match="one brick per rank"):
        partition_volume(s2, 2, "fromFile")
    with pytest.raises(UsageError, match="unknown partition strategy"):
        partition_volume(s2, 2, "roundRobin")


def test_non_guillotine_brick_table_is_rejected():
    # a pinwheel of 5 boxes tiling a 3x3 cell square (x, y) has no guillotine cut
    boxes = [[[0, 0, 0], [2, 1, 1]], [[2, 0, 0], [3, 2, 1]], [[1, 2, 0], [3, 3, 1]], [[0, 1, 0], [1, 3, 1]],
             [[1, 1, 0], [2, 2, 1]]]
    s = parse_volume_scene(_doc(field={"dims": [4, 4, 2], "data": {"generator": "blobs"}}, bricks=boxes))
    with pytest.raises(UsageError, match="not a kd"):
        partition_volume(s, 5, "fromFile")


class _Closable:
    def __init__(self, i):
        self.i = i
        self.closed = False

    def close(self):
        self.closed = True


def test_timestep_cache_lru_semantics():
    loaded = []

    def loader(i):
        loaded.append(i)
        return _Closable(i)

    c = TimestepCache(loader, 5, capacity=2)
    a = c.fetch(0)
    c.fetch(1)
    c.fetch(0)
    assert c.residents() == [1, 0] and (c.hits, c.misses) == (1, 2)
    c.fetch(2)  # evicts 1 (least recently used)
    assert c.residents() == [0, 2] and c.evictions == 1 and loaded == [0, 1, 0 + 2]
    assert not a.closed
    with pytest.raises(UsageError):
        c.fetch(5)
    with pytest.raises(UsageError):
        TimestepCache(loader, 5, capacity=0)


def test_timestep_documents(tmp_path):
    for i in range(3):
        (tmp_path / f"s{i}.json").write_bytes(
            _doc(field={"dims": [9, 8, 7], "data": {"generator": "blobs", "seed": i}}))
    root = parse_volume_scene(_doc(timeSteps=["s0.json", "s1.json", "s2.json"]))
    cache = timestep_cache_for(root, tmp_path, capacity=2)
    seeds = [cache.fetch(i).generator["seed"] for i in (0, 1, 2, 0)]
    assert seeds == [0, 1, 2, 0] and cache.evictions == 2
