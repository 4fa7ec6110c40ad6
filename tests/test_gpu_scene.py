"""A volume document with a raw f32 sidecar renders the same frame as the generated field (GPU)."""

from __future__ import annotations

import json

import numpy as np
import pytest
import torch

import oracle
from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.geom import auto_camera
from paper_2501_01628_b200.scene import parse_volume_scene, partition_volume, write_field
from paper_2501_01628_b200.volume import blob_field

pytestmark = pytest.mark.gpu


def test_sidecar_bricks_render_like_generated_bricks(cuda_device, oracle_lib, tmp_path):
    f = blob_field((48, 40, 36), seed=6)
    write_field(tmp_path / "v.f32", oracle.generate_field(f.dims, f.blobs))
    doc = {"format": "dprt-volume", "version": 1, "field": {"dims": list(f.dims), "data": {"binary": "v.f32"}}}
    s = parse_volume_scene(json.dumps(doc).encode(), base_dir=tmp_path)
    dec = partition_volume(s, 2)
    W, H = 64, 48
    cam = auto_camera(f.bounds(), W, H)
    dtf = dev.DeviceTF(s.tf, cuda_device)
    for r in range(2):
        a = dev.DeviceBrick(dec.brick(r), cuda_device).upload(s.brick_voxels(dec.brick(r)))
        b = dev.DeviceBrick(dec.brick(r), cuda_device).generate(f)
        pa = torch.empty(W * H * 4, dtype=torch.float32, device=cuda_device)
        pb = torch.empty_like(pa)
        dev.march(a, cam, dtf, 1.0, 0.99, pa, W, H)
        dev.march(b, cam, dtf, 1.0, 0.99, pb, W, H)
        torch.cuda.synchronize()
        assert torch.equal(pa, pb)
        a.close()
        b.close()
