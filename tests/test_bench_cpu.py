"""CPU checks of bench.py's host logic and the oracle entry points it uses (no GPU): workloads per config,
identical config objects in both arms, the chunked host mass function, and the oracle's fast generator /
pixel-lattice renderer against the scalar ones."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import bench
import oracle
from paper_2501_01628_b200.volume import blob_field, decompose, default_tf

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("R", [1, 2, 4, 8])
def test_c3_family_is_config3_at_eight_ranks(R):
    dims = bench.field_dims(1024, R)
    cells = np.prod([d - 1 for d in dims])
    assert cells == R * 1024 ** 3
    if R == 8:
        assert dims == (2049, 2049, 2049)
        wl = bench.build_workload("c3", 8, "even")
        assert (wl.W, wl.H) == (3840, 2160)
        assert all(tuple(int(h) - int(l) for l, h in zip(*b)) == (1024, 1024, 1024) for b in wl.dec.boxes)


def test_default_configs():
    assert bench.resolve_config("auto", 1) == "c2"
    assert bench.resolve_config("auto", 8) == "c3"
    wl = bench.build_workload("c2", 1, "mass")
    assert wl.field.dims == (513, 513, 513) and (wl.W, wl.H) == (1920, 1080) and wl.strategy == "whole"
    wl4 = bench.build_workload("c4", 8, "even")
    assert len(wl4.cams) == 36 and wl4.field.spacing == (1.0, 1.0, 2.0)


def test_reference_arm_config_matches_ours():
    """Both arms build ``config`` from the same Workload.config, so the driver's same-config check holds."""
    for cfg, R in (("c1", 2), ("c2", 1), ("c3", 8)):
        assert bench.build_workload(cfg, R, "even").config(R) == bench.build_workload(cfg, R, "even").config(R)
    src = (ROOT / "bench.py").read_text()
    assert src.count('"config": wl.config(R),') == 2  # the reference arm and ours: nothing arm-specific added


def test_reference_arm_runs_and_prints_one_line():
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2", "--config", "c1",
                        "--steps", "2", "--warmup", "3", "--decomposition", "even"],
                       capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert p.returncode == 0, p.stderr[-1500:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["config"]["bricks"] == 2


def test_host_mass_function_chunks_equal_whole_field():
    f = blob_field((97, 81, 65), seed=3)
    vox = oracle.generate_field(f.dims, f.blobs)
    mask = vox >= np.float32(0.1)

    def whole(axis, lo, hi):
        sub = mask[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        return sub.sum(axis=tuple(a for a in range(3) if a != 2 - axis), dtype=np.int64)

    assert decompose(f, 8, "mass", bench.host_mass_function(f, 0.1, chunk=16)).boxes == \
        decompose(f, 8, "mass", whole).boxes


@pytest.mark.parametrize("dims,lo,sd,seed,lop", [((2049, 2049, 2049), (900, 1000, 700), (60, 70, 80), 1, False),
                                                  ((200, 300, 250), (0, 0, 0), (200, 300, 250), 7, True),
                                                  ((65, 65, 65), (0, 0, 0), (65, 65, 65), 1, False)])
def test_fast_generator_is_bit_identical(dims, lo, sd, seed, lop):
    f = blob_field(dims, seed=seed, lopsided=lop)
    a = oracle.generate_field(f.dims, f.blobs, lo, sd)
    b = oracle.generate_field(f.dims, f.blobs, lo, sd, fast=True)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_render_lattice_equals_render_brick_at_lattice_pixels():
    f = blob_field((49, 41, 37), seed=4)
    dec = decompose(f, 2)
    W, H = 50, 38
    from paper_2501_01628_b200.geom import auto_camera

    cam = auto_camera(f.bounds(), W, H)
    ca = oracle.camera_array(cam.position, cam.view_dir, cam.up, cam.fov_y, cam.aspect)
    tf = default_tf()
    vox = oracle.generate_field(f.dims, f.blobs)
    for r in range(2):
        lo, hi = dec.boxes[r]
        ob = oracle.OracleBrick(f.dims, lo, hi, 1, f.origin, f.spacing)
        full, _ = oracle.render_brick(ob.extract(vox), ob, ca, tf.as_f32(), 0.0, 1.0, 1.0, 0.99, W, H)
        lat = oracle.render_lattice(ob.extract(vox), ob, ca, tf.as_f32(), 0.0, 1.0, 1.0, 0.99, W, H, 3, 4, x0=1, y0=2)
        assert np.array_equal(lat, full[2::4, 1::3])
