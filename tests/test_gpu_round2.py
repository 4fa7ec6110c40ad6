"""Round-2 additions on the GPU: the roofline instrumentation (dprt_march_stats), the argument bounds the
ABI now enforces (samples per ray, fp16-quad value range), the lazy API frame read-back, multi-device
rank threads, and bench.py's own entry points (self-launched ranks, compositing-only sweep)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle
from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.errors import UsageError
from paper_2501_01628_b200.geom import auto_camera
from paper_2501_01628_b200.volume import BrickDesc, FieldSpec, blob_field, decompose, default_tf

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _brick(f, P, r, device, **kw):
    return dev.DeviceBrick(decompose(f, P).brick(r), device, **kw).generate(f)


@pytest.mark.parametrize("P", [1, 2, 4])
def test_march_stats_counts_are_exact(cuda_device, P):
    """Without ERT and without skipping every owned sample is shaded exactly once: shaded == the per-pixel
    sample counts' sum.  Exact skipping only drops samples that add exact zeros, so the contributing
    samples (w > 0) are the same with and without it -- with ERT too (A evolves identically)."""
    f = blob_field((72, 64, 56), seed=5)
    W, H = 96, 80
    cam = auto_camera(f.bounds(), W, H)
    tf = default_tf()
    dtf = dev.DeviceTF(tf, cuda_device)
    for r in range(P):
        b = _brick(f, P, r, cuda_device)
        part = torch.empty(W * H * 4, dtype=torch.float32, device=cuda_device)
        s = torch.empty(W * H, dtype=torch.int32, device=cuda_device)
        dev.march(b, cam, dtf, 1.0, 2.0, part, W, H, samples=s, skip=False)
        owned = int(s.sum(dtype=torch.int64).item())
        noskip = dev.march_stats(b, cam, dtf, 1.0, 2.0, W, H, skip=False)
        assert noskip["shaded_samples"] == owned
        withskip = dev.march_stats(b, cam, dtf, 1.0, 2.0, W, H, skip=True)
        assert withskip["contributing_samples"] == noskip["contributing_samples"]
        assert withskip["shaded_samples"] <= noskip["shaded_samples"]
        ert_skip = dev.march_stats(b, cam, dtf, 1.0, 0.9, W, H, skip=True)
        ert_noskip = dev.march_stats(b, cam, dtf, 1.0, 0.9, W, H, skip=False)
        assert ert_skip["contributing_samples"] == ert_noskip["contributing_samples"]
        # needed voxels: whole macrocells the shading touched, never more than the brick's cells
        cells = int(np.prod([d - 1 for d in b.desc.stored_dims]))
        assert 0 < withskip["needed_voxels"] <= noskip["needed_voxels"] <= cells
        assert withskip["needed_bytes"] == 4 * withskip["needed_voxels"]
        b.close()


def test_march_stats_needed_macrocells_match_host_restatement(cuda_device):
    """With skipping off and ERT off, the macrocells holding a shaded sample are those some owned lattice
    sample falls in: restated on the host from the oracle's lattice ranges and f32 sample positions."""
    f = blob_field((40, 36, 33), seed=2)
    W, H = 24, 20
    cam = auto_camera(f.bounds(), W, H)
    dtf = dev.DeviceTF(default_tf(), cuda_device)
    desc = BrickDesc.whole(f, 1)
    b = dev.DeviceBrick(desc, cuda_device).generate(f)
    st = dev.march_stats(b, cam, dtf, 1.0, 2.0, W, H, skip=False)
    ms = b.macro_shift
    assert ms == 2  # a small brick: 4^3 macrocells
    ca = oracle.camera_array(cam.position, cam.view_dir, cam.up, cam.fov_y, cam.aspect)
    dirs = oracle.primary_dirs(ca, W, H).reshape(-1, 3)
    lo_w, hi_w = desc.box_world().lo, desc.box_world().hi
    marked = set()
    sd = desc.stored_dims
    for d in dirs:
        k0, n = oracle.lattice(cam.position, d, lo_w, hi_w, 1.0)
        for k in range(k0, k0 + n):
            t = k * 1.0
            p = [cam.position[a] + t * d[a] for a in range(3)]
            c = [min(max(int(np.floor(p[a])), 0), sd[a] - 2) >> ms for a in range(3)]
            marked.add(tuple(c))
    # f32 positions may round across a macrocell face: allow a handful of boundary differences
    assert abs(st["macrocells"] - len(marked)) <= max(2, len(marked) // 50)


def test_samples_per_ray_bound_is_enforced(cuda_device):
    f = blob_field((33, 33, 33), seed=1)
    b = dev.DeviceBrick(BrickDesc.whole(f), cuda_device).generate(f)
    cam = auto_camera(f.bounds(), 8, 8)
    dtf = dev.DeviceTF(default_tf(), cuda_device)
    part = torch.empty(8 * 8 * 4, dtype=torch.float32, device=cuda_device)
    with pytest.raises(UsageError, match="2\\^24"):
        dev.march(b, cam, dtf, 1e-6, 0.99, part, 8, 8)
    dev.march(b, cam, dtf, 1e-2, 0.99, part, 8, 8)  # 5.7e3 samples per ray: fine
    b.close()


def test_half_quads_reject_values_outside_range(cuda_device):
    """fp16 quads' stated bound is for values in [0, 1]; values beyond +-8 are refused at commit time."""
    f = blob_field((17, 17, 17), seed=1)
    desc = BrickDesc.whole(f, 1)
    vox = np.full(tuple(reversed(desc.stored_dims)), 0.5, np.float32)
    b = dev.DeviceBrick(desc, cuda_device, half_quads=True)
    b.upload(vox)  # in range
    vox[3, 4, 5] = 100.0
    with pytest.raises(UsageError, match="fp16 quads"):
        b.upload(vox)
    b.close()
    f32 = dev.DeviceBrick(desc, cuda_device)
    f32.upload(vox)  # f32 quads take any finite value
    f32.close()


def test_api_frame_result_is_lazy_and_invalidated(cuda_device):
    from paper_2501_01628_b200 import api
    from paper_2501_01628_b200.transport import SoloEndpoint

    d = api.Device(SoloEndpoint(cuda_device), cuda_device)
    fld = d.create("spatialField")
    fld.set_param("dims", (48, 48, 48))
    fld.commit()
    tfo = d.create("transferFunction1D")
    tfo.commit()
    vol = d.create("volume")
    vol.set_param("field", fld)
    vol.set_param("transferFunction", tfo)
    vol.commit()
    world = d.create("world")
    world.set_param("volumes", [vol])
    world.commit()
    f = blob_field((48, 48, 48))
    c = auto_camera(f.bounds(), 64, 48)
    cam = d.create("camera")
    cam.set_param("position", c.position)
    cam.set_param("direction", c.view_dir)
    cam.set_param("aspect", 64 / 48)
    cam.commit()
    rend = d.create("renderer")
    rend.commit()
    frame = d.create("frame")
    frame.set_param("world", world)
    frame.set_param("camera", cam)
    frame.set_param("renderer", rend)
    frame.set_param("size", (64, 48))
    frame.commit()
    frame.render()
    r1 = api.map_frame(frame)
    frame.render()
    with pytest.raises(UsageError, match="invalidated"):
        _ = r1.pixels  # never materialised, then invalidated by the next render
    r2 = api.map_frame(frame)
    arr = r2.array.copy()
    assert arr.shape == (48, 64, 3)
    b2 = r2.pixels
    assert b2 == arr.tobytes()
    frame.render()
    assert api.map_frame(frame).pixels == b2  # same committed state, same bytes
    with pytest.raises(UsageError, match="invalidated"):
        _ = r2.pixels  # materialised bytes follow the reference rule too: valid until the next render
    frame.wait()


def test_run_collective_maps_ranks_onto_a_device_list(cuda_device):
    from paper_2501_01628_b200.transport import run_collective

    res = run_collective(4, lambda ep: (ep.rank, str(ep.device), torch.cuda.current_device()),
                         device=[cuda_device, cuda_device])
    assert [r[0] for r in res] == [0, 1, 2, 3]
    assert all(r[1] == str(cuda_device) for r in res)


def _bench(args, timeout=900):
    env = dict(os.environ)
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=str(ROOT))
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_launches_its_own_ranks():
    """``bench.py --gpus 2`` without a launcher runs two ranks (torch.distributed.run on 127.0.0.1); on a
    one-GPU box they share it over gloo and the line says it is not a measurement."""
    line = _bench(["--gpus", "2", "--config", "c1", "--steps", "3", "--warmup", "3", "--no-traffic",
                   "--no-cpu-baseline", "--no-extras"])
    assert line["n_gpus"] == 2 and line["config"]["bricks"] == 2
    if torch.cuda.device_count() < 2:
        assert line["measurement"] is False and line["backend"] == "gloo"
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["api_e2e"]["value"] > 0
    assert line["compositor_roofline"]["fragment_bytes_per_rank"] > 0


def test_bench_compositing_sweep_single_gpu():
    line = _bench(["--config", "c5", "--steps", "3", "--warmup", "3"])
    assert line["n_gpus"] == 1 and len(line["sweep"]) == 3 and line["value"] > 0


@pytest.mark.parametrize("seed", [3, 11])
def test_skipping_is_bit_exact_in_every_octant(cuda_device, seed):
    """Exact empty-space skipping (per-lane probe loop, one-sided octant distances, branch-free cube exits)
    drops only samples whose weight is exactly 0, and the contributing samples are evaluated the same way
    either way -- so the RGBA partial with skipping is BIT-identical to the one without, for cameras in all
    eight direction octants, an axis-aligned camera (zero direction components) and a camera inside the
    brick, with a sparse TF (threshold 0.3) and both marcher configurations."""
    import math

    from paper_2501_01628_b200.geom import CameraSpec, orbit_camera

    f = blob_field((81, 70, 63), seed=seed, spacing=(1.0, 1.0, 1.5))
    W, H = 112, 90
    bb = f.bounds()
    cams = [orbit_camera(bb.center(), 1.4 * bb.diagonal(), math.radians(yaw), math.radians(pitch), 40.0, W / H)
            for yaw in (35.0, 125.0, 215.0, 305.0) for pitch in (-30.0, 30.0)]
    c = bb.center()
    cams.append(CameraSpec((c[0], c[1], c[2] + 2.0 * bb.diagonal()), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), 50.0, W / H))
    cams.append(CameraSpec(tuple(c), (0.3, -0.2, 0.9), (0.0, 1.0, 0.0), 70.0, W / H))
    dtf = dev.DeviceTF(default_tf(threshold=0.3), cuda_device)
    for P in (1, 3):
        dec = decompose(f, P)
        for r in range(P):
            b = dev.DeviceBrick(dec.brick(r), cuda_device).generate(f)
            for cam in cams:
                for deep in (False, True):
                    a = torch.empty(W * H * 4, dtype=torch.float32, device=cuda_device)
                    n = torch.empty_like(a)
                    dev.march(b, cam, dtf, 0.7, 0.99, a, W, H, skip=True, force_deep=deep)
                    dev.march(b, cam, dtf, 0.7, 0.99, n, W, H, skip=False, force_deep=deep)
                    assert torch.equal(a, n), (P, r, cam, deep)
            b.close()


def test_skip_cache_follows_alpha_support(cuda_device):
    """The bricks cache their skip distances per skip_key (alpha support + value range): an edit that only
    scales opacities or recolours keeps the key (no rebuild) and a support change gets a new one; in every
    case the frame equals a fresh renderer's frame for the new TF, byte for byte."""
    from paper_2501_01628_b200.device import skip_key
    from paper_2501_01628_b200.engine import VolumeRenderer
    from paper_2501_01628_b200.transport import SoloEndpoint
    from paper_2501_01628_b200.volume import TransferFunction1D

    f = blob_field((90, 80, 70), seed=8)
    dec = decompose(f, 1)
    W, H = 200, 150
    cam = auto_camera(f.bounds(), W, H)
    base = default_tf()
    t = base.as_f32().copy()
    scaled = TransferFunction1D(np.column_stack([t[:, :3][:, ::-1], 0.5 * t[:, 3]]).astype(np.float32), base.vmin,
                                base.vmax)
    shifted = default_tf(threshold=0.35)
    assert skip_key(scaled) == skip_key(base) != skip_key(shifted)
    b = dev.DeviceBrick(dec.brick(0), cuda_device).generate(f)
    r = VolumeRenderer(SoloEndpoint(cuda_device), b, dec, base, (0.1, 0.1, 0.1))
    r.render(cam, W, H)
    for tf in (scaled, shifted, base):
        r.dtf.update(tf)
        r.tf = tf
        got = r.render(cam, W, H).rgb8.clone()
        fresh = VolumeRenderer(SoloEndpoint(cuda_device), b, dec, tf, (0.1, 0.1, 0.1))
        fresh.dtf.version = 0  # tf_version 0: rebuild the skip distances on this call
        want = fresh.render(cam, W, H).rgb8
        assert torch.equal(got, want)
    torch.cuda.synchronize()
    b.close()
