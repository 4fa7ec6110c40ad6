"""GPU triangle traversal (csrc/trace.cu, trace.py) against the REFERENCE's own numba slot.

* golden vectors made by running the reference (tests/golden/make_trace_golden.py): every ray's
  (best_t, best_id) -- as float64 bits -- and every shadow ray's occlusion bit equal the reference's
  trace_nearest_batch / trace_any_batch outputs exactly, incl. preset cross-rank minima and exact ties;
* the host drop-in functions (same signature as bvh.py:284-311) give the same bytes;
* device-resident ray cycling over R rank threads (cycle_batch_device, engine.py:282-310's shape) ends with
  the all-rank minimum the reference reduces to;
* the reference's whole triangle renderer, installed unmodified in baseline/_ref, renders bit-identical
  frames with its traversal slot switched to the GPU (skipped when that install is absent).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2501_01628_b200 import trace
from paper_2501_01628_b200.errors import UsageError

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden" / "trace_vectors.npz"
ROOT = Path(__file__).resolve().parent.parent
ACC = ("node_lo", "node_hi", "node_left", "node_right", "node_first", "node_count")


@pytest.fixture(scope="module")
def gold():
    with np.load(GOLD) as z:  # materialised: NpzFile members decompress lazily and are not thread-safe
        return {k: z[k] for k in z.files}


def _scenes(g):
    for s in (0, 1):
        yield s, int(g[f"s{s}_R"])


def _accel_args(g, s, r):
    return [g[f"s{s}_r{r}_{k}"] for k in ACC] + [int(g[f"s{s}_r{r}_root"]), g[f"s{s}_r{r}_tri_v"], g[f"s{s}_r{r}_tri_id"]]


def _dev(a, d):
    return torch.from_numpy(np.ascontiguousarray(a)).to(d)


def test_nearest_and_any_match_reference_bits(cuda_device, gold):
    g = gold
    for s, R in _scenes(g):
        org, dirn, tmin, tmax = (_dev(g[f"s{s}_{k}"], cuda_device) for k in ("org", "dirn", "tmin", "tmax"))
        for r in range(R):
            b = trace.DeviceBvh(*_accel_args(g, s, r), device=cuda_device)
            bt, bi = _dev(g[f"s{s}_r{r}_in_best_t"], cuda_device), _dev(g[f"s{s}_r{r}_in_best_id"], cuda_device)
            b.trace_nearest(org, dirn, tmin, tmax, bt, bi)
            assert np.array_equal(bt.cpu().numpy().view(np.uint64), g[f"s{s}_r{r}_out_best_t"].view(np.uint64))
            assert np.array_equal(bi.cpu().numpy(), g[f"s{s}_r{r}_out_best_id"])
            # exact ties against a preset larger id: the lower id wins, t bits unchanged
            bt2 = _dev(g[f"s{s}_r{r}_out_best_t"], cuda_device)
            bi2 = _dev(g[f"s{s}_r{r}_tie_in_id"], cuda_device)
            b.trace_nearest(org, dirn, tmin, tmax, bt2, bi2)
            assert np.array_equal(bt2.cpu().numpy().view(np.uint64), g[f"s{s}_r{r}_tie_out_t"].view(np.uint64))
            assert np.array_equal(bi2.cpu().numpy(), g[f"s{s}_r{r}_tie_out_id"])
            so, sd, s0, s1 = (_dev(g[f"s{s}_r{r}_{k}"], cuda_device) for k in ("s_org", "s_dir", "s_tmin", "s_tmax"))
            occ = _dev(g[f"s{s}_r{r}_occ_in"], cuda_device)
            b.trace_any(so, sd, s0, s1, occ)
            assert np.array_equal(occ.cpu().numpy(), g[f"s{s}_r{r}_occ_out"])


def test_host_dropin_signature_matches_reference(cuda_device, gold):
    g = gold
    s, r = 1, 2
    args = _accel_args(g, s, r)
    org, dirn, tmin, tmax = (g[f"s{s}_{k}"] for k in ("org", "dirn", "tmin", "tmax"))
    bt, bi = g[f"s{s}_r{r}_in_best_t"].copy(), g[f"s{s}_r{r}_in_best_id"].copy()
    trace.trace_nearest_batch(*args, org, dirn, tmin, tmax, bt, bi)
    assert np.array_equal(bt.view(np.uint64), g[f"s{s}_r{r}_out_best_t"].view(np.uint64))
    assert np.array_equal(bi, g[f"s{s}_r{r}_out_best_id"])
    occ = g[f"s{s}_r{r}_occ_in"].copy()
    trace.trace_any_batch(*args, g[f"s{s}_r{r}_s_org"], g[f"s{s}_r{r}_s_dir"], g[f"s{s}_r{r}_s_tmin"],
                          g[f"s{s}_r{r}_s_tmax"], occ)
    assert np.array_equal(occ, g[f"s{s}_r{r}_occ_out"])


def test_empty_bvh_and_argument_checks(cuda_device):
    z3 = np.zeros((0, 3))
    zi = np.zeros(0, np.int64)
    b = trace.DeviceBvh(z3, z3, zi, zi, zi, zi, -1, np.zeros((0, 9)), zi, device=cuda_device)
    n = 5
    org = torch.zeros((n, 3), dtype=torch.float64, device=cuda_device)
    dirn = torch.ones((n, 3), dtype=torch.float64, device=cuda_device)
    t0 = torch.zeros(n, dtype=torch.float64, device=cuda_device)
    t1 = torch.full((n,), float("inf"), dtype=torch.float64, device=cuda_device)
    bt = torch.full((n,), 7.0, dtype=torch.float64, device=cuda_device)
    bi = torch.full((n,), 3, dtype=torch.int64, device=cuda_device)
    b.trace_nearest(org, dirn, t0, t1, bt, bi)  # nothing to hit: the preset stays
    assert torch.all(bt == 7.0) and torch.all(bi == 3)
    with pytest.raises(UsageError):
        b.trace_nearest(org, dirn, t0, t1, bt.float(), bi)


@pytest.mark.parametrize("s", [0, 1])
def test_device_ray_cycling_reaches_the_all_rank_minimum(cuda_device, gold, s):
    from paper_2501_01628_b200.transport import run_collective

    g = gold
    R = int(g[f"s{s}_R"])
    org, dirn, tmin, tmax = (g[f"s{s}_{k}"] for k in ("org", "dirn", "tmin", "tmax"))
    N = org.shape[0]
    want_t, want_id = g[f"s{s}_r{R - 1}_out_best_t"], g[f"s{s}_r{R - 1}_out_best_id"]
    chunks = [(r * N // R, (r + 1) * N // R) for r in range(R)]

    def body(ep):
        b = trace.DeviceBvh(*_accel_args(g, s, ep.rank), device=cuda_device)
        a, z = chunks[ep.rank]
        n = z - a
        batch = trace.DeviceRayBatch.from_host(0, org[a:z], dirn[a:z], tmin[a:z], tmax[a:z], np.full(n, np.inf),
                                               np.full(n, trace.MISS_ID, np.int64), np.zeros(n, np.uint8),
                                               cuda_device, owner=ep.rank)
        home = trace.cycle_batch_device(ep, batch, b)
        t, i, _ = home.results()
        return ep.rank, t, i

    for rank, t, i in run_collective(R, body, device=cuda_device):
        a, z = chunks[rank]
        assert np.array_equal(t.view(np.uint64), want_t[a:z].view(np.uint64))
        assert np.array_equal(i, want_id[a:z])


def _ref_module():
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "dprt").exists():
        pytest.skip("reference install baseline/_ref absent")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/dprt_numba_cache")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import dprt  # noqa: F401
    from dprt import cli, engine, scene, transport

    return cli, engine, scene, transport


@pytest.mark.parametrize("R", [1, 2, 3])
def test_reference_renderer_with_gpu_traversal_is_bit_identical(cuda_device, R):
    """The unmodified reference renderer (engine.render_frame: digest, primary / shadow / reflection waves,
    ray cycling over R rank threads, gather) with its traversal slot on the GPU: the same image bits."""
    cli, engine, scene, transport = _ref_module()
    sc = scene.generate_uneven_cloud(5, 4000, 4)
    part = scene.partition_scene(sc, R, "spatialSlab")
    W, H = 64, 48
    cam = cli.default_camera(sc, W, H)

    def render():
        res = transport.run_collective(R, lambda ep: engine.render_frame(ep, sc, part, cam, W, H))
        return res[0].image

    ref_img = render()
    saved = engine.trace_nearest_batch, engine.trace_any_batch
    try:
        torch.cuda.set_device(cuda_device)
        engine.trace_nearest_batch, engine.trace_any_batch = trace.trace_nearest_batch, trace.trace_any_batch
        gpu_img = render()
    finally:
        engine.trace_nearest_batch, engine.trace_any_batch = saved
    assert ref_img.shape == (H, W, 3)
    assert np.array_equal(np.asarray(gpu_img).view(np.uint64), np.asarray(ref_img).view(np.uint64))
