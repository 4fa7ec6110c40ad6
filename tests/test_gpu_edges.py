"""Edge cases of the marcher against the oracle: camera inside a brick, axis-parallel rays (zero direction
components), fully transparent and fully opaque transfer functions, odd frame sizes smaller than a
tile, ghost widths 0 and 2, anisotropic spacing with a shifted origin, dt != 1, a value range other than
[0, 1], the smallest and largest TF tables, and both marchers (beam and ray queue)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.geom import CameraSpec, auto_camera
from paper_2501_01628_b200.volume import TransferFunction1D, blob_field, decompose, default_tf
from scenes import RGBA_ATOL, cam_array, dense_tf, oracle_brick

pytestmark = pytest.mark.gpu


def _run(f, P, cam, tf, W, H, device, dt=1.0, ert=0.99, ghost=1, marcher=None, monkeypatch=None):
    if marcher is not None:
        monkeypatch.setenv("DPRT_MARCHER", marcher)
    vox = oracle.generate_field(f.dims, f.blobs)
    dec = decompose(f, P)
    dtf = dev.DeviceTF(tf, device)
    for r in range(P):
        desc = dec.brick(r, ghost)
        b = dev.DeviceBrick(desc, device).generate(f)
        p = torch.empty(W * H * 4, dtype=torch.float32, device=device)
        s = torch.empty(W * H, dtype=torch.int32, device=device)
        dev.march(b, cam, dtf, dt, ert, p, W, H, samples=s)
        torch.cuda.synchronize()
        ob = oracle_brick(dec, r, ghost)
        ref, rs = oracle.render_brick(ob.extract(vox), ob, cam_array(cam), tf.as_f32(), tf.vmin, tf.vmax, dt, ert, W, H)
        got = p.view(H, W, 4).cpu().numpy().astype(np.float64)
        assert np.array_equal(s.view(H, W).cpu().numpy().astype(np.uint32), rs), f"brick {r}: ownership"
        err = np.abs(got - ref).max()
        assert err <= RGBA_ATOL, f"brick {r}: max |dRGBA| {err:.3e}"
        b.close()
    return True


@pytest.mark.parametrize("marcher", ["beam", "queue"])
def test_camera_inside_a_brick(cuda_device, oracle_lib, monkeypatch, marcher):
    f = blob_field((40, 36, 32), seed=4)
    cam = CameraSpec((20.0, 17.5, 15.0), (0.3, -0.2, -1.0), (0.0, 1.0, 0.0), 90.0, 1.3)
    _run(f, 2, cam, dense_tf(), 65, 50, cuda_device, marcher=marcher, monkeypatch=monkeypatch)


@pytest.mark.parametrize("marcher", ["beam", "queue"])
def test_axis_parallel_rays(cuda_device, oracle_lib, monkeypatch, marcher):
    """Exactly axis-aligned view: the centre rays have zero x and y direction components."""
    f = blob_field((33, 33, 33), seed=5)
    cam = CameraSpec((16.0, 16.0, 80.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), 30.0, 1.0)
    _run(f, 4, cam, dense_tf(), 33, 33, cuda_device, marcher=marcher, monkeypatch=monkeypatch)


def test_transparent_and_opaque_transfer_functions(cuda_device, oracle_lib):
    f = blob_field((30, 30, 30), seed=6)
    cam = auto_camera(f.bounds(), 40, 40)
    clear = TransferFunction1D(np.zeros((8, 4), np.float32), 0.0, 1.0)
    _run(f, 2, cam, clear, 40, 40, cuda_device)
    opaque = TransferFunction1D(np.tile(np.array([[0.2, 0.4, 0.6, 1.0]], np.float32), (4, 1)), 0.0, 1.0)
    _run(f, 2, cam, opaque, 40, 40, cuda_device)


@pytest.mark.parametrize("W,H", [(1, 1), (7, 3), (17, 9), (33, 5)])
def test_odd_small_frames(cuda_device, oracle_lib, W, H):
    f = blob_field((24, 20, 18), seed=7)
    _run(f, 2, auto_camera(f.bounds(), W, H), dense_tf(), W, H, cuda_device)


@pytest.mark.parametrize("ghost", [0, 2])
def test_ghost_widths(cuda_device, oracle_lib, ghost):
    f = blob_field((34, 30, 28), seed=8)
    _run(f, 3, auto_camera(f.bounds(), 48, 40), dense_tf(), 48, 40, cuda_device, ghost=ghost)


def test_anisotropic_spacing_origin_dt_and_value_range(cuda_device, oracle_lib):
    f = blob_field((36, 28, 20), seed=9, spacing=(0.5, 0.75, 1.5), origin=(-3.0, 2.0, 10.0))
    t = dense_tf().as_f32()
    tf = TransferFunction1D(t, -0.25, 1.5)
    _run(f, 4, auto_camera(f.bounds(), 56, 44), tf, 56, 44, cuda_device, dt=0.37, ert=0.9)


@pytest.mark.parametrize("n", [2, 1024])
def test_table_sizes(cuda_device, oracle_lib, n):
    x = np.linspace(0, 1, n)
    t = np.column_stack([x, 1 - x, 0.5 * np.ones(n), np.where(x < 0.2, 0.0, 0.1 * x)]).astype(np.float32)
    f = blob_field((26, 26, 26), seed=10)
    _run(f, 2, auto_camera(f.bounds(), 32, 32), TransferFunction1D(t, 0.0, 1.0), 32, 32, cuda_device)
