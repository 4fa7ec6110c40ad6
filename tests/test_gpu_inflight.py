"""Frames in flight (RenderOptions.frames_in_flight): single-rank frames marched on lane
streams overlap each other; every frame must still be byte-identical to the stream-ordered render of the
same inputs, including across TF updates (staged and plain), brick rewrites and camera changes."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.engine import RenderOptions, VolumeRenderer
from paper_2501_01628_b200.errors import UsageError
from paper_2501_01628_b200.geom import auto_camera, orbit_camera
from paper_2501_01628_b200.transport import SoloEndpoint
from paper_2501_01628_b200.volume import blob_field, decompose, default_tf
from scenes import RGB8_MAX_LSB, dense_tf, oracle_partials

pytestmark = pytest.mark.gpu

BG = (0.05, 0.06, 0.08)


def _script(f):
    """(camera, tf, staged, regenerate-with-seed) per frame: orbiting camera, TF switches every few frames
    (through the pinned staging path and the plain copy), one brick rewrite half way."""
    W, H = 640, 480
    b = f.bounds()
    tfs = [default_tf(), dense_tf(), default_tf(threshold=0.3)]
    steps = []
    for k in range(14):
        cam = orbit_camera(b.center(), 1.3 * b.diagonal(), np.radians(7.0 * k), np.radians(3.0 * (k % 4) + 10.0),
                           40.0, W / H)
        steps.append((cam, tfs[(k // 3) % 3], k % 2 == 0, 9 if k == 8 else None))
    return W, H, steps


def _run(device, f, frames_in_flight):
    W, H, steps = _script(f)
    dec = decompose(f, 1)
    brick = dev.DeviceBrick(dec.brick(0), device).generate(f)
    r = VolumeRenderer(SoloEndpoint(device), brick, dec, steps[0][1], BG)
    opts = RenderOptions(frames_in_flight=frames_in_flight)
    out, pending = [], []
    for cam, tf, staged, seed in steps:
        if seed is not None:
            brick.generate(blob_field(f.dims, seed=seed))
        if staged:
            r.dtf.update(tf, staging=torch.from_numpy(tf.as_f32().reshape(-1).copy()).pin_memory())
        else:
            r.dtf.update(tf)
        r.tf = tf
        host = torch.empty((H, W, 3), dtype=torch.uint8).pin_memory()
        pending.append(r.render_to_host(cam, W, H, host, opts, verify=False))
    for hf in pending:
        out.append(hf.wait().numpy().copy())
    r.join()
    torch.cuda.synchronize()
    brick.close()
    return out


@pytest.mark.parametrize("n", [2, 3])
def test_frames_in_flight_equal_ordered_frames(cuda_device, oracle_lib, n):
    f = blob_field((161, 145, 129), seed=4)
    want = _run(cuda_device, f, 1)
    got = _run(cuda_device, f, n)
    for k, (a, b) in enumerate(zip(got, want)):
        assert np.array_equal(a, b), f"frame {k} differs with {n} frames in flight"
    # and the first frame against the oracle (the ordered path's own parity is tested elsewhere)
    W, H, steps = _script(f)
    cam, tf = steps[0][0], steps[0][1]
    vox = oracle.generate_field(f.dims, f.blobs)
    ref, _ = oracle_partials(vox, decompose(f, 1), cam, tf, 1.0, 0.99, W, H)
    exp = oracle.tone_map_rgb8(oracle.composite(ref, [0], BG)).astype(np.int16)
    assert np.abs(got[0].astype(np.int16) - exp).max() <= RGB8_MAX_LSB


def test_frames_in_flight_device_result_and_join(cuda_device):
    """render() with frames in flight returns before the frame is complete; wait_ready / join order the
    current stream after it; the frame equals the ordered render."""
    f = blob_field((97, 97, 97), seed=2)
    dec = decompose(f, 1)
    W, H = 320, 240
    cam = auto_camera(f.bounds(), W, H)
    brick = dev.DeviceBrick(dec.brick(0), cuda_device).generate(f)
    r = VolumeRenderer(SoloEndpoint(cuda_device), brick, dec, default_tf(), BG)
    want = r.render(cam, W, H).rgb8.clone()
    res = [r.render(cam, W, H, RenderOptions(frames_in_flight=2)) for _ in range(4)]
    assert all(x.ready is not None for x in res)
    res[-1].wait_ready()
    assert torch.equal(res[-1].rgb8, want)
    r.join()
    for x in res:
        assert torch.equal(x.rgb8, want)
    # back to stream-ordered frames on the same renderer
    assert torch.equal(r.render(cam, W, H).rgb8, want)
    brick.close()


def test_frames_in_flight_argument_checks(cuda_device):
    f = blob_field((33, 33, 33), seed=1)
    dec = decompose(f, 1)
    brick = dev.DeviceBrick(dec.brick(0), cuda_device).generate(f)
    r = VolumeRenderer(SoloEndpoint(cuda_device), brick, dec, default_tf(), BG)
    cam = auto_camera(f.bounds(), 32, 32)
    for bad in (0, dev.MARCH_COUNTER_SLOTS):
        with pytest.raises(UsageError, match="frames_in_flight"):
            r.render(cam, 32, 32, RenderOptions(frames_in_flight=bad))
    frame = torch.empty(32 * 32 * 3, dtype=torch.uint8, device=cuda_device)
    with pytest.raises(UsageError, match="lane"):
        dev.march_rgb8(brick, cam, r.dtf, 1.0, 0.99, BG, frame, 32, 32, slot=1)
    with pytest.raises(UsageError, match="slot"):
        dev.march_rgb8(brick, cam, r.dtf, 1.0, 0.99, BG, frame, 32, 32, lane=torch.cuda.Stream(cuda_device), slot=0)
    brick.close()


@pytest.mark.parametrize("n", [1, 2])
def test_reused_host_buffers_get_whole_frames(cuda_device, n):
    """render_to_host into reused host buffers copies only the footprint rectangle (and the rectangles written
    since the last full copy) -- the rest already holds the background.  Across zooming / orbiting cameras
    whose rectangles grow, shrink and move, a background change and a camera inside the brick (full-frame
    rectangle), every host frame must equal the device frame byte for byte."""
    import math

    f = blob_field((97, 89, 81), seed=6)
    dec = decompose(f, 1)
    W, H = 320, 200
    brick = dev.DeviceBrick(dec.brick(0), cuda_device).generate(f)
    r = VolumeRenderer(SoloEndpoint(cuda_device), brick, dec, default_tf(), BG)
    bb = f.bounds()
    hosts = [torch.empty((H, W, 3), dtype=torch.uint8).pin_memory() for _ in range(2)]
    cams = [orbit_camera(bb.center(), (1.0 + 0.6 * (k % 4)) * bb.diagonal(), math.radians(23.0 * k),
                         math.radians(12.0), 40.0, W / H) for k in range(12)]
    cams.insert(6, orbit_camera(bb.center(), 0.2 * bb.diagonal(), 0.3, 0.1, 60.0, W / H))  # eye inside the brick
    for k, cam in enumerate(cams):
        if k == 8:
            r.background = (0.3, 0.2, 0.1)
        hf = r.render_to_host(cam, W, H, hosts[k % 2], RenderOptions(frames_in_flight=n), verify=False)
        got = hf.wait().numpy().copy()
        hf.result.wait_ready() if hf.result.ready is not None else None
        want = hf.result.rgb8.cpu().numpy()
        assert np.array_equal(got, want), f"frame {k}"
    r.join()
    brick.close()
