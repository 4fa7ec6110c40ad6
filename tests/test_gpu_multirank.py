"""Multi-rank sort-last frames on ONE GPU: R rank threads in one process (the reference's run_collective
+ inproc model, transport.py:519-566), each marching its own brick and compositing through the real
exchange schedule (direct-send / binary-swap by device copies, p2p by plain peer pointers).  The frame on
rank 0 is compared with the oracle; sample ownership per rank exactly."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.api import Device, map_frame
from paper_2501_01628_b200.engine import RenderOptions, VolumeRenderer
from paper_2501_01628_b200.transport import run_collective
from scenes import RGB8_MAX_LSB, RGBA_ATOL, c1, oracle_partials

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode,R", [("direct_send", 2), ("direct_send", 3), ("binary_swap", 4), ("p2p", 2),
                                    ("p2p", 4), ("binary_swap", 8), ("auto", 3), ("p2p", 8), ("direct_send", 8),
                                    ("cycle", 8)])
def test_sort_last_frame_matches_oracle(cuda_device, oracle_lib, mode, R):
    s = c1(P=R, W=160, H=122)
    vox = oracle.generate_field(s.field.dims, s.field.blobs)
    ref, rs = oracle_partials(vox, s.dec, s.cam, s.tf, s.dt, s.ert, s.W, s.H)
    order = s.dec.visibility_order(s.cam.position)
    img_ref = oracle.composite(ref, order, s.background)

    def body(ep):
        b = dev.DeviceBrick(s.dec.brick(ep.rank), cuda_device).generate(s.field)
        vr = VolumeRenderer(ep, b, s.dec, s.tf, s.background)
        out = []
        for frame in range(2):
            res = vr.render(s.cam, s.W, s.H, RenderOptions(composite=mode, keep_float=True, collect_samples=True,
                                                           frame_index=frame))
            torch.cuda.synchronize()
            samples = res.samples.cpu().numpy().astype(np.uint32)
            out.append((res.image, None if res.rgb8 is None else res.rgb8.cpu().numpy(), samples, res.order))
        if mode == "auto":  # same process, one GPU: the peer mapping succeeds, so auto picks the fused path
            assert vr.compositor.mode == "p2p"
        return out

    results = run_collective(R, body, device=cuda_device)
    for r in range(R):
        for image, rgb8, samples, got_order in results[r]:
            assert np.array_equal(samples, rs[r])
            assert got_order == order
            if r == 0:
                assert np.abs(image - img_ref).max() <= RGBA_ATOL
                q = rgb8.astype(np.int16) - oracle.tone_map_rgb8(img_ref).astype(np.int16)
                assert np.abs(q).max() <= RGB8_MAX_LSB
            else:
                assert image is None and rgb8 is None


@pytest.mark.parametrize("mode,R,W,H", [("direct_send", 4, 176, 130), ("p2p", 3, 176, 130),
                                        ("binary_swap", 2, 176, 130), ("direct_send", 3, 157, 113),
                                        ("p2p", 4, 157, 113)])
def test_band_clipped_exchange_is_bit_identical(cuda_device, mode, R, W, H):
    """clip_exchange (only footprint rows move, partials cleared only inside their bands) changes the
    bytes exchanged, never the frame: RGB8 and float frames equal the unclipped exchange bit for bit
    (odd widths put fragment range edges inside the composite kernel's 4-pixel groups)."""
    s = c1(P=R, W=W, H=H)

    def body(ep):
        b = dev.DeviceBrick(s.dec.brick(ep.rank), cuda_device).generate(s.field)
        vr = VolumeRenderer(ep, b, s.dec, s.tf, s.background)
        out = []
        for clip in (False, True, False):
            res = vr.render(s.cam, s.W, s.H, RenderOptions(composite=mode, keep_float=True, clip_exchange=clip))
            torch.cuda.synchronize()
            out.append((None if res.rgb8 is None else res.rgb8.cpu().numpy(), res.image, res.stats.bytes_exchanged))
        return out

    res = run_collective(R, body, device=cuda_device)
    (a8, af, ab), (b8, bf, bb), (c8, cf, _) = res[0]
    assert np.array_equal(a8, b8) and np.array_equal(af, bf) and np.array_equal(a8, c8)
    if mode != "binary_swap":
        assert sum(r[1][2] for r in res) < sum(r[0][2] for r in res)


def _narrow_cameras(s, W, H):
    """Axis-parallel narrow views down one corner column of the field (bricks away from it have no screen
    footprint) and a wide view from inside a brick."""
    import math

    from paper_2501_01628_b200.geom import CameraSpec

    lo, hi = s.field.bounds().lo, s.field.bounds().hi

    def at(fx, fy, fz):
        return tuple(lo[i] + f * (hi[i] - lo[i]) for i, f in enumerate((fx, fy, fz)))

    def look(pos, tgt, fov):
        v = tuple(t - p for t, p in zip(tgt, pos))
        n = math.sqrt(sum(c * c for c in v))
        return CameraSpec(pos, tuple(c / n for c in v), (0.0, 1.0, 0.0), fov, W / H)

    return [look(at(0.1, 0.1, -1.5), at(0.1, 0.1, 0.5), 10.0), look(at(-1.5, 0.9, 0.85), at(0.5, 0.9, 0.85), 6.0),
            look(at(0.3, 0.3, 0.3), s.field.bounds().center(), 60.0)]


@pytest.mark.parametrize("mode,R", [("direct_send", 4), ("p2p", 4), ("binary_swap", 4), ("cycle", 4),
                                    ("direct_send", 8), ("p2p", 8), ("binary_swap", 8)])
def test_frames_with_offscreen_bricks_match_oracle(cuda_device, oracle_lib, mode, R):
    """Every exchange schedule when some bricks project nowhere on screen (empty footprints: no rows to
    send, fragments that are clear everywhere, row blocks blending only background) and with the eye inside
    a brick: rank 0's frame against the oracle composite, sample ownership exact on every rank."""
    W, H = 150, 110
    s = c1(P=R, W=W, H=H)
    cams = _narrow_cameras(s, W, H)
    assert any(dev.desc_footprint(s.dec.brick(r), cams[0], W, H)[3] <= dev.desc_footprint(s.dec.brick(r), cams[0], W, H)[1]
               for r in range(R))
    vox = oracle.generate_field(s.field.dims, s.field.blobs)
    refs = []
    for cam in cams:
        ref, rs = oracle_partials(vox, s.dec, cam, s.tf, s.dt, s.ert, W, H)
        order = s.dec.visibility_order(cam.position)
        refs.append((oracle.composite(ref, order, s.background), rs, order))

    def body(ep):
        b = dev.DeviceBrick(s.dec.brick(ep.rank), cuda_device).generate(s.field)
        vr = VolumeRenderer(ep, b, s.dec, s.tf, s.background)
        out = []
        for k, cam in enumerate(cams):
            res = vr.render(cam, W, H, RenderOptions(composite=mode, keep_float=True, collect_samples=True,
                                                     frame_index=k))
            torch.cuda.synchronize()
            out.append((res.image, None if res.rgb8 is None else res.rgb8.cpu().numpy(),
                        res.samples.cpu().numpy().astype(np.uint32), res.order))
        return out

    results = run_collective(R, body, device=cuda_device)
    for k, (img_ref, rs, order) in enumerate(refs):
        for r in range(R):
            image, rgb8, samples, got_order = results[r][k]
            assert np.array_equal(samples, rs[r]), f"camera {k} rank {r} ownership"
            assert got_order == order
            if r == 0:
                assert np.abs(image - img_ref).max() <= RGBA_ATOL
                q = rgb8.astype(np.int16) - oracle.tone_map_rgb8(img_ref).astype(np.int16)
                assert np.abs(q).max() <= RGB8_MAX_LSB


def test_disable_compositing_shows_only_root_brick(cuda_device, oracle_lib):
    """Negative test (engine.py:172 analog): without compositing the frame is rank 0's brick alone."""
    s = c1(P=2, W=96, H=96)
    vox = oracle.generate_field(s.field.dims, s.field.blobs)
    ref, _ = oracle_partials(vox, s.dec, s.cam, s.tf, s.dt, s.ert, s.W, s.H)
    order = s.dec.visibility_order(s.cam.position)

    def body(ep):
        b = dev.DeviceBrick(s.dec.brick(ep.rank), cuda_device).generate(s.field)
        res = VolumeRenderer(ep, b, s.dec, s.tf, s.background).render(
            s.cam, s.W, s.H, RenderOptions(disable_compositing=True, keep_float=True))
        torch.cuda.synchronize()
        return res.image

    img = run_collective(2, body, device=cuda_device)[0]
    solo = oracle.composite(ref, [0], s.background)
    full = oracle.composite(ref, order, s.background)
    assert np.abs(img - solo).max() <= RGBA_ATOL
    assert np.abs(img - full).max() > 0.01


def _api_frame(ep, cuda_device, W, H, composite="auto", fov=45.0):
    d = Device(ep, cuda_device)
    sf = d.create("spatialField")
    sf.set_param("dims", (64, 64, 64))
    sf.commit()
    tf = d.create("transferFunction1D")
    tf.commit()
    vol = d.create("volume")
    vol.set_param("field", sf)
    vol.set_param("transferFunction", tf)
    vol.commit()
    world = d.create("world")
    world.set_param("volumes", [vol])
    world.commit()
    from paper_2501_01628_b200.geom import auto_camera

    c = auto_camera(world.decomposition.field.bounds(), W, H)
    cam = d.create("camera")
    cam.set_param("position", c.position)
    cam.set_param("direction", c.view_dir)
    cam.set_param("fovY", fov)
    cam.set_param("aspect", W / H)
    cam.commit()
    rend = d.create("renderer")
    rend.set_param("background", (0.05, 0.06, 0.08))
    rend.set_param("composite", composite)
    rend.commit()
    frame = d.create("frame")
    frame.set_param("world", world)
    frame.set_param("camera", cam)
    frame.set_param("renderer", rend)
    frame.set_param("size", (W, H))
    frame.commit()
    return frame, cam, world


@pytest.mark.parametrize("R,mode", [(1, "auto"), (2, "direct_send"), (4, "p2p")])
def test_api_frame_matches_oracle_and_staging(cuda_device, oracle_lib, R, mode):
    """Device/World/Frame -> render_frame_collective -> map_frame (api.py:329-371) on R rank threads."""
    W, H = 96, 72

    def body(ep):
        frame, cam, world = _api_frame(ep, cuda_device, W, H, mode)
        frame.render()
        first = map_frame(frame)
        pix1 = first.pixels if ep.rank == 0 else None
        cam.set_param("fovY", 60.0)  # staged only
        frame.render()
        pix2 = map_frame(frame).pixels if ep.rank == 0 else None
        stale = first.valid if ep.rank == 0 else None
        cam.commit()
        frame.render()
        pix3 = map_frame(frame).pixels if ep.rank == 0 else None
        return pix1, pix2, pix3, stale, world.decomposition.boxes

    res = run_collective(R, body, device=cuda_device)
    pix1, pix2, pix3, stale, boxes = res[0]
    assert pix1 == pix2 and pix1 != pix3 and stale is False
    # frame 1 against the oracle
    from paper_2501_01628_b200.geom import auto_camera
    from paper_2501_01628_b200.volume import blob_field, decompose, default_tf

    f = blob_field((64, 64, 64))
    dec = decompose(f, R)
    assert dec.boxes == boxes
    c = auto_camera(f.bounds(), W, H)
    from paper_2501_01628_b200.geom import CameraSpec

    cam = CameraSpec(c.position, c.view_dir, (0.0, 1.0, 0.0), 45.0, W / H)
    vox = oracle.generate_field(f.dims, f.blobs)
    ref, _ = oracle_partials(vox, dec, cam, default_tf(), 1.0, 0.99, W, H)
    want = oracle.tone_map_rgb8(oracle.composite(ref, dec.visibility_order(cam.position), (0.05, 0.06, 0.08)))
    got = np.frombuffer(pix1, np.uint8).reshape(H, W, 3)
    assert np.abs(got.astype(np.int16) - want.astype(np.int16)).max() <= RGB8_MAX_LSB


def test_rankcolor_mode_shows_brick_ownership(cuda_device, oracle_lib):
    """engine.py:327-332 analog: each rank's visible data drawn opaque in RANK_PALETTE[rank]; the frame
    matches the oracle composite of the same rank-colour TFs and every rank's colour appears."""
    from paper_2501_01628_b200.engine import RANK_PALETTE, rankcolor_tf

    s = c1(P=3, W=120, H=96)
    vox = oracle.generate_field(s.field.dims, s.field.blobs)
    order = s.dec.visibility_order(s.cam.position)
    refs = []
    for r in range(3):
        t = rankcolor_tf(s.tf, r)
        ob = __import__("scenes").oracle_brick(s.dec, r)
        rgba, _ = oracle.render_brick(ob.extract(vox), ob, __import__("scenes").cam_array(s.cam), t.as_f32(),
                                      t.vmin, t.vmax, 1.0, 0.99, s.W, s.H)
        refs.append(rgba)
    want = oracle.composite(refs, order, s.background)

    def body(ep):
        b = dev.DeviceBrick(s.dec.brick(ep.rank), cuda_device).generate(s.field)
        res = VolumeRenderer(ep, b, s.dec, s.tf, s.background).render(
            s.cam, s.W, s.H, RenderOptions(mode="rankcolor", keep_float=True))
        torch.cuda.synchronize()
        return res.image

    img = run_collective(3, body, device=cuda_device)[0]
    assert np.abs(img - want).max() <= RGBA_ATOL
    flat = img.reshape(-1, 3)
    for r in range(3):
        assert np.any(np.all(np.abs(flat - RANK_PALETTE[r]) < 1e-6, axis=1)), f"rank {r} colour missing"


@pytest.mark.parametrize("R", [2, 3, 4])
def test_ray_cycling_matches_oracle(cuda_device, oracle_lib, R):
    """composite='cycle' (ray batches hop along the visibility order, ERT on accumulated opacity) against
    the oracle's serial restatement of the same schedule; ownership counts exact; with ERT out of reach
    the cycled frame equals the sort-last frame."""
    from paper_2501_01628_b200.compositor import assign_rows
    from scenes import cam_array, dense_tf, oracle_brick

    s = c1(P=R, W=150, H=118)
    vox = oracle.generate_field(s.field.dims, s.field.blobs)
    bricks = [oracle_brick(s.dec, r) for r in range(R)]
    bv = [b.extract(vox) for b in bricks]
    order = s.dec.visibility_order(s.cam.position)
    _, rs = oracle_partials(vox, s.dec, s.cam, s.tf, s.dt, s.ert, s.W, s.H)

    def body(ep):
        b = dev.DeviceBrick(s.dec.brick(ep.rank), cuda_device).generate(s.field)
        vr = VolumeRenderer(ep, b, s.dec, s.tf, s.background)
        outs = []
        for tf, ert, mode in ((s.tf, s.ert, "cycle"), (dense_tf(), s.ert, "cycle"), (s.tf, 2.0, "cycle"),
                              (s.tf, 2.0, "direct_send")):
            vr.set_tf(tf)
            res = vr.render(s.cam, s.W, s.H, RenderOptions(composite=mode, ert=ert, keep_float=True,
                                                           collect_samples=True))
            torch.cuda.synchronize()
            outs.append((res.image, None if res.rgb8 is None else res.rgb8.cpu().numpy(),
                         res.samples.cpu().numpy().astype(np.uint32)))
        return outs

    res = run_collective(R, body, device=cuda_device)
    for r in range(R):
        assert np.array_equal(res[r][0][2], rs[r]), f"rank {r}: ownership in cycle mode"
    for i, (tf, ert) in enumerate(((s.tf, s.ert), (dense_tf(), s.ert), (s.tf, 2.0))):
        want = oracle.cycle_frame(bv, bricks, order, assign_rows(s.H, R), cam_array(s.cam), tf.as_f32(), tf.vmin,
                                  tf.vmax, s.dt, ert, s.W, s.H, s.background)
        image, rgb8, _ = res[0][i]
        assert np.abs(image - want).max() <= RGBA_ATOL, f"case {i}"
        q = rgb8.astype(np.int16) - oracle.tone_map_rgb8(want).astype(np.int16)
        assert np.abs(q).max() <= RGB8_MAX_LSB
    assert np.abs(res[0][2][0] - res[0][3][0]).max() < 1e-5  # no ERT: cycling == sort-last


@pytest.mark.parametrize("mode,R", [("direct_send", 2), ("p2p", 4), ("auto", 3)])
def test_fp16_fragment_frames(cuda_device, oracle_lib, mode, R):
    """fragment_dtype='f16' halves the exchanged bytes; the frame stays within the fp16 tolerance of the
    oracle (RGBA_ATOL_F16: each fragment channel carries <= 2^-12 relative rounding; RGB8 within 2 LSB)."""
    from scenes import RGBA_ATOL_F16

    s = c1(P=R, W=144, H=104)
    vox = oracle.generate_field(s.field.dims, s.field.blobs)
    ref, _ = oracle_partials(vox, s.dec, s.cam, s.tf, s.dt, s.ert, s.W, s.H)
    want = oracle.composite(ref, s.dec.visibility_order(s.cam.position), s.background)

    def body(ep):
        b = dev.DeviceBrick(s.dec.brick(ep.rank), cuda_device).generate(s.field)
        vr = VolumeRenderer(ep, b, s.dec, s.tf, s.background)
        out = []
        for fdt in ("f16", "f32"):
            res = vr.render(s.cam, s.W, s.H, RenderOptions(composite=mode, keep_float=True, fragment_dtype=fdt))
            torch.cuda.synchronize()
            out.append((res.image, None if res.rgb8 is None else res.rgb8.cpu().numpy(), res.stats.bytes_exchanged))
        return out

    res = run_collective(R, body, device=cuda_device)
    (img16, rgb16, _), (img32, _, _) = res[0]
    assert np.abs(img16 - want).max() <= RGBA_ATOL_F16
    assert np.abs(rgb16.astype(np.int16) - oracle.tone_map_rgb8(want).astype(np.int16)).max() <= 2
    assert np.abs(img16 - img32).max() <= RGBA_ATOL_F16
    assert sum(r[0][2] for r in res) < sum(r[1][2] for r in res)
