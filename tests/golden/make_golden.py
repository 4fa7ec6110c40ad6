"""Generate golden vectors by running the REFERENCE itself (arxiv/paper_2501_01628, package `dprt`).

Run in the build container only (the reference tree does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py [/root/reference]

Writes tests/golden/reference_vectors.npz and tests/golden/reference_4x3.ppm.  The vectors cover the
parts of the DVR path that the reference does implement, at the reference call sites the oracle and the
CUDA marcher restate:

  camera rays      engine.gen_primary_batch (engine.py:224-251) == geom.camera_primary_ray (geom.py:240-259)
  slab intervals   geom.ray_aabb_intersect (geom.py:171-200), incl. zero-direction and empty-box cases
  row ownership    engine.assign_pixels (engine.py:216-221)
  tone map         engine.tone_map_rgb8 (engine.py:500-502)
  PPM              ppm.encode_ppm (ppm.py:12-16)
  longest axis     geom.Aabb.longest_axis (geom.py:107-116)
  auto camera      cli.default_camera (cli.py:23-34)
  wire format      protocol.encode_message (protocol.py:196-209) for frame / camera / control messages
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference")
sys.path.insert(0, str(REF / "pkg" / "src"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")

from dprt import cli, engine, geom, ppm, protocol, transport  # noqa: E402
from dprt.scene import SceneDesc  # noqa: E402

OUT = Path(__file__).resolve().parent


def cameras():
    return [
        geom.CameraSpec((0.0, 0.0, 0.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), 90.0, 1.0),
        geom.CameraSpec((0.0, 0.0, 0.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), 37.0, 17.0 / 11.0),
        geom.CameraSpec((3.1, -2.2, 7.5), (-0.3, 0.25, -1.0), (0.0, 1.0, 0.0), 45.0, 1.5),
        geom.CameraSpec((100.5, 80.25, 140.0), (-0.5, -0.4, -0.75), (0.0, 1.0, 0.0), 30.0, 16.0 / 9.0),
    ]


def main() -> None:
    rng = np.random.default_rng(20250101)
    data = {}

    # --- camera rays via the reference's vectorised batch generator (1 rank owns every row)
    sizes = [(17, 11), (32, 32), (9, 9), (64, 36)]
    cam_params = []
    dirs = []
    for ci, cam in enumerate(cameras()):
        w, h = sizes[ci]
        [batch] = transport.run_collective(1, lambda ep, cam=cam, w=w, h=h: engine.gen_primary_batch(ep, cam, w, h))
        # the scalar path must agree bit for bit (test_engine.py:30-44 asserts the same)
        for pix in (0, w * h - 1, (w * h) // 2):
            ray = geom.camera_primary_ray(cam, pix % w, pix // w, w, h)
            assert tuple(batch.dirn[pix]) == ray.direction
        cam_params.append([*cam.position, *cam.view_dir, *cam.up, cam.fov_y, cam.aspect, w, h])
        dirs.append(batch.dirn.copy())
    data["cam_params"] = np.array(cam_params, np.float64)
    for i, d in enumerate(dirs):
        data[f"cam_dirs_{i}"] = d

    # --- slab intervals, including axis-parallel rays, origins on faces and the empty box
    n = 400
    o = rng.uniform(-3.0, 3.0, (n, 3))
    d = rng.normal(size=(n, 3))
    d[rng.random((n, 3)) < 0.15] = 0.0
    d[np.all(d == 0.0, axis=1), 0] = 1.0
    lo = rng.uniform(-1.5, 0.5, (n, 3))
    hi = lo + rng.uniform(0.0, 2.0, (n, 3))
    o[::7, 1] = lo[::7, 1]  # origin exactly on a face
    lo[::53] = np.inf  # empty boxes
    hi[::53] = -np.inf
    hit = np.zeros(n, np.uint8)
    t01 = np.zeros((n, 2))
    for i in range(n):
        r = geom.Ray(tuple(o[i]), tuple(d[i]))
        box = geom.Aabb(tuple(lo[i]), tuple(hi[i]))
        res = geom.ray_aabb_intersect(r, box)
        if res is not None:
            hit[i] = 1
            t01[i] = res
    data.update(slab_o=o, slab_d=d, slab_lo=lo, slab_hi=hi, slab_hit=hit, slab_t=t01)

    # --- row ownership
    cases = [(7, 4, 2), (7, 5, 2), (7, 5, 1), (3, 11, 4), (1920, 1080, 8), (3840, 2160, 8), (256, 256, 2),
             (7680, 4320, 4), (100, 7, 8), (5, 3, 3)]
    data["assign_cases"] = np.array(cases, np.int64)
    data["assign_rows"] = np.array(
        [r for (w, h, R) in cases for blk in engine.assign_pixels(w, h, R) for r in blk], np.int64)

    # --- tone map, with exact half-way ties
    img = rng.uniform(-0.2, 1.2, (7, 9, 3))
    img[0, :, 0] = (np.arange(9) + 0.5) / 255.0
    img[1, 0] = (0.0, 1.0, 0.5)
    data["tone_in"] = img
    data["tone_out"] = engine.tone_map_rgb8(img)

    # --- longest axis (ties go to the lowest axis)
    boxes = np.array([[0, 0, 0, 1, 1, 1], [0, 0, 0, 1, 2, 2], [0, 0, 0, 3, 2, 3], [0, 0, 0, 1, 2, 3],
                      [0, 0, 0, 5, 1, 1], [-1, -1, -1, 1, 1, 4]], np.float64)
    data["axis_boxes"] = boxes
    data["axis_out"] = np.array([geom.Aabb(tuple(b[:3]), tuple(b[3:])).longest_axis() for b in boxes], np.int64)

    # --- auto-framing camera for a field's bounding box
    bounds = np.array([[0, 0, 0, 63, 63, 63], [0, 0, 0, 511, 511, 511], [0, 0, 0, 1535, 767, 766]], np.float64)
    autocams = []
    for b in bounds:
        lo_, hi_ = tuple(b[:3]), tuple(b[3:])
        tri_a = geom.Triangle(lo_, hi_, lo_, 0)
        scene = SceneDesc([tri_a], [0], [], [])
        cam = cli.default_camera(scene, 1920, 1080)
        autocams.append([*cam.position, *cam.view_dir, *cam.up, cam.fov_y, cam.aspect])
    data["autocam_bounds"] = bounds
    data["autocam"] = np.array(autocams, np.float64)

    # --- service wire format (protocol.py): frame, camera update, control messages
    px = (np.arange(5 * 4 * 3) % 251).astype(np.uint8).tobytes()
    msgs = [protocol.FrameMessage(width=5, height=4, sequence=7, render_millis=12, pixels=px),
            protocol.CameraUpdateMessage((1.0, 2.0, 3.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), 45.0, 640, 360),
            protocol.ControlMessage({"status": "busy"})]
    for i, m in enumerate(msgs):
        data[f"wire_{i}"] = np.frombuffer(protocol.encode_message(m), np.uint8)

    np.savez_compressed(OUT / "reference_vectors.npz", **data)

    small = np.arange(4 * 3 * 3, dtype=np.uint8).reshape(3, 4, 3) * 7
    (OUT / "reference_4x3.ppm").write_bytes(ppm.encode_ppm(small))
    print("wrote", OUT / "reference_vectors.npz")


if __name__ == "__main__":
    main()
