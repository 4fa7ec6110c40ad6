"""Two PROCESSES sharing the one GPU of the test box, gloo control plane: the fused p2p compositor's real
CUDA IPC path (export a handle per rank, map the peer's partial and rank 0's frame in the other process,
composite through the mapped pointers).  In-process rank threads (test_gpu_multirank.py) share one
address space and never exercise IPC.  No kernel waits on another process: the device barriers drain the
stream and meet on the host (DistEndpoint.device_barrier, non-NCCL branch)."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from dist_util import run_ranks
from scenes import RGB8_MAX_LSB, RGBA_ATOL, c1, oracle_partials

pytestmark = pytest.mark.gpu


def _rank_body(ep, mode, W, H, fdt="f32"):
    import torch

    from paper_2501_01628_b200 import device as dev
    from paper_2501_01628_b200.engine import RenderOptions, VolumeRenderer
    from paper_2501_01628_b200.transport import DistEndpoint

    cuda = torch.device("cuda", 0)
    ep = DistEndpoint(device=cuda)
    s = c1(P=ep.R, W=W, H=H)
    b = dev.DeviceBrick(s.dec.brick(ep.rank), cuda).generate(s.field)
    vr = VolumeRenderer(ep, b, s.dec, s.tf, s.background)
    out = []
    for frame in range(2):
        res = vr.render(s.cam, W, H, RenderOptions(composite=mode, keep_float=True, frame_index=frame,
                                                   fragment_dtype=fdt))
        torch.cuda.synchronize()
        out.append((None if res.image is None else np.asarray(res.image),
                    None if res.rgb8 is None else res.rgb8.cpu().numpy()))
    used = vr.compositor.mode
    vr.compositor = None
    b.close()
    return used, out


@pytest.mark.parametrize("mode,R,fdt", [("p2p", 2, "f32"), ("auto", 3, "f32"), ("p2p", 2, "f16")])
def test_ipc_p2p_frame_across_processes(cuda_device, oracle_lib, mode, R, fdt):
    from scenes import RGBA_ATOL_F16

    W, H = 160, 122
    tol, lsb = (RGBA_ATOL, RGB8_MAX_LSB) if fdt == "f32" else (RGBA_ATOL_F16, 2)
    results = run_ranks(R, _rank_body, mode, W, H, fdt, timeout=240.0)
    s = c1(P=R, W=W, H=H)
    vox = oracle.generate_field(s.field.dims, s.field.blobs)
    ref, _ = oracle_partials(vox, s.dec, s.cam, s.tf, s.dt, s.ert, W, H)
    want = oracle.composite(ref, s.dec.visibility_order(s.cam.position), s.background)
    for r, (used, frames) in enumerate(results):
        assert used == "p2p", f"rank {r} fell back to {used}: the IPC mapping failed"
        for image, rgb8 in frames:
            if r == 0:
                assert np.abs(image - want).max() <= tol
                q = rgb8.astype(np.int16) - oracle.tone_map_rgb8(want).astype(np.int16)
                assert np.abs(q).max() <= lsb
            else:
                assert image is None and rgb8 is None


@pytest.mark.parametrize("mode,R", [("direct_send", 2), ("binary_swap", 4), ("direct_send", 3)])
def test_exchange_modes_across_processes(cuda_device, oracle_lib, mode, R):
    """The exchange schedules through DistEndpoint.exchange (batched isend/irecv, the code NCCL runs at
    N > 1) in separate processes; gloo moves the device fragments through host staging buffers here."""
    W, H = 144, 104
    results = run_ranks(R, _rank_body, mode, W, H, "f32", timeout=240.0)
    s = c1(P=R, W=W, H=H)
    vox = oracle.generate_field(s.field.dims, s.field.blobs)
    ref, _ = oracle_partials(vox, s.dec, s.cam, s.tf, s.dt, s.ert, W, H)
    want = oracle.composite(ref, s.dec.visibility_order(s.cam.position), s.background)
    for r, (used, frames) in enumerate(results):
        assert used == mode
        for image, rgb8 in frames:
            if r == 0:
                assert np.abs(image - want).max() <= RGBA_ATOL
                q = rgb8.astype(np.int16) - oracle.tone_map_rgb8(want).astype(np.int16)
                assert np.abs(q).max() <= RGB8_MAX_LSB
            else:
                assert image is None and rgb8 is None


@pytest.mark.parametrize("fragments", ["f32", "f16"])
def test_bench_multi_rank_code_path(tmp_path, fragments):
    """bench.py's N > 1 leg (weak-scaled bricks, compositor roofline, e2e, max over ranks) run as two
    torchrun processes on this box's one GPU with the gloo control plane (DPRT_BENCH_BACKEND=gloo): a
    functional check of the code the 8-GPU scaling run executes, not a measurement.  The p2p_push frames
    leg is forced on: with both ranks on one GPU it must fail cleanly on every rank (the push compositor
    refuses ranks sharing a GPU) and be reported in the line without disturbing the rest of it."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, DPRT_BENCH_BACKEND="gloo", DPRT_BENCH_PUSH="force")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={29500 + os.getpid() % 1000}", str(root / "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--fragments", fragments]
    p = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["compositor_roofline"]["mode"] in ("p2p", "direct_send")
    assert line["config"]["bricks"] == 2 and line["run"]["fragments"] == fragments
    push = line["p2p_push_frames"]
    assert push["value"] is None and set(push["errors"]) == {"0", "1"} and not push["cuda_context_lost"]
    assert all("TransportError" in e for e in push["errors"].values())
