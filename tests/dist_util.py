"""Spawn world_size CPU ranks on the gloo backend (127.0.0.1) and collect each rank's return value."""

from __future__ import annotations

import os
import socket
import sys
import traceback
from pathlib import Path

import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _entry(rank, world, port, fn, args, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    try:
        import torch.distributed as dist

        from paper_2501_01628_b200.transport import DistEndpoint

        dist.init_process_group("gloo", rank=rank, world_size=world)
        ep = DistEndpoint()
        out = fn(ep, *args)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok", out))
    except BaseException as exc:  # noqa: BLE001
        q.put((rank, "err", f"{type(exc).__name__}: {exc}\n{traceback.format_exc()}"))


def run_ranks(world: int, fn, *args, timeout: float = 120.0):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_entry, args=(r, world, port, fn, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    results, errors = {}, {}
    try:
        for _ in range(world):
            rank, status, val = q.get(timeout=timeout)
            (results if status == "ok" else errors)[rank] = val
    finally:
        for p in procs:  # exactly the processes started here
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    if errors:
        raise RuntimeError("rank failures:\n" + "\n".join(f"rank {r}: {e}" for r, e in sorted(errors.items())))
    return [results[r] for r in range(world)]
