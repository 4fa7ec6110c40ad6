"""Control-plane collectives and the data-plane exchange over gloo (2 and 3 CPU ranks)."""

from __future__ import annotations

import pytest
import torch

from dist_util import run_ranks
from paper_2501_01628_b200.engine import RenderOptions, render_digest, verify_collective_digest
from paper_2501_01628_b200.errors import ContractError, ProtocolError, TransportError
from paper_2501_01628_b200.geom import CameraSpec
from paper_2501_01628_b200.transport import SoloEndpoint
from paper_2501_01628_b200.volume import blob_field, decompose, default_tf


def _collectives(ep):
    tiles = ep.gather_to_root(bytes([ep.rank]) * (ep.rank + 1))
    bc = ep.broadcast_from_root(b"root-payload" if ep.rank == 0 else None)
    ep.barrier()
    ring = ep.ring_exchange(b"from-%d" % ep.rank)
    allg = ep.all_gather_bytes(b"r%d" % ep.rank)
    send = torch.full((5,), float(ep.rank))
    recv = torch.empty(5)
    nxt, prv = (ep.rank + 1) % ep.R, (ep.rank - 1) % ep.R
    ep.exchange([(nxt, send)], [(prv, recv)])
    ep.device_barrier()
    return tiles, bc, ring, allg, recv.tolist(), ep.stats.device_bytes_sent


@pytest.mark.parametrize("R", [2, 3])
def test_collective_semantics(R):
    res = run_ranks(R, _collectives)
    tiles0 = res[0][0]
    assert tiles0 == [bytes([r]) * (r + 1) for r in range(R)]
    for r, (tiles, bc, ring, allg, recv, sent) in enumerate(res):
        if r:
            assert tiles == []
        assert bc == b"root-payload"
        assert ring == b"from-%d" % ((r - 1) % R)
        assert allg == [b"r%d" % s for s in range(R)]
        assert recv == [float((r - 1) % R)] * 5
        assert sent == 20


def _digest_body(ep, diverge_rank):
    f = blob_field((17, 17, 17))
    dec = decompose(f, ep.R)
    fov = 50.0 if ep.rank == diverge_rank else 45.0
    cam = CameraSpec((40.0, 30.0, 50.0), (-1.0, -0.5, -1.2), (0.0, 1.0, 0.0), fov, 1.0)
    d = render_digest(cam, 32, 32, RenderOptions(), default_tf(), (0.0, 0.0, 0.0), dec)
    try:
        verify_collective_digest(ep, d)
        return "ok"
    except ContractError as exc:
        return f"contract: {exc}"


def test_divergent_parameters_raise_contract_error_on_every_rank():
    """engine.py:427-440 contract: every rank fails, before any GPU work, naming the bad rank."""
    res = run_ranks(3, _digest_body, 2)
    assert all(r.startswith("contract") and "[2]" in r for r in res)
    assert run_ranks(2, _digest_body, -1) == ["ok", "ok"]


def test_sequence_and_kind_checks():
    ep = SoloEndpoint()
    tag = ep._tag("TILE")
    assert ep._check(tag, ("TILE", 0, b"x"), 1) == b"x"
    with pytest.raises(ProtocolError, match="mismatched"):
        ep._check(ep._tag("TILE"), ("CONTROL", 1, b""), 1)
    with pytest.raises(ProtocolError, match="sequence"):
        ep._check(ep._tag("TILE"), ("TILE", 7, b""), 1)


def test_solo_endpoint_identities():
    ep = SoloEndpoint()
    assert ep.gather_to_root(b"a") == [b"a"]
    assert ep.broadcast_from_root(b"b") == b"b"
    assert ep.ring_exchange(b"c") == b"c"
    with pytest.raises(TransportError):
        ep.broadcast_from_root(None)
    with pytest.raises(TransportError):
        ep.exchange([(1, torch.zeros(1))], [])


def test_inproc_failure_aborts_peers_quickly():
    """A raising rank aborts the others' pending collectives (transport.py:533-543); the original error
    is the one re-raised, and nobody waits for the 30 s deadline."""
    import time

    from paper_2501_01628_b200.transport import run_collective

    def body(ep):
        if ep.rank == 1:
            raise ValueError("boom")
        ep.gather_to_root(b"x")  # rank 0 would wait for rank 1 forever

    t0 = time.monotonic()
    with pytest.raises(ValueError, match="boom"):
        run_collective(2, body, timeout=30.0)
    assert time.monotonic() - t0 < 5.0


def test_inproc_timeout_names_the_peer():
    from paper_2501_01628_b200.transport import run_collective

    def body(ep):
        if ep.rank == 0:
            ep.gather_to_root(b"x")  # rank 1 never sends

    with pytest.raises(TransportError, match="TILE from rank 1"):
        run_collective(2, body, timeout=0.5)
