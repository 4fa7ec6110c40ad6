"""Rank endpoints: the reference's collective API shape over one-process-per-GPU ``torch.distributed``.

The reference runs R ranks as threads of one process and moves bytes over queues or loopback TCP
(pkg/src/dprt/transport.py:1-8, 164-204, 254-420) with four collectives: ``ring_exchange``,
``gather_to_root``, ``broadcast_from_root``, ``barrier`` (transport.py:457-507).  Here each rank is a
process bound to one GPU; the same four collectives form the host CONTROL plane (digest votes, tiny
metadata) and carry the reference's per-(channel, kind) sequence check (transport.py:129-140) so that
mismatched collective calls still raise ``ProtocolError``.  Image fragments use the DATA plane:
``exchange`` posts grouped point-to-point sends/receives of device tensors (NCCL over NVLink on
B200, gloo on CPU for tests), and ``device_barrier`` is a stream-ordered all-reduce used to order
peer-memory (P2P) access without a host synchronisation.
"""

from __future__ import annotations

import os
import pickle
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from .errors import ProtocolError, TransportError

DEFAULT_TIMEOUT_SECS = 30.0


def resolve_timeout(explicit: Optional[float] = None) -> float:
    """Explicit value, else DPRT_TIMEOUT_SECS, else 30 s (transport.py:32-39)."""
    if explicit is not None:
        return float(explicit)
    env = os.environ.get("DPRT_TIMEOUT_SECS")
    return float(env) if env else DEFAULT_TIMEOUT_SECS


@dataclass
class TransportStats:
    """Byte / message counters (transport.py:49-57); ``device_bytes_*`` count data-plane tensors."""

    bytes_sent: int = 0
    bytes_received: int = 0
    messages_sent: int = 0
    messages_received: int = 0
    device_bytes_sent: int = 0
    device_bytes_received: int = 0

    def traffic(self) -> int:
        return self.bytes_sent + self.bytes_received


class RankEndpoint:
    """One rank's handle; driven by a single thread.  Subclasses provide the byte transport."""

    def __init__(self, rank: int, num_ranks: int, device: Optional[torch.device] = None):
        if not (0 <= rank < num_ranks):
            raise TransportError(f"rank {rank} outside [0, {num_ranks})")
        self.rank = rank
        self.R = num_ranks
        self.device = device if device is not None else torch.device("cpu")
        self.stats = TransportStats()
        self._seq: Dict[str, int] = {}

    # -- sequence tagging: every control message carries (kind, seq) like transport.py:101-143
    def _tag(self, kind: str) -> Tuple[str, int]:
        seq = self._seq.get(kind, 0)
        self._seq[kind] = seq + 1
        return kind, seq

    def _check(self, tag: Tuple[str, int], got, src: int):
        kind, seq = tag
        if not (isinstance(got, tuple) and len(got) == 3):
            raise ProtocolError(f"rank {self.rank}: malformed control message from rank {src}")
        gkind, gseq, payload = got
        if gkind != kind:
            raise ProtocolError(f"rank {self.rank}: expected {kind} from rank {src}, got {gkind}; "
                                "collective calls are mismatched")
        if gseq != seq:
            raise ProtocolError(f"rank {self.rank}: sequence {gseq} from rank {src} for {kind}, expected {seq}")
        return payload

    # -- control plane (bytes), same signatures as transport.py:457-507
    def gather_to_root(self, tile: bytes) -> List[bytes]:
        raise NotImplementedError

    def broadcast_from_root(self, payload: Optional[bytes]) -> bytes:
        raise NotImplementedError

    def barrier(self) -> None:
        raise NotImplementedError

    def ring_exchange(self, outgoing: bytes) -> bytes:
        raise NotImplementedError

    # -- data plane (device tensors)
    def exchange(self, sends: Sequence[Tuple[int, torch.Tensor]], recvs: Sequence[Tuple[int, torch.Tensor]]) -> None:
        raise NotImplementedError

    def device_barrier(self) -> None:
        raise NotImplementedError

    def share_pointers(self, device_index: int, ptr: int) -> List[int]:
        """Every rank's buffer (allocated with dprt_device_alloc, or 0), usable from this rank's GPU."""
        raise NotImplementedError

    def unshare_pointers(self, device_index: int, ptrs: Sequence[int]) -> None:
        """Release mappings returned by share_pointers."""

    def all_gather_bytes(self, payload: bytes) -> List[bytes]:
        """gather_to_root + broadcast_from_root, the reference's all-gather idiom (api.py:284-293)."""
        tiles = self.gather_to_root(payload)
        blob = pickle.dumps(tiles) if self.rank == 0 else None
        return pickle.loads(self.broadcast_from_root(blob))

    def close(self) -> None:
        pass


class SoloEndpoint(RankEndpoint):
    """R == 1: every collective is the identity (transport.py:459-460, 467-468, 482-484, 499-500)."""

    def __init__(self, device: Optional[torch.device] = None):
        super().__init__(0, 1, device)

    def gather_to_root(self, tile: bytes) -> List[bytes]:
        return [tile]

    def broadcast_from_root(self, payload: Optional[bytes]) -> bytes:
        if payload is None:
            raise TransportError("rank 0 must supply the broadcast payload")
        return payload

    def barrier(self) -> None:
        return None

    def ring_exchange(self, outgoing: bytes) -> bytes:
        return outgoing

    def exchange(self, sends, recvs) -> None:
        if sends or recvs:
            raise TransportError("a single rank has no peers to exchange with")

    def device_barrier(self) -> None:
        return None

    def share_pointers(self, device_index: int, ptr: int) -> List[int]:
        return [ptr]


class DistEndpoint(RankEndpoint):
    """torch.distributed process group (NCCL on GPUs, gloo on CPU).  One process per rank/GPU."""

    def __init__(self, group=None, device: Optional[torch.device] = None):
        if not dist.is_initialized():
            raise TransportError("torch.distributed is not initialised; call init_dist() first")
        super().__init__(dist.get_rank(group), dist.get_world_size(group), device)
        self.group = group
        self.backend = dist.get_backend(group)
        self._token = None

    def _obj_device(self):
        return self.device if self.backend == "nccl" else None

    def gather_to_root(self, tile: bytes) -> List[bytes]:
        tag = self._tag("TILE")
        msg = (tag[0], tag[1], tile)
        out = [None] * self.R if self.rank == 0 else None
        try:
            dist.gather_object(msg, out, dst=0, group=self.group)
        except Exception as exc:  # noqa: BLE001
            raise TransportError(f"rank {self.rank}: gather_to_root failed: {exc}") from exc
        self.stats.messages_sent += 1
        self.stats.bytes_sent += len(tile)
        if self.rank != 0:
            return []
        res = [self._check(tag, m, src) for src, m in enumerate(out)]
        self.stats.messages_received += self.R - 1
        self.stats.bytes_received += sum(len(t) for t in res[1:])
        return res

    def broadcast_from_root(self, payload: Optional[bytes]) -> bytes:
        tag = self._tag("CONTROL")
        if self.rank == 0 and payload is None:
            raise TransportError("rank 0 must supply the broadcast payload")
        box = [(tag[0], tag[1], payload) if self.rank == 0 else None]
        try:
            dist.broadcast_object_list(box, src=0, group=self.group, device=self._obj_device())
        except Exception as exc:  # noqa: BLE001
            raise TransportError(f"rank {self.rank}: broadcast_from_root failed: {exc}") from exc
        data = self._check(tag, box[0], 0)
        if self.rank != 0:
            self.stats.messages_received += 1
            self.stats.bytes_received += len(data)
        return data

    def barrier(self) -> None:
        self.gather_to_root(b"")
        self.broadcast_from_root(b"" if self.rank == 0 else None)

    def ring_exchange(self, outgoing: bytes) -> bytes:
        allb = self.all_gather_bytes(outgoing)
        return allb[(self.rank - 1) % self.R]

    def exchange(self, sends, recvs) -> None:
        if self.backend != "nccl" and any(t.is_cuda for _, t in list(sends) + list(recvs)):
            return self._exchange_staged(sends, recvs)
        ops = []
        for peer, t in sends:
            ops.append(dist.P2POp(dist.isend, t, peer, group=self.group))
            self.stats.device_bytes_sent += t.numel() * t.element_size()
        for peer, t in recvs:
            ops.append(dist.P2POp(dist.irecv, t, peer, group=self.group))
            self.stats.device_bytes_received += t.numel() * t.element_size()
        if not ops:
            return
        try:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        except Exception as exc:  # noqa: BLE001
            raise TransportError(f"rank {self.rank}: fragment exchange failed: {exc}") from exc

    def _exchange_staged(self, sends, recvs) -> None:
        """Non-NCCL backends (gloo) move CPU tensors only: device fragments are staged through host memory
        (the functional multi-process mode on a shared GPU and CPU hosts; NCCL moves them device to device)."""
        hs = [(peer, t.detach().to("cpu")) if t.is_cuda else (peer, t) for peer, t in sends]
        hr = [(peer, torch.empty(t.shape, dtype=t.dtype) if t.is_cuda else t) for peer, t in recvs]
        ops = [dist.P2POp(dist.isend, t, peer, group=self.group) for peer, t in hs]
        ops += [dist.P2POp(dist.irecv, t, peer, group=self.group) for peer, t in hr]
        for _, t in hs:
            self.stats.device_bytes_sent += t.numel() * t.element_size()
        for _, t in hr:
            self.stats.device_bytes_received += t.numel() * t.element_size()
        if not ops:
            return
        try:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        except Exception as exc:  # noqa: BLE001
            raise TransportError(f"rank {self.rank}: fragment exchange failed: {exc}") from exc
        for (_, dst), (_, src) in zip(recvs, hr):
            if dst.is_cuda:
                dst.copy_(src)

    def share_pointers(self, device_index: int, ptr: int) -> List[int]:
        """CUDA IPC: export this rank's buffer, map every peer's (lazily enabling NVLink peer access)."""
        from . import device as dev

        handle = b""
        if ptr:
            try:
                handle = dev.ipc_handle(device_index, ptr)
            except Exception:  # noqa: BLE001 - a 0 entry tells every rank this mapping failed
                handle = b""
        handles = self.all_gather_bytes(handle)  # always collective, even after a local failure
        out = []
        for r, h in enumerate(handles):
            if r == self.rank:
                out.append(ptr)
            elif h:
                try:
                    out.append(dev.ipc_open(device_index, h))
                except Exception:  # noqa: BLE001
                    out.append(0)
            else:
                out.append(0)
        return out

    def unshare_pointers(self, device_index: int, ptrs: Sequence[int]) -> None:
        from . import device as dev

        for r, p in enumerate(ptrs):
            if r != self.rank and p:
                try:
                    dev.ipc_close(device_index, p)
                except Exception:  # noqa: BLE001 - best effort on teardown
                    pass

    def device_barrier(self) -> None:
        """Every rank's stream-ordered work issued so far is complete before any rank's later work.
        NCCL: a 4-byte all-reduce on the current stream (stream ordered, the host does not block).
        Other backends (gloo with CUDA buffers): drain this rank's stream, then a host all-reduce."""
        if self._token is None:
            dev = self.device if self.backend == "nccl" else torch.device("cpu")
            self._token = torch.zeros(1, dtype=torch.int32, device=dev)
        if self.backend != "nccl" and self.device is not None and self.device.type == "cuda":
            torch.cuda.current_stream(self.device).synchronize()
        dist.all_reduce(self._token, group=self.group)


def init_dist(backend: Optional[str] = None) -> DistEndpoint:
    """Initialise the default process group from torchrun's env (RANK, WORLD_SIZE, MASTER_*) and bind
    this process to cuda:LOCAL_RANK when using NCCL."""
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    device = None
    if backend == "nccl":
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        device = torch.device("cuda", local)
    if not dist.is_initialized():
        kwargs = {}
        if device is not None:
            kwargs["device_id"] = device
        dist.init_process_group(backend, **kwargs)
    return DistEndpoint(device=device)


def endpoint_for(device: Optional[torch.device] = None) -> RankEndpoint:
    """DistEndpoint under an initialised process group with >1 rank, else SoloEndpoint."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        return DistEndpoint(device=device)
    return SoloEndpoint(device)


# ---------------------------------------------------------------------------------------------------
# in-process ranks (threads), the reference's inproc backend + run_collective harness
# (transport.py:164-204, 519-566): R ranks share one process -- and, for tests on a single GPU, one
# device.  Fragments move by device-to-device copy; peer pointers are plain pointers.


class _InprocSession:
    def __init__(self, num_ranks: int, timeout: float):
        import queue
        import threading

        self.R = num_ranks
        self.timeout = timeout
        self.ctrl = {(s, d): queue.Queue() for s in range(num_ranks) for d in range(num_ranks)}
        self.data = {(s, d): queue.Queue() for s in range(num_ranks) for d in range(num_ranks)}
        self.acks = {(s, d): queue.Queue() for s in range(num_ranks) for d in range(num_ranks)}
        self.barrier = threading.Barrier(num_ranks, timeout=timeout)
        self.aborted = threading.Event()

    def abort(self) -> None:
        self.aborted.set()
        self.barrier.abort()


class InprocEndpoint(RankEndpoint):
    """A rank thread of an in-process group."""

    def __init__(self, rank: int, session: _InprocSession, device: Optional[torch.device] = None):
        super().__init__(rank, session.R, device)
        self.session = session

    def _get(self, q, what: str):
        """Blocking receive that gives up at the deadline or as soon as another rank has failed
        (the abort-on-failure behaviour of run_collective, transport.py:533-543)."""
        import queue
        import time as _time

        deadline = _time.monotonic() + self.session.timeout
        while True:
            try:
                return q.get(timeout=0.02)
            except queue.Empty:
                if self.session.aborted.is_set():
                    raise TransportError(f"rank {self.rank}: collective aborted while waiting for {what}") from None
                if _time.monotonic() > deadline:
                    raise TransportError(f"rank {self.rank}: timeout after {self.session.timeout:g}s waiting "
                                         f"for {what}") from None

    def _send_ctrl(self, dst: int, kind: str, payload) -> None:
        tag = self._tag(f"{kind}->{dst}")
        self.session.ctrl[(self.rank, dst)].put((tag[0], tag[1], payload))
        if payload is not None:
            self.stats.messages_sent += 1
            self.stats.bytes_sent += len(payload)

    def _recv_ctrl(self, src: int, kind: str):
        tag = self._tag(f"{kind}<-{src}")
        got = self._get(self.session.ctrl[(src, self.rank)], f"{kind} from rank {src}")
        payload = self._check((f"{kind}->{self.rank}", tag[1]), got, src)
        self.stats.messages_received += 1
        self.stats.bytes_received += len(payload)
        return payload

    def gather_to_root(self, tile: bytes) -> List[bytes]:
        if self.rank == 0:
            return [tile] + [self._recv_ctrl(s, "TILE") for s in range(1, self.R)]
        self._send_ctrl(0, "TILE", tile)
        return []

    def broadcast_from_root(self, payload: Optional[bytes]) -> bytes:
        if self.rank == 0:
            if payload is None:
                raise TransportError("rank 0 must supply the broadcast payload")
            for d in range(1, self.R):
                self._send_ctrl(d, "CONTROL", payload)
            return payload
        return self._recv_ctrl(0, "CONTROL")

    def barrier(self) -> None:
        self.gather_to_root(b"")
        self.broadcast_from_root(b"" if self.rank == 0 else None)

    def ring_exchange(self, outgoing: bytes) -> bytes:
        if self.R == 1:
            return outgoing
        self._send_ctrl((self.rank + 1) % self.R, "RING", outgoing)
        return self._recv_ctrl((self.rank - 1) % self.R, "RING")

    def exchange(self, sends, recvs) -> None:
        """Point-to-point tensor exchange; a send buffer is reusable when exchange returns."""
        if sends:
            torch.cuda.current_stream(self.device).synchronize() if self.device.type == "cuda" else None
        for peer, t in sends:
            self.session.data[(self.rank, peer)].put(t)
            self.stats.device_bytes_sent += t.numel() * t.element_size()
        for peer, t in recvs:
            src = self._get(self.session.data[(peer, self.rank)], f"fragment from rank {peer}")
            if src.numel() != t.numel():
                raise ProtocolError(f"rank {self.rank}: fragment from rank {peer} has {src.numel()} elements, "
                                    f"expected {t.numel()}")
            t.copy_(src.view_as(t))
            if t.is_cuda:
                torch.cuda.current_stream(t.device).synchronize()
            self.session.acks[(peer, self.rank)].put(True)
            self.stats.device_bytes_received += t.numel() * t.element_size()
        for peer, _ in sends:
            self._get(self.session.acks[(self.rank, peer)], f"receipt from rank {peer}")

    def share_pointers(self, device_index: int, ptr: int) -> List[int]:
        """Same process: peer pointers are plain pointers.  A peer on another GPU is usable once peer access
        to its device is enabled (NVLink P2P); where that fails the entry is 0, like a refused IPC mapping."""
        from . import device as dev

        entries = [b.decode().split(":") for b in self.all_gather_bytes(f"{ptr}:{device_index}".encode())]
        out = []
        for r, (p, d) in enumerate(entries):
            p, d = int(p), int(d)
            if r != self.rank and p and d != device_index:
                try:
                    dev.enable_peer(device_index, d)
                except Exception:  # noqa: BLE001 - no P2P between these GPUs: report the mapping as failed
                    p = 0
            out.append(p)
        return out

    def device_barrier(self) -> None:
        import threading

        if self.device.type == "cuda":
            torch.cuda.current_stream(self.device).synchronize()
        try:
            self.session.barrier.wait()
        except threading.BrokenBarrierError:
            raise TransportError(f"rank {self.rank}: collective aborted") from None


def run_collective(num_ranks: int, body, device=None, timeout: Optional[float] = None):
    """Drive ``body(ep)`` on R rank threads of one process (transport.py:519-566); returns per-rank
    results, re-raising the first rank failure.  A failing rank aborts the others' pending calls.

    ``device``: one torch device for every rank (tests on one GPU), or a sequence of devices -- rank r is
    bound to ``device[r % len(device)]``, so one process drives every GPU of the box with one thread per
    rank, the reference's harness shape (transport.py:545-548).  Rank threads bind their device in each
    native call (dprt_* bind themselves) and ctypes releases the GIL, so the ranks' launches overlap."""
    import threading

    session = _InprocSession(num_ranks, resolve_timeout(timeout))
    if isinstance(device, (list, tuple)):
        if not device:
            raise TransportError("run_collective needs at least one device")
        devs = [device[r % len(device)] for r in range(num_ranks)]
    else:
        devs = [device] * num_ranks
    eps = [InprocEndpoint(r, session, devs[r]) for r in range(num_ranks)]
    results: List[object] = [None] * num_ranks
    errors: Dict[int, BaseException] = {}

    def runner(ep):
        try:
            if ep.device is not None and ep.device.type == "cuda":
                torch.cuda.set_device(ep.device)
            results[ep.rank] = body(ep)
        except BaseException as exc:  # noqa: BLE001
            errors[ep.rank] = exc
            session.abort()

    threads = [threading.Thread(target=runner, args=(ep,), daemon=True, name=f"dprt-rank-{ep.rank}") for ep in eps]
    for t in threads:
        t.start()
    for t in threads:
        t.join(session.timeout * (num_ranks + 2) + 60.0)
    if any(t.is_alive() for t in threads):
        raise TransportError("rank threads failed to finish; session leaked")
    if errors:
        first = [e for _, e in sorted(errors.items()) if not isinstance(e, TransportError)]
        raise (first[0] if first else next(iter(sorted(errors.items())))[1])
    return results
