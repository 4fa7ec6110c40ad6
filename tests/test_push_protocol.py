"""The fused march + exchange's cross-GPU protocol (p2p_push), model-checked on the CPU.

On real hardware every rank runs on its own GPU and ranks meet only through device memory: rank s's march of
frame e writes its fragment of every row block into that block owner's inbox slot (``PushLayout.slot_ptr``:
double-buffered by frame parity) and then raises its arrival flag at the owner to e; an owner's blend of
frame e waits (``wait_flags_kernel``: flag - e >= 0, wrap-safe) for every source's flag, reads the slots,
writes its rows of rank 0's frame and raises its done flag at rank 0; rank 0 waits for every done flag and
reads the frame, and (engine.py, push path) its next march starts only after that read.  Each rank's
operations run in its stream's order; nothing else orders them.

This test runs that protocol as a state machine over R ranks and several frames, with the production slot
arithmetic (``p2p.PushLayout``), under thousands of random interleavings of the ranks' streams, and checks:
every slot a blend reads holds exactly that frame's fragment from that source (never stale, never already
overwritten), every frame rank 0 reads is complete and unmixed, and no schedule deadlocks.  Two negative
controls show the checker has teeth: a single-buffered inbox is caught overwriting unread fragments, and an
equality flag test (instead of >=) is caught deadlocking."""

from __future__ import annotations

import random

import pytest

from paper_2501_01628_b200.p2p import PushLayout


class ProtocolError(AssertionError):
    pass


def run_protocol(R: int, frames: int, rng: random.Random, double_buffer: bool = True, ge_wait: bool = True) -> int:
    """One random schedule of ``frames`` frames on ``R`` ranks; returns the number of steps taken."""
    L = PushLayout(R, 64, 8 * R, 16)
    base = [(o + 1) << 32 for o in range(R)]  # disjoint inbox address spaces

    def slot(o, e, s):
        return L.slot_ptr(base[o], e if double_buffer else 0, s)

    inbox = {}                     # slot address -> (epoch, source) last written
    consumed = set()               # (owner, epoch, source) fragments an owner's blend has read
    arrival = [[0] * R for _ in range(R)]  # arrival[o][s]: epoch word source s raised at owner o
    done = [0] * R                 # done[o] at rank 0: epoch of block o's last blend
    frame = [0] * R                # epoch whose rows block o of rank 0's frame holds
    read = set()                   # epochs rank 0 has read back

    def reached(word, e):
        return (word - e) >= 0 if ge_wait else word == e

    # each rank's stream, in issue order (rank 0 also waits for all blocks and reads the frame)
    streams = []
    for r in range(R):
        ops = []
        for e in range(1, frames + 1):
            ops += [("march", e), ("wait", e), ("blend", e)]
            if r == 0:
                ops += [("wait_done", e), ("read", e)]
        streams.append(ops)
    pc = [0] * R

    def enabled(r):
        if pc[r] >= len(streams[r]):
            return False
        op, e = streams[r][pc[r]]
        if op == "wait":
            return all(reached(arrival[r][s], e) for s in range(R))
        if op == "wait_done":
            return all(reached(done[o], e) for o in range(R))
        return True

    steps = 0
    while any(pc[r] < len(streams[r]) for r in range(R)):
        ready = [r for r in range(R) if enabled(r)]
        if not ready:
            raise ProtocolError(f"deadlock at {[streams[r][pc[r]] if pc[r] < len(streams[r]) else 'end' for r in range(R)]}")
        r = rng.choice(ready)
        op, e = streams[r][pc[r]]
        pc[r] += 1
        steps += 1
        if op == "march":  # rank r = source: its fragment of every owner's block, then the arrival flags
            for o in range(R):
                a = slot(o, e, r)
                prev = inbox.get(a)
                if prev is not None and (o, prev[0], prev[1]) not in consumed:
                    raise ProtocolError(f"march {e} of rank {r} overwrites owner {o}'s unread fragment {prev}")
                inbox[a] = (e, r)
            for o in range(R):
                arrival[o][r] = e
        elif op == "blend":  # rank r = owner of block r
            for s in range(R):
                got = inbox.get(slot(r, e, s))
                if got != (e, s):
                    raise ProtocolError(f"blend {e} at owner {r} reads {got} from source {s}'s slot")
                consumed.add((r, e, s))
            if frame[r] and frame[r] not in read:
                raise ProtocolError(f"blend {e} at owner {r} overwrites frame {frame[r]} before rank 0 read it")
            frame[r] = e
            done[r] = e
        elif op == "read":
            if any(f != e for f in frame):
                raise ProtocolError(f"rank 0 reads frame {e} holding blocks of frames {frame}")
            read.add(e)
    return steps


@pytest.mark.parametrize("R", [2, 3, 4, 8])
def test_push_protocol_holds_under_random_schedules(R):
    rng = random.Random(1000 + R)
    for _ in range(400 if R <= 4 else 150):
        run_protocol(R, frames=6, rng=rng)


def test_single_buffered_inbox_is_caught():
    rng = random.Random(7)
    with pytest.raises(ProtocolError, match="overwrites owner"):
        for _ in range(400):
            run_protocol(3, frames=6, rng=rng, double_buffer=False)


def test_equality_flag_wait_is_caught_deadlocking():
    rng = random.Random(11)
    with pytest.raises(ProtocolError, match="deadlock"):
        for _ in range(400):
            run_protocol(3, frames=6, rng=rng, ge_wait=False)


def test_layout_slots_tile_the_inbox_by_parity_and_source():
    """The slots the model addresses are the production ones: per owner, 2 x P disjoint slots of
    ``slot`` pixels covering the inbox exactly, frame e and e + 2 sharing a slot, e and e + 1 not."""
    for P, W, H in [(2, 64, 50), (3, 37, 29), (8, 160, 90)]:
        L = PushLayout(P, W, H, 16)
        spans = sorted((L.slot_ptr(0, e, s), L.slot_ptr(0, e, s) + 16 * L.slot) for e in (0, 1) for s in range(P))
        assert spans[0][0] == 0 and spans[-1][1] == 16 * L.inbox_pixels()
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        for s in range(P):
            assert L.slot_ptr(0, 5, s) == L.slot_ptr(0, 7, s) != L.slot_ptr(0, 6, s)
        assert L.slot >= max(b1 - b0 for b0, b1 in L.blocks) * W
