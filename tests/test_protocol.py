"""The thin-client wire format against bytes produced by the reference's own encoder."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from paper_2501_01628_b200.errors import DecodeError
from paper_2501_01628_b200.protocol import (CameraUpdateMessage, ControlMessage, FrameMessage, MsgKind,
                                            StreamSplitter, decode_message, encode_message, envelope)

GOLD = np.load(Path(__file__).parent / "golden" / "reference_vectors.npz")


def _wire(i):
    return GOLD[f"wire_{i}"].tobytes()


def test_frame_message_matches_reference_bytes():
    px = (np.arange(5 * 4 * 3) % 251).astype(np.uint8).tobytes()
    mine = FrameMessage(5, 4, 7, 12, px)
    assert encode_message(mine) == _wire(0)
    assert decode_message(_wire(0)) == mine


def test_camera_and_control_messages_match_reference_bytes():
    cam = CameraUpdateMessage((1.0, 2.0, 3.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), 45.0, 640, 360)
    assert encode_message(cam) == _wire(1)
    assert decode_message(_wire(1)) == cam
    assert encode_message(ControlMessage({"status": "busy"})) == _wire(2)


def test_stream_splitter_handles_fragments():
    blob = _wire(1) + _wire(0) + _wire(2)
    sp = StreamSplitter()
    got = []
    for i in range(0, len(blob), 7):
        sp.feed(blob[i:i + 7])
        got.extend(k for k, _ in sp.messages())
    assert got == [MsgKind.CAMERA_UPDATE, MsgKind.FRAME, MsgKind.CONTROL]


@pytest.mark.parametrize("data", [b"XXXX\x06\x00\x00\x00\x00", envelope(MsgKind.FRAME, b"\x01\x00"),
                                  envelope(MsgKind.CAMERA_UPDATE, b"{\"pos\":1}"), _wire(0)[:-1],
                                  _wire(0) + b"\x00"])
def test_decode_errors(data):
    with pytest.raises(DecodeError):
        decode_message(data)


def test_ppm_matches_reference_bytes():
    from paper_2501_01628_b200.ppm import decode_ppm, encode_ppm

    ref = (Path(__file__).parent / "golden" / "reference_4x3.ppm").read_bytes()
    small = np.arange(4 * 3 * 3, dtype=np.uint8).reshape(3, 4, 3) * 7
    assert encode_ppm(small) == ref
    assert np.array_equal(decode_ppm(ref), small)
