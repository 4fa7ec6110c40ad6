"""Wire format of the thin-client stream ("next" row 3): the reference's DPRT framing and
service messages (pkg/src/dprt/protocol.py:21-216), so a reference viewer can display GPU frames.

Envelope: ``b"DPRT" | u8 kind | u32 LE length | payload``.  A frame payload is the 17-byte header
``<IIBII`` (width, height, format = 0 RGB8, sequence, render milliseconds) followed by row-major RGB8,
top row first -- exactly the bytes of the RGB8 tile the compositor leaves on rank 0.  Camera updates are
UTF-8 JSON ``{"pos", "dir", "up", "fovy", "w", "h"}``; control messages are JSON objects.
"""

from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass
from enum import IntEnum
from typing import Iterator, Tuple, Union

from .errors import DecodeError

MAGIC = b"DPRT"
ENVELOPE = struct.Struct("<4sBI")
FRAME_HEADER = struct.Struct("<IIBII")
FORMAT_RGB8 = 0
MIN_DIMENSION, MAX_DIMENSION = 16, 8192


class MsgKind(IntEnum):
    """Message kinds shared with the reference's framing (protocol.py:31-37)."""

    RAY_BATCH = 1
    TILE = 2
    BARRIER = 3
    CONTROL = 4
    CAMERA_UPDATE = 5
    FRAME = 6


@dataclass(frozen=True)
class CameraUpdateMessage:
    position: Tuple[float, float, float]
    view_dir: Tuple[float, float, float]
    up: Tuple[float, float, float]
    fov_y: float
    width: int
    height: int


@dataclass(frozen=True)
class FrameMessage:
    width: int
    height: int
    sequence: int
    render_millis: int
    pixels: bytes
    format: int = FORMAT_RGB8


@dataclass(frozen=True)
class ControlMessage:
    data: dict


Message = Union[CameraUpdateMessage, FrameMessage, ControlMessage]


def envelope(kind: MsgKind, payload: bytes) -> bytes:
    return ENVELOPE.pack(MAGIC, int(kind), len(payload)) + payload


def open_envelope(data: bytes, offset: int = 0) -> Tuple[MsgKind, bytes, int]:
    """(kind, payload, offset after the message); DecodeError on a bad or short envelope."""
    if len(data) - offset < ENVELOPE.size:
        raise DecodeError(f"truncated header at offset {offset}")
    magic, kind, length = ENVELOPE.unpack_from(data, offset)
    if magic != MAGIC:
        raise DecodeError(f"bad magic at offset {offset}")
    try:
        kind = MsgKind(kind)
    except ValueError:
        raise DecodeError(f"unknown msgKind {kind} at offset {offset + 4}") from None
    start = offset + ENVELOPE.size
    if len(data) - start < length:
        raise DecodeError(f"truncated payload at offset {start}")
    return kind, bytes(data[start:start + length]), start + length


class StreamSplitter:
    """Incremental envelope splitter for a byte stream (the reference's FrameParser role)."""

    def __init__(self) -> None:
        self._buf = bytearray()

    def feed(self, data: bytes) -> None:
        self._buf.extend(data)

    def messages(self) -> Iterator[Tuple[MsgKind, bytes]]:
        while len(self._buf) >= ENVELOPE.size:
            magic, kind, length = ENVELOPE.unpack_from(self._buf, 0)
            if magic != MAGIC:
                raise DecodeError("bad magic in stream")
            if len(self._buf) < ENVELOPE.size + length:
                return
            k, payload, end = open_envelope(bytes(self._buf[:ENVELOPE.size + length]))
            del self._buf[:end]
            yield k, payload


def _vec3(obj: dict, key: str):
    v = obj.get(key)
    if not (isinstance(v, list) and len(v) == 3
            and all(isinstance(c, (int, float)) and not isinstance(c, bool) for c in v)):
        raise DecodeError(f"camera update field {key!r} must hold 3 numbers")
    return tuple(float(c) for c in v)


def decode_payload(kind: MsgKind, payload: bytes) -> Message:
    if kind == MsgKind.FRAME:
        if len(payload) < FRAME_HEADER.size:
            raise DecodeError("frame payload truncated")
        w, h, fmt, seq, ms = FRAME_HEADER.unpack_from(payload, 0)
        if fmt != FORMAT_RGB8:
            raise DecodeError(f"unknown frame format {fmt}")
        if len(payload) != FRAME_HEADER.size + 3 * w * h:
            raise DecodeError(f"frame payload length mismatch for {w}x{h} RGB8")
        return FrameMessage(w, h, seq, ms, payload[FRAME_HEADER.size:])
    if kind in (MsgKind.CAMERA_UPDATE, MsgKind.CONTROL):
        try:
            obj = json.loads(payload.decode("utf-8"))
        except (UnicodeDecodeError, json.JSONDecodeError) as exc:
            raise DecodeError(f"payload is not UTF-8 JSON: {exc}") from exc
        if not isinstance(obj, dict):
            raise DecodeError("payload must be a JSON object")
        if kind == MsgKind.CONTROL:
            return ControlMessage(obj)
        pos, d, up = _vec3(obj, "pos"), _vec3(obj, "dir"), _vec3(obj, "up")
        fovy = obj.get("fovy")
        if not isinstance(fovy, (int, float)) or isinstance(fovy, bool) or not 0.0 < fovy < 180.0:
            raise DecodeError("camera update field 'fovy' must be in (0, 180)")
        w, h = obj.get("w"), obj.get("h")
        for name, val in (("w", w), ("h", h)):
            if not isinstance(val, int) or isinstance(val, bool) or not MIN_DIMENSION <= val <= MAX_DIMENSION:
                raise DecodeError(f"camera update field {name!r} must be an integer in [16, 8192]")
        if abs(math.sqrt(sum(c * c for c in d)) - 1.0) > 1e-6:
            raise DecodeError("camera update field 'dir' must be normalized")
        cx, cy, cz = d[1] * up[2] - d[2] * up[1], d[2] * up[0] - d[0] * up[2], d[0] * up[1] - d[1] * up[0]
        if cx * cx + cy * cy + cz * cz == 0.0:
            raise DecodeError("camera update fields 'dir' and 'up' must not be parallel")
        return CameraUpdateMessage(pos, d, up, float(fovy), w, h)
    raise DecodeError(f"msgKind {kind.name} is not a service message")


def encode_message(msg: Message) -> bytes:
    if isinstance(msg, FrameMessage):
        return envelope(MsgKind.FRAME, FRAME_HEADER.pack(msg.width, msg.height, msg.format, msg.sequence,
                                                          msg.render_millis) + msg.pixels)
    if isinstance(msg, CameraUpdateMessage):
        body = {"pos": list(msg.position), "dir": list(msg.view_dir), "up": list(msg.up), "fovy": msg.fov_y,
                "w": msg.width, "h": msg.height}
        return envelope(MsgKind.CAMERA_UPDATE, json.dumps(body, separators=(",", ":")).encode("utf-8"))
    if isinstance(msg, ControlMessage):
        return envelope(MsgKind.CONTROL, json.dumps(msg.data, separators=(",", ":")).encode("utf-8"))
    raise TypeError(f"cannot encode {type(msg).__name__}")


def decode_message(data: bytes) -> Message:
    kind, payload, end = open_envelope(data, 0)
    if end != len(data):
        raise DecodeError(f"trailing bytes at offset {end}")
    return decode_payload(kind, payload)
