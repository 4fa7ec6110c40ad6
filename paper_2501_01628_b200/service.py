"""Thin-client streaming of GPU frames ("next" row 3): camera updates in, RGB8 frames out.

Same session contract as the reference's render service (pkg/src/dprt/service.py:222-296): rank 0
accepts ONE client speaking raw DPRT framing over TCP; pending camera updates coalesce so only the newest
is rendered (latest wins, service.py:67-70,274); rank 0 broadcasts each command on the control plane so
every rank renders the same collective frame (service.py:285-289); extra clients are refused with a
``{"status": "busy"}`` control message (service.py:151-170); a client decode error is reported back
before shutdown.  The frame payload is the RGB8 image the compositor leaves on rank 0, copied once to
pinned host memory.  (The reference's WebSocket upgrade, ws.py, is browser plumbing and out of scope.)
"""

from __future__ import annotations

import json
import socket as socketlib
import threading
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Tuple

from . import api
from .errors import DecodeError, DprtError
from .protocol import (CameraUpdateMessage, ControlMessage, FrameMessage, MsgKind, StreamSplitter, decode_payload,
                       encode_message)
from .scene import VolumeScene
from .transport import RankEndpoint

_POLL = 0.005


@dataclass
class ServeOptions:
    host: str = "127.0.0.1"
    port: int = 0
    accept_timeout_secs: float = 30.0
    composite: str = "auto"
    on_listening: Optional[Callable[[Tuple[str, int]], None]] = None


@dataclass
class ServeReport:
    frames_sent: int = 0
    render_millis: List[int] = field(default_factory=list)
    records: List[str] = field(default_factory=list)


class _Client:
    def __init__(self, sock: socketlib.socket):
        self.sock = sock
        self.closed = False
        self.error: Optional[str] = None
        self._latest: Optional[CameraUpdateMessage] = None
        self._lock = threading.Lock()
        self._thread = threading.Thread(target=self._recv, daemon=True, name="dprt-client")
        self._thread.start()

    def _recv(self) -> None:
        split = StreamSplitter()
        try:
            while True:
                chunk = self.sock.recv(1 << 16)
                if not chunk:
                    break
                split.feed(chunk)
                for kind, payload in split.messages():
                    if kind == MsgKind.CAMERA_UPDATE:
                        msg = decode_payload(kind, payload)
                        with self._lock:
                            self._latest = msg  # latest wins
        except DecodeError as exc:
            self.error = str(exc)
        except OSError:
            pass
        finally:
            self.closed = True

    def take_latest(self) -> Optional[CameraUpdateMessage]:
        with self._lock:
            msg, self._latest = self._latest, None
        return msg

    def send(self, msg) -> None:
        self.sock.sendall(encode_message(msg))

    def close(self) -> None:
        self.closed = True
        try:
            self.sock.shutdown(socketlib.SHUT_RDWR)
        except OSError:
            pass
        self.sock.close()


def build_rank_objects(ep: RankEndpoint, scene: VolumeScene, composite: str = "auto", cuda=None):
    """Per-rank committed render graph for a volume scene (service.py:173-204 analog)."""
    d = api.Device(ep, cuda)
    sf = d.create("spatialField")
    f = scene.field
    sf.set_param("dims", f.dims)
    sf.set_param("origin", f.origin)
    sf.set_param("spacing", f.spacing)
    if scene.data_path is not None:
        sf.set_param("data", scene.voxels())  # memory map: each rank copies only its brick
    else:
        g = scene.generator or {}
        sf.set_param("generator", g.get("generator", "blobs"))
        if g.get("generator") == "marschnerLobb":
            sf.set_param("frequency", g["frequency"])
            sf.set_param("alpha", g["alpha"])
        else:
            sf.set_param("seed", g.get("seed", 1))
            sf.set_param("blobCount", g.get("blobCount", 16))
            sf.set_param("lopsided", g.get("lopsided", False))
    sf.commit()
    tf = d.create("transferFunction1D")
    tf.set_param("table", scene.tf.as_f32())
    tf.set_param("valueRange", (scene.tf.vmin, scene.tf.vmax))
    tf.commit()
    vol = d.create("volume")
    vol.set_param("field", sf)
    vol.set_param("transferFunction", tf)
    vol.commit()
    world = d.create("world")
    world.set_param("volumes", [vol])
    world.commit()
    renderer = d.create("renderer")
    renderer.set_param("background", scene.background)
    renderer.set_param("composite", composite)
    renderer.commit()
    camera = d.create("camera")
    frame = d.create("frame")
    frame.set_param("world", world)
    frame.set_param("camera", camera)
    frame.set_param("renderer", renderer)
    return camera, frame


def _apply_and_render(camera, frame, cmd: dict):
    camera.set_param("position", tuple(cmd["pos"]))
    camera.set_param("direction", tuple(cmd["dir"]))
    camera.set_param("up", tuple(cmd["up"]))
    camera.set_param("fovY", float(cmd["fovy"]))
    camera.set_param("aspect", cmd["w"] / cmd["h"])
    camera.commit()
    frame.set_param("size", (cmd["w"], cmd["h"]))
    frame.commit()
    t0 = time.perf_counter()
    result = api.render_frame_collective(frame)
    return result, int(round((time.perf_counter() - t0) * 1e3))


def _refuse(sock: socketlib.socket) -> None:
    try:
        sock.sendall(encode_message(ControlMessage({"status": "busy"})))
    except OSError:
        pass
    finally:
        sock.close()


def serve_session(ep: RankEndpoint, scene: VolumeScene, options: Optional[ServeOptions] = None,
                  cuda=None) -> Optional[ServeReport]:
    """Collective: one thin-client session; the report comes back on rank 0."""
    options = options or ServeOptions()
    camera, frame = build_rank_objects(ep, scene, options.composite, cuda)
    if ep.rank != 0:
        while True:
            cmd = json.loads(ep.broadcast_from_root(None).decode("utf-8"))
            if cmd["cmd"] == "shutdown":
                return None
            _apply_and_render(camera, frame, cmd)
    report = ServeReport()
    listener = socketlib.socket(socketlib.AF_INET, socketlib.SOCK_STREAM)
    listener.setsockopt(socketlib.SOL_SOCKET, socketlib.SO_REUSEADDR, 1)
    listener.bind((options.host, options.port))
    listener.listen(4)
    listener.settimeout(0.05)
    if options.on_listening:
        options.on_listening(listener.getsockname())
    client: Optional[_Client] = None
    alive = True

    def shutdown_ranks() -> None:
        ep.broadcast_from_root(json.dumps({"cmd": "shutdown"}).encode("utf-8"))

    try:
        deadline = time.monotonic() + options.accept_timeout_secs
        while client is None:
            if time.monotonic() > deadline:
                shutdown_ranks()
                raise DprtError("no client connected before the accept deadline")
            try:
                sock, _ = listener.accept()
            except socketlib.timeout:
                continue
            client = _Client(sock)

        def refuser() -> None:
            while alive:
                try:
                    extra, _ = listener.accept()
                except socketlib.timeout:
                    continue
                except OSError:
                    return
                _refuse(extra)

        threading.Thread(target=refuser, daemon=True, name="dprt-busy").start()
        while True:
            update = client.take_latest()
            if update is None:
                if client.closed:
                    if client.error:
                        try:
                            client.send(ControlMessage({"error": client.error}))
                        except OSError:
                            pass
                    break
                time.sleep(_POLL)
                continue
            cmd = {"cmd": "frame", "pos": list(update.position), "dir": list(update.view_dir),
                   "up": list(update.up), "fovy": update.fov_y, "w": update.width, "h": update.height}
            ep.broadcast_from_root(json.dumps(cmd).encode("utf-8"))
            result, millis = _apply_and_render(camera, frame, cmd)
            buf = api.map_frame(frame)
            client.send(FrameMessage(buf.width, buf.height, buf.sequence, millis, buf.pixels))
            report.frames_sent += 1
            report.render_millis.append(millis)
            report.records.extend(result.stats.records)
        shutdown_ranks()
        return report
    finally:
        alive = False
        if client is not None:
            client.close()
        listener.close()
