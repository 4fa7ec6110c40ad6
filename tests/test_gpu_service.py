"""Thin-client streaming of GPU frames over TCP (service.serve_session) with 2 rank threads on one GPU."""

from __future__ import annotations

import socket
import threading
import time

import numpy as np
import pytest

from paper_2501_01628_b200.geom import auto_camera
from paper_2501_01628_b200.protocol import (CameraUpdateMessage, ControlMessage, FrameMessage, StreamSplitter,
                                            decode_payload, encode_message)
from paper_2501_01628_b200.scene import VolumeScene
from paper_2501_01628_b200.service import ServeOptions, serve_session
from paper_2501_01628_b200.transport import run_collective
from paper_2501_01628_b200.volume import blob_field, default_tf

pytestmark = pytest.mark.gpu


def _recv_messages(sock, want, timeout=60.0):
    split = StreamSplitter()
    out = []
    sock.settimeout(timeout)
    while len(out) < want:
        chunk = sock.recv(1 << 20)
        if not chunk:
            break
        split.feed(chunk)
        out.extend(decode_payload(k, p) for k, p in split.messages())
    return out


def test_serve_streams_frames_latest_wins_and_refuses_second_client(cuda_device):
    f = blob_field((48, 48, 48), seed=2)
    scene = VolumeScene(f, default_tf(), (0.05, 0.06, 0.08), generator={"generator": "blobs", "seed": 2,
                                                                       "blobCount": 16, "lopsided": False})
    W, H = 96, 64
    cam = auto_camera(f.bounds(), W, H)
    addr = {}
    ready = threading.Event()
    client_out = {}

    def on_listening(a):
        addr["a"] = a
        ready.set()

    def client():
        ready.wait(60)
        s = socket.create_connection(addr["a"])
        first = CameraUpdateMessage(cam.position, cam.view_dir, cam.up, 45.0, W, H)
        s.sendall(encode_message(first))
        msgs = _recv_messages(s, 1)
        # burst of updates: at least the newest one must be rendered
        for fov in (30.0, 35.0, 40.0):
            s.sendall(encode_message(CameraUpdateMessage(cam.position, cam.view_dir, cam.up, fov, W, H)))
        # a second client is refused while the session runs
        s2 = socket.create_connection(addr["a"])
        client_out["busy"] = _recv_messages(s2, 1)
        s2.close()
        got = msgs
        while True:  # drain until the server goes quiet
            try:
                more = _recv_messages(s, 1, timeout=3.0)
            except socket.timeout:
                break
            if not more:
                break
            got.extend(more)
        client_out["frames"] = got
        s.close()

    th = threading.Thread(target=client, daemon=True)
    th.start()
    reports = run_collective(2, lambda ep: serve_session(ep, scene, ServeOptions(on_listening=on_listening),
                                                         cuda=cuda_device), device=cuda_device)
    th.join(30)
    frames = [m for m in client_out["frames"] if isinstance(m, FrameMessage)]
    assert frames and all(m.width == W and m.height == H and len(m.pixels) == W * H * 3 for m in frames)
    assert reports[0].frames_sent == len(frames) and reports[1] is None
    assert 2 <= len(frames) <= 4  # the burst of 3 updates coalesced to at most 3 renders
    assert client_out["busy"] == [ControlMessage({"status": "busy"})]
    img = np.frombuffer(frames[-1].pixels, np.uint8).reshape(H, W, 3)
    assert img.std() > 1.0  # a real image, not a cleared buffer
