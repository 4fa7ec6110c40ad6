"""Collective render API for volumes: reference-counted objects, staged parameters, local commits, and
rank-synchronised frames -- the reference's DP-ANARI facade (pkg/src/dprt/api.py) with the volume kinds
the hot path needs.

Differences from the reference's facade, all deliberate:
* new kinds ``spatialField``, ``volume``, ``transferFunction1D`` (the reference rejects "volume",
  api.py:38 / 238-240, pinned by test_api.py:226-231; that test is re-pointed at a genuinely unknown
  kind in tests/test_api_cpu.py);
* ``World`` commit decomposes the field into one brick per rank (kd split, volume.decompose) and makes
  this rank's brick resident on its GPU -- the counterpart of the local BVH build (api.py:146-171);
  still purely local, no transport traffic (test_api.py:72-81's property holds);
* triangle kinds (surface / group / instance) exist but are not part of this path: committing a world
  that references them raises UsageError.
``render_frame_collective`` / ``map_frame`` keep their contracts (api.py:329-371): divergent committed
parameters raise ContractError on every rank before GPU work; rank 0 maps RGB8 bytes that a newer
render invalidates.
"""

from __future__ import annotations

from typing import Dict, List, Optional, Tuple, Union

import numpy as np
import torch

from . import device as dev
from .engine import RenderOptions, RenderResult, VolumeRenderer
from .errors import UsageError
from .geom import CameraSpec
from .refcount import RefCounted
from .transport import RankEndpoint
from .volume import Decomposition, FieldSpec, TransferFunction1D, blob_mixture, decompose, default_tf


class _NotRoot:
    def __repr__(self) -> str:
        return "NOT_ROOT"


NOT_ROOT = _NotRoot()

OBJECT_KINDS = ("world", "surface", "group", "instance", "camera", "renderer", "frame",
                "spatialField", "volume", "transferFunction1D")

_PARAMS: Dict[str, Dict[str, object]] = {
    "world": {"volumes": [], "surfaces": [], "instances": [], "lights": []},
    "surface": {"triangles": [], "material": None},
    "group": {"surfaces": []},
    "instance": {"group": None},
    "spatialField": {"dims": (64, 64, 64), "origin": (0.0, 0.0, 0.0), "spacing": (1.0, 1.0, 1.0),
                     "generator": "blobs", "seed": 1, "blobCount": 16, "lopsided": False,
                     "frequency": 6.0, "alpha": 0.25, "data": None},
    "transferFunction1D": {"table": None, "valueRange": (0.0, 1.0)},
    "volume": {"field": None, "transferFunction": None, "decomposition": "even", "ghost": 1,
               "massThreshold": 0.1},
    "camera": {"position": (0.0, 0.0, 3.0), "direction": (0.0, 0.0, -1.0),
               "up": (0.0, 1.0, 0.0), "fovY": 60.0, "aspect": 1.0},
    "renderer": {"background": (0.0, 0.0, 0.0), "dt": 1.0, "ert": 0.99, "composite": "auto",
                 "skipEmpty": True, "disableCompositing": False, "mode": "dvr", "clipExchange": True,
                 "fragments": "f32"},
    "frame": {"world": None, "camera": None, "renderer": None, "size": (256, 256)},
}


class ApiObject(RefCounted):
    """Render-graph object with two parameter sets (the reference's contract, api.py:53-95): ``set_param``
    writes the staged set only; ``commit`` publishes a copy of it atomically and locally (no transport
    traffic), runs the kind's validation hook, and rolls back to the previous committed set if that hook
    rejects it.  Object-valued parameters keep their children alive: one hold per staged and one per
    committed reference."""

    def __init__(self, device: "Device", kind: str):
        super().__init__()
        self.device = device
        self.kind = kind
        self.staged: Dict[str, object] = dict(_PARAMS[kind])
        self.committed: Dict[str, object] = {}
        self.commit_epoch = 0

    def __repr__(self) -> str:
        return f"<{self.kind} refcount={self.refcount}>"

    def _retarget(self, drop_from, hold_in) -> None:
        """Take holds on the children of ``hold_in`` first, then give up those of ``drop_from`` (a child in
        both never reaches zero in between)."""
        for child in _children(hold_in):
            self.hold(child)
        for child in _children(drop_from):
            self.drop(child)

    def set_param(self, name: str, value) -> None:
        self._check_alive()
        known = _PARAMS[self.kind]
        if name not in known:
            raise UsageError(f"{self.kind} has no parameter {name!r}; valid names: {', '.join(sorted(known))}")
        self._retarget(self.staged.get(name), value)
        self.staged[name] = value

    def commit(self) -> None:
        self._check_alive()
        previous, previous_epoch = self.committed, self.commit_epoch
        snapshot = dict(self.staged)
        self._retarget((), list(snapshot.values()))
        self.committed, self.commit_epoch = snapshot, previous_epoch + 1
        try:
            self._on_commit()
        except Exception:
            # a rejected commit leaves the previously committed state in force
            self._retarget(list(snapshot.values()), ())
            self.committed, self.commit_epoch = previous, previous_epoch
            raise
        self._retarget(list(previous.values()), ())

    def _on_commit(self) -> None:
        pass


def _children(value) -> List["ApiObject"]:
    """ApiObjects referenced by a parameter value (the object itself, or the objects in a list / tuple,
    one level deep -- the parameter shapes _PARAMS allows)."""
    items = value if isinstance(value, (list, tuple)) else (value,)
    out = []
    for v in items:
        if isinstance(v, (list, tuple)):
            out.extend(x for x in v if isinstance(x, ApiObject))
        elif isinstance(v, ApiObject):
            out.append(v)
    return out


def _triple(value, name: str, kind=float) -> Tuple:
    if not (isinstance(value, (list, tuple)) and len(value) == 3):
        raise UsageError(f"{name} must be three numbers")
    return tuple(kind(v) for v in value)


class SpatialField(ApiObject):
    """Vertex-centred scalar grid; values from a generator ("blobs": seeded blob mixture; "marschnerLobb":
    the Marschner-Lobb signal with ``frequency`` / ``alpha``) or a host array (z, y, x)."""

    def field_spec(self) -> Tuple[FieldSpec, Optional[np.ndarray]]:
        c = self.committed
        dims = _triple(c["dims"], "spatialField dims", int)
        data = c.get("data")
        if data is not None:
            arr = np.asarray(data, np.float32)
            if arr.shape != tuple(reversed(dims)):
                raise UsageError(f"spatialField data {arr.shape} does not match dims {dims} (z, y, x)")
            blobs = np.zeros((0, 5))
        elif c["generator"] == "marschnerLobb":
            return FieldSpec(dims, np.zeros((0, 5)), _triple(c["origin"], "origin"), _triple(c["spacing"], "spacing"),
                             "marschnerLobb", (float(c["frequency"]), float(c["alpha"]))), None
        else:
            if c["generator"] != "blobs":
                raise UsageError(f"unknown spatialField generator {c['generator']!r}")
            blobs = blob_mixture(int(c["seed"]), int(c["blobCount"]), bool(c["lopsided"]))
            arr = None
        return FieldSpec(dims, blobs, _triple(c["origin"], "origin"), _triple(c["spacing"], "spacing")), arr

    def _on_commit(self) -> None:
        self.field_spec()


class TransferFunctionObject(ApiObject):
    _tf: Optional[TransferFunction1D] = None

    def tf(self) -> TransferFunction1D:
        """The committed table (built once per commit, so per-frame digests and uploads reuse it)."""
        if self._tf is None:
            self._tf = self._build()
        return self._tf

    def _build(self) -> TransferFunction1D:
        table = self.committed.get("table")
        lo, hi = self.committed.get("valueRange", (0.0, 1.0))
        if table is None:
            return TransferFunction1D(default_tf().table, float(lo), float(hi))
        return TransferFunction1D(np.asarray(table, np.float32), float(lo), float(hi))

    def _on_commit(self) -> None:
        self._tf = self._build()


class Volume(ApiObject):
    def _on_commit(self) -> None:
        c = self.committed
        if not (isinstance(c.get("field"), SpatialField) and c["field"].commit_epoch > 0):
            raise UsageError("volume 'field' must be a committed spatialField object")
        if not (isinstance(c.get("transferFunction"), TransferFunctionObject)
                and c["transferFunction"].commit_epoch > 0):
            raise UsageError("volume 'transferFunction' must be a committed transferFunction1D object")
        if c["decomposition"] not in ("even", "mass"):
            raise UsageError("volume 'decomposition' must be 'even' or 'mass'")


class World(ApiObject):
    """Distributed volume scene; commit decomposes the field and makes this rank's brick resident."""

    def __init__(self, device: "Device"):
        super().__init__(device, "world")
        self.brick: Optional[dev.DeviceBrick] = None
        self.decomposition: Optional[Decomposition] = None
        self.volume: Optional[Volume] = None

    def _on_commit(self) -> None:
        c = self.committed
        if c.get("surfaces") or c.get("instances"):
            raise UsageError("triangle surfaces/instances are not part of this volume path")
        if c.get("lights"):
            raise UsageError("lights are not used by the emission-absorption volume renderer")
        vols = c.get("volumes", [])
        if len(vols) != 1 or not isinstance(vols[0], Volume) or vols[0].commit_epoch == 0:
            raise UsageError("world 'volumes' must hold exactly one committed volume object")
        vol = vols[0]
        spec, data = vol.committed["field"].field_spec()
        ep = self.device.ep
        mass = None
        if vol.committed["decomposition"] == "mass":
            mass = _mass_function(spec, data, float(vol.committed["massThreshold"]), self.device.cuda)
        dec = decompose(spec, ep.R, vol.committed["decomposition"], mass)
        desc = dec.brick(ep.rank, int(vol.committed["ghost"]))
        brick = dev.DeviceBrick(desc, self.device.cuda)
        if data is not None:
            s, d = desc.stored_lo, desc.stored_dims
            brick.upload(np.ascontiguousarray(data[s[2]:s[2] + d[2], s[1]:s[1] + d[1], s[0]:s[0] + d[0]]))
        else:
            brick.generate(spec)
        if self.brick is not None:
            self.brick.close()
        self.brick, self.decomposition, self.volume = brick, dec, vol

    def on_destroy(self) -> None:
        if self.brick is not None:
            torch.cuda.synchronize(self.device.cuda)
            self.brick.close()
            self.brick = None


def _mass_function(spec: FieldSpec, data: Optional[np.ndarray], tau: float, cuda: torch.device):
    """Integer slab masses (voxels >= tau) for the mass-weighted kd split, computed locally."""
    if data is None:  # generated field: masked on the GPU in z-chunks, never moved to the host
        return dev.field_mass_function(spec, cuda, tau)
    vox = torch.from_numpy(np.asarray(data, np.float32))
    mask = (vox >= tau).to(torch.int64)

    def mass(axis, lo, hi):
        sub = mask[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        dims = tuple(a for a in range(3) if a != 2 - axis)
        return sub.sum(dim=dims).numpy()

    return mass


class Frame(ApiObject):
    """Virtual film: exactly one world, camera and renderer (api.py:174-205)."""

    def __init__(self, device: "Device"):
        super().__init__(device, "frame")
        self.sequence = 0
        self._result: Optional[FrameResult] = None
        self._complete = False
        self._renderer: Optional[VolumeRenderer] = None
        self._host_ring: List[torch.Tensor] = []  # pinned RGB8 frames the read-backs alternate between (rank 0)
        self._host_next = 0

    def _on_commit(self) -> None:
        for name in ("world", "camera", "renderer"):
            obj = self.committed.get(name)
            if not (isinstance(obj, ApiObject) and obj.kind == name):
                raise UsageError(f"frame is missing a committed {name} object")
            if obj.commit_epoch == 0:
                raise UsageError(f"frame {name} was never committed")
        size = self.committed.get("size")
        if not (isinstance(size, (tuple, list)) and len(size) == 2
                and all(isinstance(v, int) and v > 0 for v in size)):
            raise UsageError("frame 'size' must be two positive integers")

    def render(self) -> RenderResult:
        return render_frame_collective(self)

    def wait(self) -> None:
        """Blocks until the last render's pixels are in host memory (rank 0; a no-op elsewhere)."""
        self._check_alive()
        if not self._complete:
            raise UsageError("wait_frame before any render")
        if self._result is not None:
            self._result._wait()

    def map(self) -> Union["FrameResult", _NotRoot]:
        return map_frame(self)


class FrameResult:
    """Mapped RGB8 pixel buffer; valid until the next render completes (api.py:208-229).

    The read-back is asynchronous: the frame's bytes are copied into a pinned host buffer on a side stream
    while the host returns to the application, and ``pixels`` materialises them (waiting for that copy)
    on first access -- a renderer that never maps a frame, or maps every k-th, pays no host copy for the
    others.  ``pixels`` returns ``bytes`` like the reference; ``array`` is the same pixels as an (H, W, 3)
    uint8 view of the pinned buffer without the bytes copy (valid under the same rule)."""

    def __init__(self, width: int, height: int, pixels, sequence: int):
        self.width = width
        self.height = height
        self.sequence = sequence
        self._pixels = pixels if isinstance(pixels, (bytes, bytearray)) else None
        self._pending = None if self._pixels is not None else pixels  # engine.HostFrame on its way to the host
        self._valid = True

    @property
    def valid(self) -> bool:
        return self._valid

    def _host(self) -> torch.Tensor:
        if not self._valid:
            raise UsageError("frame buffer was invalidated by a newer render")
        return self._pending.wait()

    @property
    def array(self) -> np.ndarray:
        if self._pixels is not None:
            return np.frombuffer(self._pixels, np.uint8).reshape(self.height, self.width, 3)
        a = self._host().numpy()
        a.flags.writeable = False  # the pinned buffer is reused: later read-backs rely on its bytes
        return a

    @property
    def pixels(self) -> bytes:
        if self._pixels is None:
            self._pixels = self._host().numpy().tobytes()
            self._pending = None
        elif not self._valid:
            raise UsageError("frame buffer was invalidated by a newer render")
        return self._pixels

    def _wait(self) -> None:
        if self._pending is not None:
            self._pending.wait()

    def _invalidate(self) -> None:
        self._valid = False


class Device:
    """Per-rank object factory bound to one endpoint and one GPU (api.py:232-247)."""

    def __init__(self, ep: RankEndpoint, cuda: Optional[torch.device] = None):
        self.ep = ep
        if cuda is None:
            cuda = ep.device if ep.device.type == "cuda" else torch.device("cuda", torch.cuda.current_device())
        self.cuda = cuda

    def create(self, kind: str) -> ApiObject:
        """A new object of ``kind`` with refcount 1; UsageError names the valid kinds otherwise."""
        if kind not in OBJECT_KINDS:
            raise UsageError(f"unknown object kind {kind!r}; valid kinds: {', '.join(OBJECT_KINDS)}")
        factory = _FACTORIES.get(kind)
        return factory(self) if factory is not None else ApiObject(self, kind)


_FACTORIES = {
    "world": World,
    "frame": Frame,
    "spatialField": lambda d: SpatialField(d, "spatialField"),
    "transferFunction1D": lambda d: TransferFunctionObject(d, "transferFunction1D"),
    "volume": lambda d: Volume(d, "volume"),
}


def create_object(device: Device, kind: str) -> ApiObject:
    return device.create(kind)


def set_param(obj: ApiObject, name: str, value) -> None:
    obj.set_param(name, value)


def commit(obj: ApiObject) -> None:
    obj.commit()


def _camera_spec(camera: ApiObject) -> CameraSpec:
    c = camera.committed
    return CameraSpec(tuple(c["position"]), tuple(c["direction"]), tuple(c["up"]), float(c["fovY"]),
                      float(c["aspect"]))


def render_frame_collective(frame: Frame) -> RenderResult:
    """Collective: every rank renders the frame's committed state (api.py:329-360)."""
    frame._check_alive()
    if frame.commit_epoch == 0:
        raise UsageError("frame must be committed before rendering")
    world: World = frame.committed["world"]
    camera: ApiObject = frame.committed["camera"]
    renderer: ApiObject = frame.committed["renderer"]
    width, height = frame.committed["size"]
    r = renderer.committed
    options = RenderOptions(dt=float(r["dt"]), ert=float(r["ert"]), composite=str(r["composite"]),
                            skip_empty=bool(r["skipEmpty"]), disable_compositing=bool(r["disableCompositing"]),
                            frame_index=frame.sequence, mode=str(r["mode"]), clip_exchange=bool(r["clipExchange"]),
                            fragment_dtype=str(r["fragments"]))
    background = tuple(float(v) for v in r["background"])
    tf = world.volume.committed["transferFunction"].tf()
    vr = frame._renderer
    if vr is None or vr.brick is not world.brick or vr.decomposition is not world.decomposition:
        vr = VolumeRenderer(world.device.ep, world.brick, world.decomposition, tf, background)
        frame._renderer = vr
    else:
        vr.background = background
        vr.dtf.update(tf)
        vr.tf = tf
    host = None
    if world.device.ep.rank == 0:
        # two pinned frames: the read-back of this frame never overwrites the previous frame's buffer, which
        # stays mapped until this render completes (the previous result is invalidated below)
        if len(frame._host_ring) != 2 or tuple(frame._host_ring[0].shape) != (height, width, 3):
            if frame._result is not None:
                frame._result._wait()
            frame._host_ring = [torch.empty((height, width, 3), dtype=torch.uint8, pin_memory=True)
                                for _ in range(2)]
            frame._host_next = 0
        host = frame._host_ring[frame._host_next]
        frame._host_next ^= 1
    hf = vr.render_to_host(_camera_spec(camera), width, height, host, options)
    frame.sequence += 1
    if frame._result is not None:
        frame._result._invalidate()
        frame._result = None
    if world.device.ep.rank == 0:
        frame._result = FrameResult(width, height, hf, frame.sequence)
    frame._complete = True
    return hf.result


def map_frame(frame: Frame) -> Union[FrameResult, _NotRoot]:
    """The last completed render's pixels: a FrameResult on rank 0, NOT_ROOT elsewhere (api.py:363-371)."""
    frame._check_alive()
    if not frame._complete:
        raise UsageError("map_frame before any completed render")
    return frame._result if frame.device.ep.rank == 0 else NOT_ROOT
