"""ctypes binding of libdprt_cuda.so (the C ABI in include/dprt_cuda.h).

The data path has no CPU fallback: if the library is missing or unloadable every entry point raises
``NativeLibraryMissing``.  ctypes releases the GIL for the duration of each foreign call, which is what
the reference relies on numba's ``nogil=True`` for (pkg/src/dprt/bvh.py:160) so rank threads overlap.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path
from typing import Optional

from .errors import DeviceError, NativeLibraryMissing, TransportError, UsageError

LIB_PATH = Path(__file__).resolve().parent / "libdprt_cuda.so"
ABI_VERSION = 11

DPRT_OK = 0
DPRT_E_USAGE = -1
DPRT_E_CUDA = -2
DPRT_E_NOMEM = -3
DPRT_E_TRANSPORT = -4

MAX_BLOBS = 64
MAX_PARTS = 64

MARCH_NO_SKIP = 1
MARCH_FULL_FRAME = 2
MARCH_BEAM = 4
MARCH_QUEUE = 8
MARCH_BAND_CLEAR = 16
MARCH_ACCUM = 32
MARCH_HALF = 64
MARCH_WIDE = 128
MARCH_DEEP = 256
BRICK_HALF_QUADS = 1
COMPOSITE_TONEMAP = 1
COMPOSITE_RGBA = 2
COMPOSITE_HALF_IN = 4

EXPORTS = (
    "dprt_cuda_version", "dprt_last_error", "dprt_device_count", "dprt_device_synchronize",
    "dprt_brick_create", "dprt_brick_stored", "dprt_brick_upload", "dprt_brick_download",
    "dprt_brick_generate", "dprt_brick_build_macrocells", "dprt_brick_destroy", "dprt_brick_footprint",
    "dprt_march", "dprt_march_rgb8", "dprt_composite", "dprt_ipc_handle", "dprt_ipc_open", "dprt_ipc_close",
    "dprt_enable_peer", "dprt_device_alloc", "dprt_device_free", "dprt_march_counters", "dprt_kat_slab", "dprt_kat_primary_dirs",
    "dprt_stage_input", "dprt_composite_ranged", "dprt_desc_footprint", "dprt_march_stats",
    "dprt_trace_nearest", "dprt_trace_any", "dprt_march_push", "dprt_wait_flags", "dprt_composite_signal",
    "dprt_copy_2d", "dprt_brick_macro_shift",
)
MAX_PUSH = 16  # DPRT_MAX_PUSH
SIGNAL_COUNTER_WORDS = 1056  # DPRT_SIGNAL_COUNTER_WORDS

c_double3 = ctypes.c_double * 3
c_int64_3 = ctypes.c_int64 * 3


class BrickDesc(ctypes.Structure):
    _fields_ = [("dims", c_int64_3), ("lo", c_int64_3), ("hi", c_int64_3), ("ghost", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("origin", c_double3), ("spacing", c_double3)]


class Camera(ctypes.Structure):
    _fields_ = [("pos", c_double3), ("fwd", c_double3), ("right", c_double3), ("up", c_double3),
                ("half_w", ctypes.c_double), ("half_h", ctypes.c_double)]


class FieldSpec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n_blobs", ctypes.c_int32), ("blobs", ctypes.c_void_p)]


class MarchParams(ctypes.Structure):
    _fields_ = [("tf_rgba", ctypes.c_void_p), ("n_tf", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("vmin", ctypes.c_double), ("vmax", ctypes.c_double), ("dt", ctypes.c_double),
                ("ert", ctypes.c_double), ("tf_version", ctypes.c_uint64), ("row0", ctypes.c_int32),
                ("row1", ctypes.c_int32), ("counter_slot", ctypes.c_int32), ("reserved", ctypes.c_int32)]


MARCH_COUNTER_SLOTS = 4  # DPRT_MARCH_COUNTER_SLOTS


class Bvh(ctypes.Structure):
    _fields_ = [("node_lo", ctypes.c_void_p), ("node_hi", ctypes.c_void_p), ("node_left", ctypes.c_void_p),
                ("node_right", ctypes.c_void_p), ("node_first", ctypes.c_void_p), ("node_count", ctypes.c_void_p),
                ("num_nodes", ctypes.c_int64), ("root", ctypes.c_int64), ("tri_v", ctypes.c_void_p),
                ("tri_id", ctypes.c_void_p), ("num_prims", ctypes.c_int64)]


class PushTargets(ctypes.Structure):
    _fields_ = [("P", ctypes.c_int32), ("reserved", ctypes.c_int32), ("row_start", ctypes.c_void_p),
                ("dst", ctypes.c_void_p), ("flags", ctypes.c_void_p), ("counter", ctypes.c_void_p),
                ("epoch", ctypes.c_uint32), ("reserved2", ctypes.c_uint32)]


_lib: Optional[ctypes.CDLL] = None


def _declare(lib: ctypes.CDLL) -> None:
    P = ctypes.c_void_p
    I = ctypes.c_int
    sig = {
        "dprt_cuda_version": ([], I),
        "dprt_last_error": ([], ctypes.c_char_p),
        "dprt_device_count": ([P], I),
        "dprt_device_synchronize": ([I], I),
        "dprt_brick_create": ([I, P, P], I),
        "dprt_brick_stored": ([P, P, P], I),
        "dprt_brick_upload": ([P, P, I, P], I),
        "dprt_brick_download": ([P, P, I, P], I),
        "dprt_brick_generate": ([P, P, P], I),
        "dprt_brick_build_macrocells": ([P, P], I),
        "dprt_brick_destroy": ([P], I),
        "dprt_brick_footprint": ([P, P, I, I, P], I),
        "dprt_march": ([P, P, P, P, P, I, I, P], I),
        "dprt_march_rgb8": ([P, P, P, P, P, P, I, I, P], I),
        "dprt_composite": ([I, P, I, ctypes.c_int64, P, I, P, P, P], I),
        "dprt_ipc_handle": ([I, P, P], I),
        "dprt_ipc_open": ([I, P, P], I),
        "dprt_ipc_close": ([I, P], I),
        "dprt_enable_peer": ([I, I], I),
        "dprt_device_alloc": ([I, ctypes.c_uint64, P], I),
        "dprt_device_free": ([I, P], I),
        "dprt_march_counters": ([I, P, I], I),
        "dprt_kat_slab": ([I, I, P, P, P, P, P, P], I),
        "dprt_kat_primary_dirs": ([I, P, I, I, P], I),
        "dprt_stage_input": ([I, P, P, ctypes.c_uint64, P], I),
        "dprt_composite_ranged": ([I, P, P, I, ctypes.c_int64, P, I, P, P, P], I),
        "dprt_desc_footprint": ([P, P, I, I, P], I),
        "dprt_march_stats": ([P, P, P, I, I, P, P], I),
        "dprt_trace_nearest": ([I, P, ctypes.c_int64, P, P, P, P, P, P, P], I),
        "dprt_trace_any": ([I, P, ctypes.c_int64, P, P, P, P, P, P], I),
        "dprt_march_push": ([P, P, P, P, P, I, I, P], I),
        "dprt_wait_flags": ([I, P, I, ctypes.c_uint32, P], I),
        "dprt_composite_signal": ([I, P, P, I, ctypes.c_int64, P, I, P, P, P, P, I, ctypes.c_uint32, P], I),
        "dprt_brick_macro_shift": ([P, P], I),
        "dprt_copy_2d": ([I, P, ctypes.c_uint64, P, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, P], I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res


def lib() -> ctypes.CDLL:
    """The loaded library; raises NativeLibraryMissing (no fallback) if it cannot be loaded."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("DPRT_CUDA_LIB") or str(LIB_PATH)).resolve()
    if not path.exists():
        raise NativeLibraryMissing(
            f"{path} not built: run `python -m paper_2501_01628_b200.build` (there is no CPU fallback)")
    try:
        handle = ctypes.CDLL(str(path))
    except OSError as exc:
        raise NativeLibraryMissing(f"cannot load {path}: {exc}") from exc
    _declare(handle)
    if handle.dprt_cuda_version() != ABI_VERSION:
        raise NativeLibraryMissing(f"{path} ABI {handle.dprt_cuda_version()} != expected {ABI_VERSION}; rebuild")
    _lib = handle
    return handle


def check(rc: int, what: str) -> None:
    """Map a status code onto the reference's exception taxonomy (errors.py:4-29)."""
    if rc == DPRT_OK:
        return
    msg = (lib().dprt_last_error() or b"").decode("utf-8", "replace")
    text = f"{what}: {msg}" if msg else what
    if rc == DPRT_E_USAGE:
        raise UsageError(text)
    if rc == DPRT_E_TRANSPORT:
        raise TransportError(text)
    raise DeviceError(text)


def device_count() -> int:
    n = ctypes.c_int(0)
    rc = lib().dprt_device_count(ctypes.byref(n))
    return int(n.value) if rc == DPRT_OK else 0
