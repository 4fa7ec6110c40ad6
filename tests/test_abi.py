"""The C-ABI library loads, exports every symbol include/dprt_cuda.h declares, and its struct layouts
match the ctypes mirrors.  No compute calls (CPU-only test)."""

from __future__ import annotations

import ctypes
import re
import shutil
import subprocess
from pathlib import Path

import pytest

from paper_2501_01628_b200 import _lib
from paper_2501_01628_b200.errors import DeviceError, NativeLibraryMissing, UsageError

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "dprt_cuda.h"


def _declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(dprt_\w+)\s*\(", text, re.M)))


def test_header_and_python_binding_agree():
    assert sorted(_lib.EXPORTS) == _declared()
    m = re.search(r"#define DPRT_ABI_VERSION (\d+)", HEADER.read_text())
    assert int(m.group(1)) == _lib.ABI_VERSION


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.dprt_cuda_version() == _lib.ABI_VERSION
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    for name in _declared():
        assert re.search(rf"\bT {name}\b", out), f"{name} not exported with C linkage"


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_struct_layouts_match_ctypes(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text("""
#include <stdio.h>
#include <stddef.h>
#include "dprt_cuda.h"
#define F(T, m) printf(#T "." #m " %zu\\n", offsetof(T, m))
int main(void) {
  printf("DprtBrickDesc %zu\\n", sizeof(DprtBrickDesc)); F(DprtBrickDesc, ghost); F(DprtBrickDesc, origin); F(DprtBrickDesc, spacing);
  printf("DprtCamera %zu\\n", sizeof(DprtCamera)); F(DprtCamera, half_w); F(DprtCamera, half_h);
  printf("DprtFieldSpec %zu\\n", sizeof(DprtFieldSpec)); F(DprtFieldSpec, blobs);
  printf("DprtMarchParams %zu\\n", sizeof(DprtMarchParams)); F(DprtMarchParams, vmin); F(DprtMarchParams, ert); F(DprtMarchParams, tf_version); F(DprtMarchParams, row1); F(DprtMarchParams, counter_slot);
  return 0;
}
""")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = dict(line.rsplit(" ", 1) for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n") if line)
    mirrors = {"DprtBrickDesc": _lib.BrickDesc, "DprtCamera": _lib.Camera, "DprtFieldSpec": _lib.FieldSpec,
               "DprtMarchParams": _lib.MarchParams}
    for cname, ct in mirrors.items():
        assert int(got[cname]) == ctypes.sizeof(ct), cname
    for key, val in got.items():
        if "." in key:
            cname, field = key.split(".")
            assert getattr(mirrors[cname], field).offset == int(val), key


def test_argument_errors_map_to_usage_error():
    lib = _lib.lib()
    with pytest.raises(UsageError):
        _lib.check(lib.dprt_march(None, None, None, None, None, 8, 8, None), "dprt_march")
    bad = _lib.BrickDesc()
    bad.dims[:] = [4, 4, 4]
    bad.lo[:] = [2, 0, 0]
    bad.hi[:] = [1, 3, 3]
    bad.spacing[:] = [1.0, 1.0, 1.0]
    h = ctypes.c_void_p()
    with pytest.raises(UsageError, match="invalid on axis 0"):
        _lib.check(lib.dprt_brick_create(0, ctypes.byref(bad), ctypes.byref(h)), "dprt_brick_create")
    with pytest.raises(UsageError):
        _lib.check(lib.dprt_composite(0, None, 0, 0, None, 1, None, None, None), "dprt_composite")


def test_no_gpu_raises_device_error_not_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    good = _lib.BrickDesc()
    good.dims[:] = [4, 4, 4]
    good.hi[:] = [3, 3, 3]
    good.spacing[:] = [1.0, 1.0, 1.0]
    h = ctypes.c_void_p()
    with pytest.raises(DeviceError):
        _lib.check(_lib.lib().dprt_brick_create(0, ctypes.byref(good), ctypes.byref(h)), "dprt_brick_create")


def test_missing_library_is_loud(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setenv("DPRT_CUDA_LIB", str(tmp_path / "absent.so"))
    with pytest.raises(NativeLibraryMissing):
        _lib.lib()
