"""The C ABI library without a GPU: it loads, exports every declared symbol, its
struct layouts match the ctypes mirror, and device calls fail cleanly."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2605_25040_b200 import _lib
from paper_2605_25040_b200 import build as pkg_build

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "cafs_b200.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        pkg_build.build()
    return _lib.load()


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|uint64_t|const char\*)\s+(cafs_\w+)\(", text, re.M)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert "cafs_sort_i64" in syms and "cafs_emit_i64" in syms
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table and header disagree"


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (cafs_\w+)$", out, re.M))
    missing = set(declared_symbols()) - exported
    assert not missing, f"not exported: {missing}"
    for name in declared_symbols():
        assert getattr(lib, name) is not None


def test_abi_version_and_status_strings(lib):
    assert lib.cafs_abi_version() == 2
    assert lib.cafs_status_string(0) == b"ok"
    assert b"invalid" in lib.cafs_status_string(-1)


def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include "cafs_b200.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                   "int main(){printf(\"%zu %zu %zu %zu %zu\\n\", sizeof(cafs_estimate_t),"
                   " sizeof(cafs_decision_t), sizeof(cafs_telemetry_t),"
                   " offsetof(cafs_telemetry_t, stage_ms), offsetof(cafs_telemetry_t,"
                   " kernels_launched));return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [ctypes.sizeof(_lib.Estimate), ctypes.sizeof(_lib.Decision),
            ctypes.sizeof(_lib.Telemetry), _lib.Telemetry.stage_ms.offset,
            _lib.Telemetry.kernels_launched.offset]
    assert got == want


def test_device_calls_fail_cleanly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    rc = lib.cafs_ctx_create(0, ctypes.byref(h))
    assert rc != 0 and not h.value
    assert lib.cafs_sort_i64(None, None, 0, 1, 1, 0, None, None) == _lib.EINVAL
