"""The C-ABI library loads and exports every symbol include/tgl.h declares (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tgl.h")
LIB = os.path.join(ROOT, "paper_2203_14883_b200", "libtgl.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^TGL_API\s+[\w\s\*]*?\b(tgl_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ("tgl_tcsr_build", "tgl_sample", "tgl_gather", "tgl_check", "tgl_strerror"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "run make / __graft_entry__.build() first"
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol():
    from paper_2203_14883_b200 import _lib
    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_host_only_calls_without_gpu():
    """Calls that do no device work: version, strerror, capacity and workspace queries."""
    import paper_2203_14883_b200 as tgl
    L = tgl._L
    assert L.tgl_abi_version() == 3
    assert L.tgl_strerror(-2) == b"node or row id out of range"
    b = ctypes.c_size_t()
    assert L.tgl_tcsr_build_workspace(1000, 50, 1, ctypes.byref(b)) == 0 and b.value > 0
    assert L.tgl_tcsr_build_workspace(2**31, 50, 1, ctypes.byref(b)) == -1   # E_s >= 2^32
    rc = (ctypes.c_int64 * 2)()
    ec = (ctypes.c_int64 * 2)()
    fan = (ctypes.c_int32 * 2)(10, 10)
    assert L.tgl_sample_capacity(600, 2, fan, 1, 1, float("inf"), rc, ec, ctypes.byref(b)) == 0
    assert list(rc) == [600, 6000] and list(ec) == [6000, 60000]
    assert L.tgl_sample_capacity(600, 2, fan, 3, 1, float("inf"), rc, ec, ctypes.byref(b)) == -1   # S>1, inf
    assert L.tgl_sample_capacity(600, 2, fan, 3, 1, 0.0, rc, ec, ctypes.byref(b)) == -1            # ts <= 0
    fan1 = (ctypes.c_int32 * 1)(1025)
    assert L.tgl_sample_capacity(600, 1, fan1, 1, 0, float("inf"), rc, ec, ctypes.byref(b)) == -1  # k > max
    assert L.tgl_shard_bucket_workspace(4000, 8, ctypes.byref(b)) == 0


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2203_14883_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "tgl_oracle" not in text, f
