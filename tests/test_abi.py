"""The C-ABI library: builds, loads without a GPU, exports every symbol
declared in include/ttagg_b200.h; argument validation paths that need no
device.  (No compute calls here — those are in the -m gpu tests.)"""

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_1905_09071_b200 import _lib

HEADER = os.path.join(ROOT, "include", "ttagg_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ttagg_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.EXPORTED_SYMBOLS, f"{name} has no ctypes signature"
    assert set(_lib.EXPORTED_SYMBOLS) == set(names)


def test_shared_object_is_sm100a_native():
    """The fatbin carries sm_100a SASS (no PTX-only / other-arch fallback)."""
    import subprocess

    cuobjdump = "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_version_and_geometry():
    lib = _lib.load()
    assert lib.ttagg_version() >= 100
    assert _lib.geometry(1 << 20) == (1 << 20, 4096, 256)
    assert _lib.geometry(4096) == (4096, 16, 256)
    assert _lib.geometry(2) == (64, 4, 16)
    np_, n1, n2 = _lib.geometry(5000)
    assert np_ == 8192 and n1 * n2 == np_


def test_geometry_rejects_bad_sizes():
    out = (ctypes.c_int64 * 3)()
    lib = _lib.load()
    assert lib.ttagg_geometry(1, out) == _lib.TTAGG_ERR_ARG
    assert "length >= 2" in _lib.lib_error()
    assert lib.ttagg_geometry((1 << 20) + 1, out) == _lib.TTAGG_ERR_UNSUPPORTED


def test_null_arguments_are_rejected_without_crashing():
    lib = _lib.load()
    assert lib.ttagg_ctx_create(0, None) == _lib.TTAGG_ERR_ARG
    assert lib.ttagg_kernel_info(None, None) == _lib.TTAGG_ERR_ARG
    assert lib.ttagg_rhs(None, None, 0, None, None, None, None, 0, None) == _lib.TTAGG_ERR_ARG
    assert lib.ttagg_kernel_free(None) == _lib.TTAGG_OK
    assert lib.ttagg_ctx_destroy(None) == _lib.TTAGG_OK
