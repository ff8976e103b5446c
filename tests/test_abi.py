"""CPU-side checks of the C ABI: the library loads and exports every symbol
that include/seisgpu.h declares, and the shim binds them all.  No compute."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "seisgpu.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sg_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2008_11778_b200 import build
    build.build()
    return ctypes.CDLL(build.LIB)


def test_every_declared_symbol_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_shim_binds_every_symbol():
    from paper_2008_11778_b200 import _lib
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_desc_layout_matches_header():
    from paper_2008_11778_b200 import _lib
    # 20 int32 fields (incl. reserved[4]) then 5 doubles
    assert ctypes.sizeof(_lib.SgDesc) == 20 * 4 + 5 * 8
    assert _lib.SgDesc.dx.offset == 80


def test_version_and_error_string(lib):
    from paper_2008_11778_b200 import _lib
    L = _lib.load()
    assert L.sg_version() == 2
    # argument validation needs no device: a null descriptor is rejected
    h = ctypes.c_void_p()
    rc = L.sg_create(None, ctypes.byref(h))
    assert rc == _lib.SG_ERR_ARG
    assert "null" in _lib.last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_sass_is_sm100a(lib):
    import shutil
    import subprocess
    from paper_2008_11778_b200 import build
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([cuobjdump, "--list-elf", build.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
