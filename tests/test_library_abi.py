"""CPU: the C-ABI library builds, loads, and exports exactly the declared API.

No compute calls here — without a GPU every compute entry point must fail
loudly (there is no CPU fallback), which is checked too.
"""

import ctypes as C
import re
from pathlib import Path

import pytest

from paper_1302_0120_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "phasemask_b200.h"


def declared_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(?:int|const char \*)\s*\*?\s*(pm_\w+)\s*\(", text)))


def test_header_declares_api():
    syms = declared_symbols()
    assert "pm_solve" in syms and "pm_fft2" in syms and "pm_plan_create" in syms
    assert len(syms) >= 20


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, f"not exported: {missing}"


def test_python_binding_covers_the_header():
    assert set(declared_symbols()) <= set(_lib.SIGNATURES)


def test_library_is_sm100a_and_links_no_torch():
    so = _lib.LIB_PATH.read_bytes()
    assert b"sm_100a" in so or b"sm_100" in so
    assert b"libtorch" not in so


def test_version_and_device_query():
    lib = _lib.load()
    assert lib.pm_version() >= 100
    n = C.c_int(-1)
    assert lib.pm_device_count(C.byref(n)) == 0
    assert n.value >= 0


def test_errors_without_gpu_are_loud():
    if _lib.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.Plan(64, 64, 0)
    with pytest.raises(RuntimeError):
        _lib.norm2(__import__("numpy").ones(4))


def test_invalid_arguments_rejected_before_device():
    lib = _lib.load()
    h = C.c_void_p()
    assert lib.pm_plan_create(0, 110, 64, 0, 1, C.byref(h)) == _lib.PM_ERR_UNSUPPORTED   # factor 11
    assert "prime factors 2, 3, 5, 7" in _lib.last_error()
    assert lib.pm_plan_create(0, 64, 64, 7, 1, C.byref(h)) == _lib.PM_ERR_ARG
    assert lib.pm_plan_create(0, 8192, 64, 0, 1, C.byref(h)) == _lib.PM_ERR_UNSUPPORTED
