"""The C-ABI library builds, loads and exports every symbol include/jfftb200.h
declares (no compute calls: runs without a GPU)."""

import ctypes
import os
import re

import pytest

from paper_2508_02613_b200 import _native as N

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "jfftb200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(jfftb_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_binding_table():
    assert set(declared_symbols()) == set(N.EXPORTED)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(N.LIB_PATH):
        from paper_2508_02613_b200 import build
        build.build()
    lib = ctypes.CDLL(N.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.jfftb_version() == 100


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_errors_map_to_reference_exceptions():
    lib = N.load()
    # no GPU here: grid creation must fail loudly (never fall back to the CPU)
    out = ctypes.c_void_p()
    ns = (ctypes.c_int64 * 2)(8, 8)
    ls = (ctypes.c_double * 2)(1.0, 1.0)
    st = lib.jfftb_grid_create(2, ns, ls, 0, ctypes.byref(out))
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        assert st == N.OK
        lib.jfftb_grid_destroy(out)
    else:
        assert st != N.OK
        with pytest.raises((RuntimeError, ValueError)):
            N.check(st)
    # invalid dimension -> ValueError-class status, before touching CUDA
    st = lib.jfftb_grid_create(4, ns, ls, 0, ctypes.byref(out))
    assert st == N.EINVAL
    with pytest.raises(ValueError):
        N.check(st)
    with pytest.raises(N.SolverAbortError):
        N.check(N.ENONFINITE)
