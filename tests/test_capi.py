"""C-ABI checks that need no GPU: the library builds for sm_100a, loads, and
exports exactly what include/paball_b200.h declares."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "paball_b200.h")


def declared_symbols():
    text = open(HEADER, encoding="utf-8").read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pab_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2601_00551_b200 import _build
    return _build.build()


def test_header_declares_the_path(lib_path):
    syms = declared_symbols()
    for need in ("pab_forward", "pab_adjoint", "pab_residual", "pab_grad_finalize", "pab_pack",
                 "pab_adam", "pab_compact", "pab_decimate", "pab_sumsq_diff_f64"):
        assert need in syms


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (pab_[a-z0-9_]+)", out))
    assert exported == set(declared_symbols())


def test_binding_matches_header(lib_path):
    from paper_2601_00551_b200 import _lib
    assert set(_lib.EXPORTED) == set(declared_symbols())
    lib = _lib.load(lib_path)
    assert lib.pab_version() == 100
    a, b, g = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    lib.pab_record_sizes(ctypes.byref(a), ctypes.byref(b), ctypes.byref(g))
    assert (a.value, b.value, g.value) == (16, 16, 48)


def test_library_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_bad_arguments_return_1_without_gpu(lib_path):
    from paper_2601_00551_b200 import _lib
    lib = _lib.load(lib_path)
    # null pointers are rejected before any CUDA call
    assert lib.pab_pack(None, None, None, None, 10, None, None, None, None) == 1
    assert lib.pab_compact(None, 10, 0, None, None, None, None) == 1
    assert lib.pab_decimate(None, 1, 4, 0, None, None) == 1


def test_record_length_limit(lib_path):
    """Sample indices are rounded with FP32 magic constants (pab_common.cuh):
    records beyond 2^21 full-rate samples are rejected at the boundary, before
    any CUDA call, and by the host acquisition type."""
    from paper_2601_00551_b200 import _lib
    from paper_2601_00551_b200 import engine as E
    lib = _lib.load(lib_path)
    buf = (ctypes.c_double * 64)()
    p = ctypes.cast(buf, ctypes.c_void_p)
    n_out = (1 << 20) + 1   # x f = 2 -> 2^21 + 2 full-rate samples
    args = (p, p, p, 1, p, p, 1, 1500.0, 0.0, 2.5e-8, 2, n_out, 6.0, 0, 0.0)
    assert lib.pab_adjoint(*args, p, ctypes.c_float(1.0), 2, 1, 1, p, None, p, None) == 1
    assert lib.pab_forward(p, p, p, None, 1, p, p, 1, 1500.0, 0.0, 2.5e-8, 2, n_out, 6.0, 0, 0.0, 0, 1, 1, 0,
                           p, p, 0, p, p, None) == 1
    assert E.Acq(1500.0, 0.0, 2.5e-8, 1 << 21, 1, 6.0, 0, 0.0).n_out == 1 << 21
    with pytest.raises(ValueError, match="exceeds"):
        E.Acq(1500.0, 0.0, 2.5e-8, (1 << 21) + 1, 1, 6.0, 0, 0.0)
