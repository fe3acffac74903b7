"""C-ABI boundary checks that need no GPU: the library builds/loads, exports
every symbol include/rnsntt.h declares, and rejects bad plans synchronously
(before touching CUDA) with the documented status codes."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "rnsntt.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2410_05934_b200 import build

    build.build()
    import paper_2410_05934_b200 as R

    return R


def declared_symbols():
    src = open(HDR).read()
    return sorted(set(re.findall(r"\b(rnt_[a-z_]+)\s*\(", src)))


def test_header_declares_boundary():
    syms = declared_symbols()
    for s in ["rnt_plan_create", "rnt_plan_destroy", "rnt_plan_query", "rnt_ntt_forward",
              "rnt_ntt_inverse", "rnt_pointwise_mul", "rnt_polymul", "rnt_status_string",
              "rnt_last_cuda_error", "rnt_execute_host", "rnt_launch_count"]:
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    so = ctypes.CDLL(lib.lib_path())
    for s in declared_symbols():
        assert hasattr(so, s), s
    from paper_2410_05934_b200 import _lib

    assert set(_lib.SIGNATURES) == set(declared_symbols())


def test_status_strings(lib):
    for code in range(8):
        assert lib.status_string(code).startswith("RNT_")


def _create(lib, logn, moduli, psi=None):
    h = ctypes.c_void_p()
    m = (ctypes.c_uint64 * len(moduli))(*moduli)
    p = (ctypes.c_uint64 * len(psi))(*psi) if psi is not None else None
    from paper_2410_05934_b200 import _lib

    rc = _lib.L.rnt_plan_create(ctypes.byref(h), logn, len(moduli), m, p, 0)
    if rc == 0:
        _lib.L.rnt_plan_destroy(h)
    return rc


Q10 = 1152921504606830593  # 2^60 - 2^14 + 1


def test_plan_rejects_bad_arguments(lib):
    from paper_2410_05934_b200 import _lib

    assert _lib.L.rnt_plan_create(None, 10, 1, None, None, 0) == lib.RNT_E_INVALID_ARG
    assert _create(lib, 3, [97]) == lib.RNT_E_UNSUPPORTED_N
    assert _create(lib, 17, [Q10]) == lib.RNT_E_UNSUPPORTED_N
    assert _create(lib, 10, [Q10 + 2]) == lib.RNT_E_MODULUS          # not prime
    assert _create(lib, 10, [97]) == lib.RNT_E_MODULUS               # 97 != 1 mod 2048
    assert _create(lib, 10, [Q10, Q10]) == lib.RNT_E_MODULUS         # duplicate
    big = (1 << 62) + 1
    assert _create(lib, 4, [big]) == lib.RNT_E_MODULUS               # >= 2^62
    assert _create(lib, 10, [Q10], psi=[2]) == lib.RNT_E_ROOT         # not a primitive root
    assert _create(lib, 10, [Q10], psi=[0]) == lib.RNT_E_ROOT


def test_null_plan_calls(lib):
    from paper_2410_05934_b200 import _lib

    assert _lib.L.rnt_ntt_forward(None, None, None, 1, None) == lib.RNT_E_INVALID_ARG
    assert _lib.L.rnt_polymul(None, None, None, None, 1, 0, 0, None) == lib.RNT_E_INVALID_ARG
    assert _lib.L.rnt_plan_destroy(None) == lib.RNT_OK


def test_product_path_never_touches_oracle():
    """The product package must not import, link or call oracle/ (test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2410_05934_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "ntt_oracle" not in src and "liboracle" not in src, f
    hdr = open(HDR).read()
    assert "oracle" not in hdr
