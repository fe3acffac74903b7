"""ctypes loader for librnsntt.so (declarations mirror include/rnsntt.h)."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_PATH = os.path.join(_HERE, "librnsntt.so")

RNT_OK = 0
RNT_E_INVALID_ARG = 1
RNT_E_UNSUPPORTED_N = 2
RNT_E_MODULUS = 3
RNT_E_ROOT = 4
RNT_E_PLAN_MISMATCH = 5
RNT_E_CUDA = 6
RNT_E_OOM = 7

# Exported symbols and their C signatures (include/rnsntt.h).
_vp, _u32, _i32, _u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int, ctypes.c_uint64
_u64p = ctypes.POINTER(ctypes.c_uint64)
SIGNATURES = {
    "rnt_plan_create": (_i32, [ctypes.POINTER(_vp), _u32, _u32, _u64p, _u64p, _i32]),
    "rnt_plan_destroy": (_i32, [_vp]),
    "rnt_plan_query": (_i32, [_vp, ctypes.POINTER(_u32), ctypes.POINTER(_u32), _u64p, ctypes.POINTER(_i32)]),
    "rnt_ntt_forward": (_i32, [_vp, _vp, _vp, _u32, _vp]),
    "rnt_ntt_inverse": (_i32, [_vp, _vp, _vp, _u32, _vp]),
    "rnt_pointwise_mul": (_i32, [_vp, _vp, _vp, _vp, _u32, _i32, _vp]),
    "rnt_polymul": (_i32, [_vp, _vp, _vp, _vp, _u32, _i32, _i32, _vp]),
    "rnt_automorph": (_i32, [_vp, _vp, _vp, _u32, _u32, _i32, _vp]),
    "rnt_external_product": (_i32, [_vp, _vp, _vp, _vp, _u32, _u32, _u32, _vp]),
    "rnt_hrf_matvec": (_i32, [_vp, _vp, _vp, _vp, _u32, _vp, _vp]),
    "rnt_bconv_create": (_i32, [ctypes.POINTER(_vp), _vp, _vp]),
    "rnt_bconv_destroy": (_i32, [_vp]),
    "rnt_bconv_apply": (_i32, [_vp, _vp, _vp, _u32, _vp]),
    "rnt_keyswitch_create": (_i32, [ctypes.POINTER(_vp), _vp, _vp, _u32]),
    "rnt_keyswitch_destroy": (_i32, [_vp]),
    "rnt_keyswitch_query": (_i32, [_vp, ctypes.POINTER(_u32), _u64p]),
    "rnt_keyswitch_apply": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "rnt_execute_host": (_i32, [_vp, _i32, _vp, _vp, _vp, _vp, _u32, _i32, _vp]),
    "rnt_status_string": (ctypes.c_char_p, [_i32]),
    "rnt_last_cuda_error": (_i32, []),
    "rnt_launch_count": (_u64, []),
}


class RntError(RuntimeError):
    def __init__(self, code: int, msg: str | None = None):
        self.code = code
        super().__init__(msg or status_string(code))


def _load():
    if not os.path.exists(_PATH):
        raise ImportError(
            f"{_PATH} is missing: build it with `python -m paper_2410_05934_b200.build` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    lib = ctypes.CDLL(_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_L = None


def __getattr__(name):
    # The library is loaded on first use (PEP 562), so the package (and its
    # build module) imports on a box where librnsntt.so is not built yet; any
    # call into the library then raises ImportError -- there is no fallback.
    global _L
    if name == "L":
        if _L is None:
            _L = _load()
        return _L
    raise AttributeError(name)


def lib_path() -> str:
    return _PATH


def status_string(code: int) -> str:
    s = __getattr__("L").rnt_status_string(int(code))
    return s.decode() if s else f"rnt_status {code}"


def check(code: int) -> None:
    if code != RNT_OK:
        extra = ""
        if code in (RNT_E_CUDA, RNT_E_OOM):
            extra = f" (cudaError {__getattr__('L').rnt_last_cuda_error()})"
        raise RntError(code, status_string(code) + extra)


def launch_count() -> int:
    return int(__getattr__("L").rnt_launch_count())
