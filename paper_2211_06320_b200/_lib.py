"""ctypes loader for libfpe.so (the C ABI of include/fpe.h).

Argument marshalling only.  There is no fallback: if the in-tree library is
missing this raises, so a GPU run can never silently use anything else.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libfpe.so")

FPE_OK, FPE_ERR_INVALID_ARG, FPE_ERR_ZERO_POLY, FPE_ERR_NONFINITE_COEFF = 0, 1, 2, 3
FPE_ERR_UNSUPPORTED, FPE_ERR_OOM, FPE_ERR_CUDA = 4, 5, 6
FPE_R64, FPE_C64, FPE_R32, FPE_C32 = 0, 1, 2, 3


class FpeInfo(C.Structure):
    _fields_ = [("d", C.c_int64), ("k_min", C.c_int64), ("k_max", C.c_int64), ("n_hull", C.c_int64),
                ("n_good", C.c_int64), ("p", C.c_int32), ("drop", C.c_int32), ("shift", C.c_int32),
                ("sparse", C.c_int32), ("dtype", C.c_int32), ("reserved", C.c_int32), ("bytes", C.c_size_t)]


DIAG_BYTES = 48  # fpe_diag: double lambda; int32 region, l, r, kept, hard, cancel, trusted, err_exp, pad

_lock = threading.Lock()
_lib = None


class FpeError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: status {status} ({_STATUS.get(status, '?')}): {detail}")
        self.status = status


_STATUS = {0: "FPE_OK", 1: "FPE_ERR_INVALID_ARG", 2: "FPE_ERR_ZERO_POLY", 3: "FPE_ERR_NONFINITE_COEFF",
           4: "FPE_ERR_UNSUPPORTED", 5: "FPE_ERR_OOM", 6: "FPE_ERR_CUDA"}

# name -> (restype, argtypes)
_P, _I32, _I64, _SZ = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
SIGNATURES = {
    "fpe_precondition": (C.c_int, [_P, _I64, C.c_int, _I32, _I32, C.c_int, _P, C.POINTER(_P)]),
    "fpe_precondition_gpu": (C.c_int, [_P, _I64, C.c_int, _I32, _I32, C.c_int, _P, C.POINTER(_P)]),
    "fpe_cover_build": (C.c_int, [_P, _I64, C.c_int, C.c_int, _P, C.POINTER(_P)]),
    "fpe_cover_finish": (C.c_int, [_P, _I32, _I32, _P, C.POINTER(_P)]),
    "fpe_cover_destroy": (None, [_P]),
    "fpe_analyse": (C.c_int, [_P, C.c_double, C.c_double, _P, _I64, C.POINTER(_I64)]),
    "fpe_precondition_host": (C.c_int, [_P, _I64, C.c_int, _I32, _I32, _P, _SZ, C.POINTER(_SZ)]),
    "fpe_poly_get_info": (C.c_int, [_P, C.POINTER(FpeInfo)]),
    "fpe_poly_get_hull": (C.c_int, [_P, _P, _P, _I64, C.POINTER(_I64)]),
    "fpe_poly_device_buffer": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_SZ)]),
    "fpe_poly_export": (C.c_int, [_P, _P, _SZ, _P]),
    "fpe_poly_from_device_buffer": (C.c_int, [_P, _SZ, C.c_int, _P, C.POINTER(_P)]),
    "fpe_eval_workspace_size": (C.c_int, [_P, _I64, C.POINTER(_SZ)]),
    "fpe_evaluate": (C.c_int, [_P, _P, C.c_int, _I64, _P, _P, _P, _P, _SZ, _P]),
    "fpe_evaluate_host": (C.c_int, [_P, _P, C.c_int, _I64, _P, _P, _P]),
    "fpe_horner": (C.c_int, [_P, _P, C.c_int, _I64, _P, _P, _P, _SZ, _P]),
    "fpe_last_stats": (C.c_int, [_P, _P]),
    "fpe_workspace_stats": (C.c_int, [_P, _P, _P, C.c_int, C.POINTER(C.c_int)]),
    "fpe_precondition_derivative": (C.c_int, [_P, _I64, C.c_int, _I32, _I32, C.c_int, _P, C.POINTER(_P)]),
    "fpe_newton_workspace_size": (C.c_int, [_P, _P, _I64, C.POINTER(_SZ)]),
    "fpe_newton_step": (C.c_int, [_P, _P, _P, C.c_int, _I64, _P, _P, _P, _SZ, _P]),
    "fpe_set_profiling": (C.c_int, [_P, C.c_int]),
    "fpe_last_stage_ms": (C.c_int, [_P, _P, C.c_int, C.POINTER(C.c_int)]),
    "fpe_stage_name": (C.c_char_p, [_P, C.c_int]),
    "fpe_destroy": (None, [_P]),
    "fpe_status_string": (C.c_char_p, [C.c_int]),
    "fpe_last_error_detail": (C.c_char_p, []),
}


def lib():
    """The loaded libfpe.so.  Raises ImportError when it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(SO):
                raise ImportError(f"{SO} is missing -- build it with `python -m paper_2211_06320_b200.build` "
                                  "(there is no non-CUDA fallback)")
            L = C.CDLL(SO)
            for name, (res, args) in SIGNATURES.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def check(status: int, where: str):
    if status != FPE_OK:
        detail = lib().fpe_last_error_detail()
        raise FpeError(status, where, detail.decode() if detail else "")
