"""ctypes wrapper around oracle/fpe_oracle.c (TEST INFRASTRUCTURE ONLY).

Build: ``gcc -O2 -fopenmp -shared -fPIC fpe_oracle.c -lquadmath`` into
``oracle/liboracle.so`` (no fast-math: the oracle relies on IEEE semantics).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "fpe_oracle.c")
SO = os.path.join(HERE, "liboracle.so")
NEG_INF_SCALE = -(2**31)

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-std=gnu11", "-fopenmp", "-shared", "-fPIC", "-Wall",
               "-o", SO, SRC, "-lquadmath", "-lm"]
        subprocess.run(cmd, check=True)
    return SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(SO)
            i32, i64, dbl = C.c_int32, C.c_int64, C.c_double
            P = C.c_void_p
            L.or_scale_real.argtypes = [dbl]; L.or_scale_real.restype = i32
            L.or_scale_complex.argtypes = [dbl, dbl]; L.or_scale_complex.restype = i32
            L.or_scales.argtypes = [P, i64, C.c_int, P]; L.or_scales.restype = None
            L.or_scale_int.argtypes = [i64]; L.or_scale_int.restype = i32
            L.or_drop.argtypes = [i32, i64]; L.or_drop.restype = i32
            L.or_hull.argtypes = [P, i64, P, P]; L.or_hull.restype = i64
            L.or_good.argtypes = [P, i64, P, P, i64, i32, P]; L.or_good.restype = None
            L.or_lambda.argtypes = [dbl, dbl, C.c_int, P]; L.or_lambda.restype = dbl
            L.or_classify.argtypes = [P, i64, C.c_int, P, P, i64, i32, P, P, P, P, P]
            L.or_classify.restype = None
            L.or_classify_lambda.argtypes = [P, i64, P, P, i64, i32, P, P, P]
            L.or_classify_lambda.restype = None
            L.or_fpe_eval.argtypes = [P, P, C.c_int, P, i64, P, P, P, P]; L.or_fpe_eval.restype = None
            L.or_horner.argtypes = [P, i64, i64, C.c_int, P, i64, P, P]; L.or_horner.restype = None
            L.or_horner_dd.argtypes = [P, i64, i64, C.c_int, P, i64, P, P]; L.or_horner_dd.restype = None
            L.or_direct_sum.argtypes = [P, P, i64, C.c_int, P, i64, P, P]; L.or_direct_sum.restype = None
            L.or_abs_sum.argtypes = [P, i64, i64, C.c_int, P, i64, P, P]; L.or_abs_sum.restype = None
            L.or_log2abs.argtypes = [P, i64, C.c_int, P]; L.or_log2abs.restype = None
            L.or_log2_maxterm.argtypes = [P, i64, P, i64, C.c_int, P]; L.or_log2_maxterm.restype = None
            _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _flat(a: np.ndarray):
    """complex -> interleaved float64 (re, im); real -> float64.  Exact."""
    a = np.asarray(a)
    if np.iscomplexobj(a):
        return np.ascontiguousarray(a.astype(np.complex128)).view(np.float64), 1
    return np.ascontiguousarray(a.astype(np.float64)), 0


def scale(z) -> int:
    """s(z) = 1 + floor(log2|z|); NEG_INF_SCALE for 0."""
    z = complex(z) if isinstance(z, complex) or np.iscomplexobj(z) else float(z)
    if isinstance(z, complex):
        return int(lib().or_scale_complex(z.real, z.imag))
    return int(lib().or_scale_real(z))


def scales(a: np.ndarray) -> np.ndarray:
    f, cplx = _flat(a)
    out = np.empty(len(a), dtype=np.int32)
    lib().or_scales(_ptr(f), len(a), cplx, _ptr(out))
    return out


def hull(s: np.ndarray):
    """Canonical concave cover (hk, hh) of (k, s_k) by the paper's insertion."""
    s = np.ascontiguousarray(s, dtype=np.int32)
    hk = np.empty(max(len(s), 1), dtype=np.int32)
    hh = np.empty(max(len(s), 1), dtype=np.int32)
    m = lib().or_hull(_ptr(s), len(s), _ptr(hk), _ptr(hh))
    if m < 0:
        raise RuntimeError("oracle hull construction produced a non-concave vertex list")
    return hk[:m].copy(), hh[:m].copy()


def drop_for(p: int, d_eff: int) -> int:
    return int(lib().or_drop(p, d_eff))


def lam(z, is_complex: bool | None = None):
    """(lambda, hard): correctly rounded fp64 log2|z| and the Ziv hard-case flag."""
    if is_complex is None:
        is_complex = isinstance(z, complex) or np.iscomplexobj(z)
    z = complex(z)
    hard = C.c_int32(0)
    v = lib().or_lambda(z.real, z.imag, 1 if is_complex else 0, C.byref(hard))
    return float(v), int(hard.value)


class OraclePoly:
    """Preconditioned polynomial (Algorithm FPE_p lines 2-4).

    coeffs: complex128 / float64 (fp32 inputs are widened exactly).
    p: precision in bits (default 53 for fp64 inputs, 24 for fp32).
    drop: overrides D = p + s(d_eff) + 3 (tests only).
    """

    def __init__(self, coeffs, p: int | None = None, drop: int | None = None):
        coeffs = np.asarray(coeffs)
        if p is None:
            p = 24 if coeffs.dtype in (np.float32, np.complex64) else 53
        self.is_complex = bool(np.iscomplexobj(coeffs))
        self.a, _ = _flat(coeffs)
        self.coeffs = coeffs.astype(np.complex128 if self.is_complex else np.float64)
        self.n = len(coeffs)
        self.p = int(p)
        self.s = scales(coeffs)
        nz = np.flatnonzero(self.s != NEG_INF_SCALE)
        if len(nz) == 0:
            raise ValueError("zero polynomial")
        self.k_min, self.k_max = int(nz[0]), int(nz[-1])
        self.d_eff = self.k_max - self.k_min
        self.hk, self.hh = hull(self.s)
        self.drop = int(drop) if drop else drop_for(self.p, self.d_eff)
        self.good = np.zeros(self.n, dtype=np.uint8)
        lib().or_good(_ptr(self.s), self.n, _ptr(self.hk), _ptr(self.hh), len(self.hk),
                      self.drop, _ptr(self.good))
        self.good_prefix = np.concatenate([[0], np.cumsum(self.good, dtype=np.int64)])

    # -- evaluation phase -------------------------------------------------
    def _pts(self, pts):
        pts = np.asarray(pts)
        cplx = self.is_complex or np.iscomplexobj(pts)
        if cplx:
            f = np.ascontiguousarray(pts.astype(np.complex128)).view(np.float64)
        else:
            f = np.ascontiguousarray(pts.astype(np.float64))
        return f, int(cplx), len(pts)

    def _coef_for(self, cplx: int):
        if cplx and not self.is_complex:
            return np.ascontiguousarray(self.coeffs.astype(np.complex128)).view(np.float64)
        return self.a

    def classify(self, pts):
        """lambda, i*, l, r, K and the hard-case flag per point (lines 5-8)."""
        f, cplx, n = self._pts(pts)
        lam_ = np.empty(n); ist = np.empty(n, np.int32)
        l = np.empty(n, np.int64); r = np.empty(n, np.int64); hard = np.empty(n, np.int32)
        lib().or_classify(_ptr(f), n, cplx, _ptr(self.hk), _ptr(self.hh), len(self.hk),
                          self.drop, _ptr(lam_), _ptr(ist), _ptr(l), _ptr(r), _ptr(hard))
        K = np.where(l >= 0, self.good_prefix[np.maximum(r, 0) + 1] - self.good_prefix[np.maximum(l, 0)], 0)
        return dict(lam=lam_, istar=ist, l=l, r=r, K=K.astype(np.int64), hard=hard)

    def search(self, lams):
        """(i*, l, r) for given lambda values (lines 6-8 without line 5)."""
        lams = np.ascontiguousarray(lams, dtype=np.float64)
        n = len(lams)
        ist = np.empty(n, np.int32); l = np.empty(n, np.int64); r = np.empty(n, np.int64)
        lib().or_classify_lambda(_ptr(lams), n, _ptr(self.hk), _ptr(self.hh), len(self.hk),
                                 self.drop, _ptr(ist), _ptr(l), _ptr(r))
        return ist, l, r

    def fpe_eval(self, pts, cls=None):
        """Q_lambda(z) (line 9) as (mantissa hi complex, mantissa lo complex, exponent)."""
        f, cplx, n = self._pts(pts)
        if cls is None:
            cls = self.classify(pts)
        out = np.empty(4 * n); e = np.empty(n, np.int64)
        l = np.ascontiguousarray(cls["l"], dtype=np.int64)
        r = np.ascontiguousarray(cls["r"], dtype=np.int64)
        lib().or_fpe_eval(_ptr(self._coef_for(cplx)), _ptr(self.good), cplx, _ptr(f), n,
                          _ptr(l), _ptr(r), _ptr(out), _ptr(e))
        return _unpack(out, e)

    def horner(self, pts):
        """Reference P(z) by full binary128 Horner (the plain definition)."""
        f, cplx, n = self._pts(pts)
        out = np.empty(4 * n); e = np.empty(n, np.int64)
        lib().or_horner(_ptr(self._coef_for(cplx)), self.k_min, self.k_max, cplx, _ptr(f), n,
                        _ptr(out), _ptr(e))
        return _unpack(out, e)

    def horner_dd(self, pts):
        """Reference P(z) by full double-double Horner with an exponent counter (the plain definition;
        faster than horner() for the full-size value checks)."""
        f, cplx, n = self._pts(pts)
        out = np.empty(4 * n); e = np.empty(n, np.int64)
        lib().or_horner_dd(_ptr(self._coef_for(cplx)), self.k_min, self.k_max, cplx, _ptr(f), n,
                           _ptr(out), _ptr(e))
        return _unpack(out, e)

    def direct_sum(self, pts):
        """Reference P(z) = sum of a_k z^k over the nonzero terms (sparse inputs)."""
        f, cplx, n = self._pts(pts)
        idx = np.flatnonzero(self.s != NEG_INF_SCALE).astype(np.int64)
        vals = self.coeffs[idx]
        if cplx:
            vf = np.ascontiguousarray(vals.astype(np.complex128)).view(np.float64)
        else:
            vf = np.ascontiguousarray(vals.astype(np.float64))
        out = np.empty(4 * n); e = np.empty(n, np.int64)
        lib().or_direct_sum(_ptr(idx), _ptr(vf), len(idx), cplx, _ptr(f), n, _ptr(out), _ptr(e))
        return _unpack(out, e)

    def abs_sum(self, pts):
        """S(z) = sum |a_k||z|^k as (mantissa, exponent)."""
        f, cplx, n = self._pts(pts)
        out = np.empty(n); e = np.empty(n, np.int64)
        lib().or_abs_sum(_ptr(self._coef_for(cplx)), self.k_min, self.k_max, cplx, _ptr(f), n,
                         _ptr(out), _ptr(e))
        return out, e

    def log2_maxterm(self, pts):
        """log2 of M(z) = max_k |a_k z^k| (eq:def_prec_loss)."""
        f, cplx, n = self._pts(pts)
        l2a = np.empty(self.n)
        lib().or_log2abs(_ptr(self.a), self.n, int(self.is_complex), _ptr(l2a))
        out = np.empty(n)
        lib().or_log2_maxterm(_ptr(l2a), self.n, _ptr(f), n, cplx, _ptr(out))
        return out


class XVal:
    """Extended-range values (hi + lo) 2^e, with hi, lo complex128."""

    def __init__(self, hi, lo, e):
        self.hi, self.lo, self.e = hi, lo, e

    def __len__(self):
        return len(self.e)

    def scaled(self, e_ref):
        """Value times 2^-e_ref as complex128 (hi + lo folded)."""
        sh = (self.e - e_ref).astype(np.int64)
        sh = np.clip(sh, -2000, 2000)
        return np.ldexp(self.hi.real, sh) + np.ldexp(self.lo.real, sh) + \
            1j * (np.ldexp(self.hi.imag, sh) + np.ldexp(self.lo.imag, sh))


def _unpack(out, e):
    o = out.reshape(-1, 4)
    hi = o[:, 0] + 1j * o[:, 2]
    lo = o[:, 1] + 1j * o[:, 3]
    return XVal(hi, lo, e)
