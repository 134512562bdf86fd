"""B200-native Fast Polynomial Evaluator (arXiv 2211.06320) -- Python binding.

A thin layer over libfpe.so (include/fpe.h): it marshals torch tensors to
pointers and back.  Every step of the evaluation runs in the library's sm_100a
kernels; torch provides device memory, streams and process groups only.

    import paper_2211_06320_b200 as fpe
    poly = fpe.precondition(coeffs)              # Algorithm FPE_p lines 2-4
    vals, exps = poly.evaluate(points_cuda)      # lines 5-9: value = vals * 2**exps
    vals, exps = poly.horner(points_cuda)        # full Horner (context baseline)
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from ._lib import (DIAG_BYTES, FPE_C32, FPE_C64, FPE_R32, FPE_R64, FpeError, FpeInfo, check, lib)

__all__ = ["precondition", "precondition_derivative", "newton_step", "precondition_buffer", "Poly", "FpeError",
           "diag_fields", "header_fields"]

_TORCH_DT = None


def _torch():
    import torch
    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    m = {torch.float64: FPE_R64, torch.complex128: FPE_C64, torch.float32: FPE_R32, torch.complex64: FPE_C32}
    if isinstance(t, torch.Tensor):
        if t.dtype not in m:
            raise TypeError(f"unsupported dtype {t.dtype}")
        return m[t.dtype]
    dt = np.asarray(t).dtype
    nm = {np.dtype(np.float64): FPE_R64, np.dtype(np.complex128): FPE_C64,
          np.dtype(np.float32): FPE_R32, np.dtype(np.complex64): FPE_C32}
    if dt not in nm:
        raise TypeError(f"unsupported dtype {dt}")
    return nm[dt]


def _stream_ptr(stream, device):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return C.c_void_p(stream.cuda_stream)


def _out_dtype(poly_dt: int, pt_dt: int):
    torch = _torch()
    cplx = poly_dt in (FPE_C64, FPE_C32) or pt_dt in (FPE_C64, FPE_C32)
    f32 = pt_dt in (FPE_R32, FPE_C32)
    if f32:
        return torch.complex64 if cplx else torch.float32
    return torch.complex128 if cplx else torch.float64


class Poly:
    """Handle of an immutable preconditioned polynomial on one CUDA device."""

    def __init__(self, handle: C.c_void_p, device: int):
        self._h = handle
        self.device = device
        info = FpeInfo()
        check(lib().fpe_poly_get_info(self._h, C.byref(info)), "fpe_poly_get_info")
        self.info = {f: getattr(info, f) for f, _ in FpeInfo._fields_ if f != "reserved"}
        self._last = threading.local()   # the workspace and stream of this thread's last call (last_stats)

    # -- metadata -----------------------------------------------------------
    @property
    def nbytes(self) -> int:
        return int(self.info["bytes"])

    def hull(self):
        n = int(self.info["n_hull"])
        hk = np.empty(n, np.int32); hh = np.empty(n, np.int32); cnt = C.c_int64(0)
        check(lib().fpe_poly_get_hull(self._h, hk.ctypes.data, hh.ctypes.data, n, C.byref(cnt)), "fpe_poly_get_hull")
        return hk, hh

    def analyse(self, lam_lo: float, lam_hi: float) -> np.ndarray:
        """The -analyse task (fpe_analyse): the lambda = log2|z| intervals on which (i*, l, r) is constant,
        as a structured array (lam_lo, lam_hi, region, l, r, kept)."""
        dt = np.dtype([("lam_lo", np.float64), ("lam_hi", np.float64), ("region", np.int32), ("l", np.int32),
                       ("r", np.int32), ("kept", np.int32)])
        cnt = C.c_int64(0)
        check(lib().fpe_analyse(self._h, float(lam_lo), float(lam_hi), None, 0, C.byref(cnt)), "fpe_analyse")
        out = np.zeros(cnt.value, dt)
        check(lib().fpe_analyse(self._h, float(lam_lo), float(lam_hi), out.ctypes.data, len(out), C.byref(cnt)),
              "fpe_analyse")
        return out

    def device_buffer(self):
        p = C.c_void_p(); b = C.c_size_t()
        check(lib().fpe_poly_device_buffer(self._h, C.byref(p), C.byref(b)), "fpe_poly_device_buffer")
        return p.value, b.value

    def export(self, dst_ptr: int, cap: int, stream=None):
        check(lib().fpe_poly_export(self._h, C.c_void_p(dst_ptr), cap, _stream_ptr(stream, self.device)),
              "fpe_poly_export")

    @classmethod
    def from_buffer(cls, ptr: int, nbytes: int, device: int = 0, stream=None):
        h = C.c_void_p()
        check(lib().fpe_poly_from_device_buffer(C.c_void_p(ptr), nbytes, device, _stream_ptr(stream, device),
                                                C.byref(h)), "fpe_poly_from_device_buffer")
        return cls(h, device)

    # -- evaluation ---------------------------------------------------------
    def workspace_bytes(self, n: int) -> int:
        sz = C.c_size_t()
        check(lib().fpe_eval_workspace_size(self._h, n, C.byref(sz)), "fpe_eval_workspace_size")
        return max(int(sz.value), 256)

    def workspace(self, n: int, stream=None):
        """A fresh workspace for n points, allocated on `stream` (default: the current stream) by torch's
        stream-ordered caching allocator: concurrent calls on different streams never share one."""
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(st):
            return torch.empty(self.workspace_bytes(n), dtype=torch.uint8, device=f"cuda:{self.device}")

    def evaluate(self, points, exps: bool = True, diag: bool = False, out=None, stream=None, workspace=None):
        """Q_lambda(z) for every point (device tensor).  Returns (values, exps[, diag]).
        workspace: optional uint8 CUDA tensor of at least workspace_bytes(n) (else one is allocated on the
        call's stream)."""
        return self._run(lib().fpe_evaluate, points, exps, diag, out, stream, workspace, "fpe_evaluate")

    def horner(self, points, exps: bool = True, out=None, stream=None, workspace=None):
        """Full Horner over all stored coefficients (context baseline)."""
        return self._run(lib().fpe_horner, points, exps, False, out, stream, workspace, "fpe_horner")

    def _run(self, fn, points, want_exps, want_diag, out, stream, ws, where):
        torch = _torch()
        if not points.is_cuda:
            raise ValueError("points must be a CUDA tensor (use evaluate_host for host arrays)")
        points = points.contiguous()
        n = points.numel()
        pdt = _dtype_code(points)
        dev = points.device
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        vals = out if out is not None else torch.empty(n, dtype=_out_dtype(self.info["dtype"], pdt), device=dev)
        e = torch.empty(n, dtype=torch.int64, device=dev) if want_exps else None
        dg = torch.empty((n, DIAG_BYTES), dtype=torch.uint8, device=dev) if want_diag else None
        if ws is None:
            self._last.ws = None   # let the previous call's workspace go back to the allocator first
            ws = self.workspace(n, st)
        elif ws.numel() < self.workspace_bytes(n):
            raise ValueError("workspace too small")
        args = [self._h, C.c_void_p(points.data_ptr()), pdt, n, C.c_void_p(vals.data_ptr()),
                C.c_void_p(e.data_ptr() if e is not None else 0)]
        if fn is lib().fpe_evaluate:
            args.append(C.c_void_p(dg.data_ptr() if dg is not None else 0))
        args += [C.c_void_p(ws.data_ptr()), ws.numel(), C.c_void_p(st.cuda_stream)]
        check(fn(*args), where)
        self._last.ws, self._last.stream = ws, st
        if want_diag:
            return vals, e, dg
        return vals, e

    def workspace_stats(self, ws=None, stream=None) -> dict:
        """Counters of the last evaluate() that used workspace `ws` (default: this thread's last call)."""
        if ws is None:
            ws, stream = getattr(self._last, "ws", None), getattr(self._last, "stream", None)
            if ws is None:
                raise ValueError("no evaluate() call on this thread yet")
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        v = np.zeros(8, np.int64)
        cnt = C.c_int(0)
        check(lib().fpe_workspace_stats(C.c_void_p(ws.data_ptr()), C.c_void_p(st.cuda_stream), v.ctypes.data, 8,
                                        C.byref(cnt)), "fpe_workspace_stats")
        names = ["hard_lambdas", "mma_items", "mma_inwarp_items", "piece_items", "serial_long_groups",
                 "slice_mismatch", "window_escapes"]
        return {k: int(v[i]) for i, k in enumerate(names[:cnt.value])}

    def evaluate_host(self, points: np.ndarray, exps: bool = True):
        """End-to-end evaluation from host memory (pinned for full bandwidth)."""
        pts = np.ascontiguousarray(points)
        pdt = _dtype_code(pts)
        n = len(pts)
        torch = _torch()
        odt = _out_dtype(self.info["dtype"], pdt)
        npdt = {torch.complex128: np.complex128, torch.float64: np.float64,
                torch.complex64: np.complex64, torch.float32: np.float32}[odt]
        vals = np.empty(n, npdt)
        e = np.empty(n, np.int64) if exps else None
        check(lib().fpe_evaluate_host(self._h, pts.ctypes.data, pdt, n, vals.ctypes.data,
                                      e.ctypes.data if e is not None else None, None), "fpe_evaluate_host")
        return vals, e

    def evaluate_host_ptr(self, pts_ptr: int, pdt: int, n: int, vals_ptr: int, exps_ptr: int):
        """Raw-pointer variant of evaluate_host (pinned torch tensors in bench.py)."""
        check(lib().fpe_evaluate_host(self._h, C.c_void_p(pts_ptr), pdt, n, C.c_void_p(vals_ptr),
                                      C.c_void_p(exps_ptr), None), "fpe_evaluate_host")

    def set_profiling(self, on: bool = True):
        check(lib().fpe_set_profiling(self._h, 1 if on else 0), "fpe_set_profiling")

    def last_stage_ms(self):
        """[(stage name, ms)] of the last evaluate/horner call (profiling must be on)."""
        ms = (C.c_float * 16)()
        n = C.c_int(0)
        check(lib().fpe_last_stage_ms(self._h, ms, 16, C.byref(n)), "fpe_last_stage_ms")
        return [(lib().fpe_stage_name(self._h, i).decode(), float(ms[i])) for i in range(n.value)]

    def last_stats(self):
        """Counters of this thread's last library call (fpe_last_stats): hard lambdas, kernel launches,
        tensor-core items and those run in-warp."""
        s = np.zeros(4, np.int64)
        check(lib().fpe_last_stats(self._h, s.ctypes.data), "fpe_last_stats")
        return {"hard_lambdas": int(s[0]), "launches": int(s[1]), "mma_items": int(s[2]),
                "mma_inwarp_items": int(s[3])}

    def close(self):
        if self._h:
            lib().fpe_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def precondition(coeffs, p: int | None = None, drop: int | None = None, device: int | None = None,
                 stream=None) -> Poly:
    """Algorithm FPE_p lines 2-4 on a numpy array or torch tensor (host or device)."""
    torch = _torch()
    dt = _dtype_code(coeffs)
    if device is None:
        device = coeffs.device.index if isinstance(coeffs, torch.Tensor) and coeffs.is_cuda else torch.cuda.current_device()
    keep = coeffs
    if isinstance(coeffs, torch.Tensor):
        keep = coeffs.contiguous()
        ptr = keep.data_ptr()
    else:
        keep = np.ascontiguousarray(coeffs)
        ptr = keep.ctypes.data
    n = keep.numel() if isinstance(keep, torch.Tensor) else len(keep)
    h = C.c_void_p()
    check(lib().fpe_precondition(C.c_void_p(ptr), n, dt, p or 0, drop or 0, device,
                                 _stream_ptr(stream, device), C.byref(h)), "fpe_precondition")
    return Poly(h, device)


def precondition_gpu(coeffs, p: int | None = None, drop: int | None = None, stream=None) -> Poly:
    """Algorithm FPE_p lines 2-4 computed on the device (fpe_precondition_gpu) from a CUDA tensor;
    the handle's buffer is byte-identical to precondition()'s."""
    torch = _torch()
    if not (isinstance(coeffs, torch.Tensor) and coeffs.is_cuda):
        raise ValueError("precondition_gpu needs a CUDA tensor")
    dt = _dtype_code(coeffs)
    keep = coeffs.contiguous()
    device = keep.device.index
    h = C.c_void_p()
    check(lib().fpe_precondition_gpu(C.c_void_p(keep.data_ptr()), keep.numel(), dt, p or 0, drop or 0, device,
                                     _stream_ptr(stream, device), C.byref(h)), "fpe_precondition_gpu")
    return Poly(h, device)


class Cover:
    """Partial preprocessing: scales and concave cover of P on the device, once;
    finish(p) completes G_p and the flat buffer for a precision p in O(d)."""

    def __init__(self, coeffs, stream=None):
        torch = _torch()
        if not (isinstance(coeffs, torch.Tensor) and coeffs.is_cuda):
            raise ValueError("Cover needs a CUDA tensor")
        keep = coeffs.contiguous()
        self.device = keep.device.index
        self._h = C.c_void_p()
        check(lib().fpe_cover_build(C.c_void_p(keep.data_ptr()), keep.numel(), _dtype_code(keep), self.device,
                                    _stream_ptr(stream, self.device), C.byref(self._h)), "fpe_cover_build")

    def finish(self, p: int | None = None, drop: int | None = None, stream=None) -> "Poly":
        h = C.c_void_p()
        check(lib().fpe_cover_finish(self._h, p or 0, drop or 0, _stream_ptr(stream, self.device), C.byref(h)),
              "fpe_cover_finish")
        return Poly(h, self.device)

    def close(self):
        if self._h:
            lib().fpe_cover_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def precondition_derivative(coeffs, p: int | None = None, drop: int | None = None, device: int | None = None,
                            stream=None) -> Poly:
    """P' preconditioned (fpe_precondition_derivative): coefficients (j+1) a_{j+1} of P's coefficients."""
    torch = _torch()
    dt = _dtype_code(coeffs)
    if device is None:
        device = coeffs.device.index if isinstance(coeffs, torch.Tensor) and coeffs.is_cuda else torch.cuda.current_device()
    keep = coeffs.contiguous() if isinstance(coeffs, torch.Tensor) else np.ascontiguousarray(coeffs)
    ptr = keep.data_ptr() if isinstance(keep, torch.Tensor) else keep.ctypes.data
    n = keep.numel() if isinstance(keep, torch.Tensor) else len(keep)
    h = C.c_void_p()
    check(lib().fpe_precondition_derivative(C.c_void_p(ptr), n, dt, p or 0, drop or 0, device,
                                            _stream_ptr(stream, device), C.byref(h)), "fpe_precondition_derivative")
    return Poly(h, device)


def newton_step(P: Poly, dP: Poly, points, incr: bool = False, stream=None):
    """One Newton step N_P(z) = z - P(z)/P'(z) on a CUDA tensor of points (fpe_newton_step).
    Returns the new points (and the increments P/P' when incr=True)."""
    torch = _torch()
    points = points.contiguous()
    n = points.numel()
    pdt = _dtype_code(points)
    odt = _out_dtype(P.info["dtype"], pdt)
    out = torch.empty(n, dtype=odt, device=points.device)
    inc = torch.empty(n, dtype=odt, device=points.device) if incr else None
    sz = C.c_size_t()
    check(lib().fpe_newton_workspace_size(P._h, dP._h, n, C.byref(sz)), "fpe_newton_workspace_size")
    ws = torch.empty(max(sz.value, 256), dtype=torch.uint8, device=points.device)
    check(lib().fpe_newton_step(P._h, dP._h, C.c_void_p(points.data_ptr()), pdt, n, C.c_void_p(out.data_ptr()),
                                C.c_void_p(inc.data_ptr() if inc is not None else 0), C.c_void_p(ws.data_ptr()),
                                ws.numel(), _stream_ptr(stream, points.device)), "fpe_newton_step")
    return (out, inc) if incr else out


def precondition_buffer(coeffs: np.ndarray, p: int | None = None, drop: int | None = None) -> np.ndarray:
    """Host-only preconditioning: the flat buffer (uint8) a handle would hold.  No GPU needed."""
    a = np.ascontiguousarray(coeffs)
    dt = _dtype_code(a)
    sz = C.c_size_t(0)
    st = lib().fpe_precondition_host(a.ctypes.data, len(a), dt, p or 0, drop or 0, None, 0, C.byref(sz))
    if st != 1:   # INVALID_ARG carries the size query
        check(st, "fpe_precondition_host")
    buf = np.zeros(sz.value, np.uint8)
    check(lib().fpe_precondition_host(a.ctypes.data, len(a), dt, p or 0, drop or 0, buf.ctypes.data,
                                      sz.value, C.byref(sz)), "fpe_precondition_host")
    return buf


_HDR = np.dtype([("magic", "<u8"), ("version", "<u4"), ("dtype", "<i4"), ("n_coeffs", "<i8"), ("k_min", "<i8"),
                 ("k_max", "<i8"), ("n_hull", "<i8"), ("n_good", "<i8"), ("p", "<i4"), ("drop", "<i4"),
                 ("shift", "<i4"), ("sparse", "<i4"), ("all_good", "<i4"), ("wide", "<i4"), ("off_hull", "<u8"),
                 ("off_coef", "<u8"), ("off_prefix", "<u8"), ("off_sidx", "<u8"), ("bytes", "<u8")])


def header_fields(buf: np.ndarray) -> dict:
    """Decode the 256-byte header and the sections of a flat buffer (host uint8 array)."""
    h = np.frombuffer(buf[:_HDR.itemsize].tobytes(), dtype=_HDR)[0]
    d = {k: int(h[k]) for k in _HDR.names}
    nv = d["n_hull"]
    hull = np.frombuffer(buf[d["off_hull"]:d["off_hull"] + 8 * nv].tobytes(), dtype=np.int32).reshape(nv, 2)
    d["hk"], d["hh"] = hull[:, 0].copy(), hull[:, 1].copy()
    cdt = {FPE_R64: np.float64, FPE_C64: np.complex128, FPE_R32: np.float32, FPE_C32: np.complex64}[d["dtype"]]
    ncoef = d["n_good"] if d["sparse"] else d["k_max"] - d["k_min"] + 1
    sz = np.dtype(cdt).itemsize
    d["coef"] = np.frombuffer(buf[d["off_coef"]:d["off_coef"] + sz * ncoef].tobytes(), dtype=cdt)
    if d["off_sidx"]:
        d["sidx"] = np.frombuffer(buf[d["off_sidx"]:d["off_sidx"] + 4 * d["n_good"]].tobytes(), dtype=np.int32)
    if d["off_prefix"]:
        m = d["k_max"] - d["k_min"] + 2
        d["prefix"] = np.frombuffer(buf[d["off_prefix"]:d["off_prefix"] + 4 * m].tobytes(), dtype=np.int32)
    return d


def diag_fields(dg):
    """Split a (n, DIAG_BYTES) uint8 diag tensor into named tensors (lambda, region, l, r, kept, hard, cancel,
    trusted, err_exp)."""
    raw = dg.contiguous()
    lam = raw[:, 0:8].contiguous().view(_torch().float64).reshape(-1)
    ints = raw[:, 8:44].contiguous().view(_torch().int32).reshape(-1, 9)
    return {"lambda": lam, "region": ints[:, 0], "l": ints[:, 1], "r": ints[:, 2],
            "kept": ints[:, 3], "hard": ints[:, 4], "cancel": ints[:, 5], "trusted": ints[:, 6],
            "err_exp": ints[:, 7]}
