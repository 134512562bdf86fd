"""Helpers comparing the CUDA path (through the C ABI) with the oracle."""
from __future__ import annotations

import numpy as np

import oracle


def gpu_eval(poly, pts_np, diag=True, exps=True, horner=False):
    import torch
    import paper_2211_06320_b200 as fpe
    t = torch.from_numpy(np.ascontiguousarray(pts_np)).cuda()
    if horner:
        v, e = poly.horner(t, exps=exps)
        dg = None
    elif diag:
        v, e, dg = poly.evaluate(t, exps=exps, diag=True)
    else:
        v, e = poly.evaluate(t, exps=exps)
        dg = None
    torch.cuda.synchronize()
    if not horner:   # the library's self-checks of its work bucketing and plan (fpe_workspace_stats [5], [6])
        st = poly.workspace_stats()
        assert st.get("slice_mismatch", 0) == 0 and st.get("window_escapes", 0) == 0, st
    out = {"v": v.cpu().numpy(), "e": e.cpu().numpy() if e is not None else None}
    if dg is not None:
        out["diag"] = {k: t_.cpu().numpy() for k, t_ in fpe.diag_fields(dg).items()}
    return out


def abs_sum_log2(coeffs: np.ndarray, pts: np.ndarray) -> np.ndarray:
    """log2 S(z), S = sum_k |a_k||z|^k, in the log domain with numpy (a tolerance scale)."""
    a = np.abs(coeffs.astype(np.complex128))
    nz = np.flatnonzero(a)
    la = np.log2(a[nz])
    out = np.empty(len(pts))
    for i, z in enumerate(np.asarray(pts).astype(np.complex128)):
        if z == 0:
            out[i] = la[0] if nz[0] == 0 else -np.inf
            continue
        t = la + nz * np.log2(abs(z))
        m = t.max()
        out[i] = m + np.log2(np.sum(np.exp2(t - m)))
    return out


def check_indexing(P: oracle.OraclePoly, pts, diag):
    """Bit-exact lambda, region, l, r, K against the oracle.  Returns the oracle record."""
    c = P.classify(pts)
    ok = c["l"] >= 0
    assert np.array_equal(diag["lambda"][ok], c["lam"][ok]), _first_diff(diag["lambda"], c["lam"], ok)
    assert np.array_equal(diag["region"], c["istar"]), _first_diff(diag["region"], c["istar"])
    assert np.array_equal(diag["l"][ok], c["l"][ok]), _first_diff(diag["l"], c["l"], ok)
    assert np.array_equal(diag["r"][ok], c["r"][ok]), _first_diff(diag["r"], c["r"], ok)
    assert np.array_equal(diag["kept"][ok], c["K"][ok])
    assert np.all(diag["hard"] == 0) and np.all(c["hard"] == 0)
    return c


def _first_diff(a, b, mask=None):
    a = np.asarray(a); b = np.asarray(b)
    m = np.ones(len(a), bool) if mask is None else mask
    bad = np.flatnonzero(m & (a != b))
    if len(bad) == 0:
        return "ok"
    i = bad[0]
    return f"{len(bad)} mismatches; first at {i}: gpu={a[i]!r} oracle={b[i]!r}"


def rel_err_vs(ref: oracle.oracle.XVal, gpu_v, gpu_e, log2S):
    """|P_gpu - P_ref| / S per point (P_gpu = v 2^e; exponents aligned to S)."""
    eS = np.floor(log2S).astype(np.int64)
    Sm = np.exp2(log2S - eS)
    sh = np.clip(gpu_e - eS, -2000, 2000)
    g = np.ldexp(gpu_v.real.astype(np.float64), sh) + 1j * np.ldexp(np.imag(gpu_v).astype(np.float64), sh)
    r = ref.scaled(eS)
    return np.abs(g - r) / Sm
