"""GPU parity: the CUDA path through the C ABI against the oracle.

Indexing (lambda, region = k_lambda vertex, l, r, K) must match bit-exactly;
values must satisfy |P_gpu - P_ref| <= 2^-45 S (fp64) or 2^-16 S (fp32),
S = sum_k |a_k||z|^k (BASELINE.json north_star), with P_ref the oracle's
Q_lambda in binary128.
"""
import math

import numpy as np
import pytest

import oracle
import workloads
from parity import abs_sum_log2, check_indexing, gpu_eval, rel_err_vs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL64 = 2.0 ** -45
TOL32 = 2.0 ** -16


@pytest.fixture(scope="module")
def fpe():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2211_06320_b200 import build
    build.build()
    import paper_2211_06320_b200 as m
    return m


def _values_ok(P, poly_coeffs, pts, out, idx, tol, cls=None):
    sub = pts[idx]
    c = P.classify(sub) if cls is None else {k: v[idx] for k, v in cls.items()}
    Q = P.fpe_eval(sub, c)
    l2S = abs_sum_log2(poly_coeffs, sub)
    err = rel_err_vs(Q, out["v"][idx], out["e"][idx], l2S)
    fin = np.isfinite(l2S) & (c["l"] >= 0)
    assert np.all(err[fin] <= tol), (np.max(err[fin]), idx[np.argmax(np.where(fin, err, 0))])
    return err[fin]


# ------------------------------------------------------------------ cfg 1 -----
def test_cfg1_all_points(fpe):
    a = workloads.coefficients(1)
    pts = workloads.points(1)
    poly = fpe.precondition(a)
    P = oracle.OraclePoly(a)
    out = gpu_eval(poly, pts)
    cls = check_indexing(P, pts, out["diag"])
    err = _values_ok(P, a, pts, out, np.arange(len(pts)), TOL64, cls)
    assert np.max(err) < 2.0 ** -48
    # Theorem thm:equivAlgo on the sphere: mean #[l, r] < 1 + 1.9046 sqrt(d (p + s(d) + 3))
    width = cls["r"] - cls["l"] + 1
    assert width.mean() < 1 + 1.9046 * math.sqrt(P.d_eff * P.drop)


def test_worked_example_through_abi(fpe, worked):
    s = np.array(worked["scales"])
    a = np.ldexp(1.0, s - 1).astype(np.complex128)
    pts = np.array([np.exp(0.3j), 0.125 * np.exp(1.1j), 1.0 + 0j, 0.125 + 0j])
    for drop, tag in ((6, "drop6"), (None, "drop13")):
        poly = fpe.precondition(a, p=6, drop=drop)
        out = gpu_eval(poly, pts)
        d = out["diag"]
        band = worked["derived_not_printed"]["band_" + tag]
        W = worked["derived_not_printed"]["W_" + tag]
        for i in (0, 2):
            assert [d["l"][i], d["r"][i]] == band["lambda0"] and d["kept"][i] == len(W["lambda0"])
        for i in (1, 3):
            assert [d["l"][i], d["r"][i]] == band["lambda_m3"] and d["kept"][i] == len(W["lambda_m3"])
        P = oracle.OraclePoly(a, p=6, drop=drop)
        check_indexing(P, pts, d)


def test_special_points(fpe):
    a = workloads.coefficients(1, d=200)
    poly = fpe.precondition(a)
    P = oracle.OraclePoly(a)
    hk, hh = P.hk, P.hh
    sp = [0j, 1 + 0j, -1 + 0j, 1j, -1j, 2.0 + 0j, 0.5j, 2.0 ** -1074 + 0j, complex(2.0 ** 1000, 0),
          complex(1e300, 1e300), complex(1e-300, 1e-310), complex(1.0, 2.0 ** -30), complex(1.0, 1e-200),
          complex(1 - 2 ** -53, 2 ** -26), complex(math.nextafter(1.0, 2.0), 0), complex(0.6, 0.8),
          complex(3 / 5, -4 / 5), np.exp(1j * 2.0), complex(math.sqrt(0.5), math.sqrt(0.5))]
    # |z| = 2^slope exactly for integer hull slopes (argmax ties), and dyadic radii
    for j in range(len(hk) - 1):
        sl = (hh[j + 1] - hh[j]) / (hk[j + 1] - hk[j])
        if float(sl).is_integer():
            sp.append(complex(2.0 ** (-sl), 0))
    rng = np.random.default_rng(3)
    for _ in range(300):
        t = rng.uniform(0, 2 * np.pi)
        sp.append(np.exp(1j * t) * (1 + rng.choice([-1, 1]) * 2.0 ** -rng.integers(1, 60)))
    pts = np.array(sp, dtype=np.complex128)
    out = gpu_eval(poly, pts)
    cls = check_indexing(P, pts, out["diag"])
    finite = np.isfinite(pts)
    _values_ok(P, a, pts, out, np.flatnonzero(finite & (pts != 0)), TOL64, cls)
    # z = 0 gives a_0 exactly
    v0 = out["v"][0] * 2.0 ** out["e"][0]
    assert v0 == a[0]
    nanpts = np.array([complex(np.nan, 0), complex(np.inf, 1), complex(0, -np.inf)])
    o2 = gpu_eval(poly, nanpts)
    assert np.all(np.isnan(o2["v"].real)) and np.all(o2["diag"]["region"] == -1)


def test_empty_and_ragged(fpe):
    a = workloads.coefficients(1, d=50)
    poly = fpe.precondition(a)
    P = oracle.OraclePoly(a)
    e = torch.empty(0, dtype=torch.complex128, device="cuda")
    v, ex = poly.evaluate(e)
    assert v.numel() == 0
    for n in (1, 31, 127, 129, 1000, 4097):
        pts = workloads.sphere_points(1, n)
        out = gpu_eval(poly, pts)
        cls = check_indexing(P, pts, out["diag"])
        _values_ok(P, a, pts, out, np.arange(n), TOL64, cls)


# ------------------------------------------------------- full-size configs ----
# (every point of cfg2-5 and cfg5-fp32 against the oracle: tests/test_gpu_fullsize.py)
# --------------------------------------------------------- other entry points --
def test_horner_context(fpe):
    a = workloads.coefficients(1)
    pts = workloads.points(1, 2048)
    poly = fpe.precondition(a)
    P = oracle.OraclePoly(a)
    out = gpu_eval(poly, pts, horner=True)
    H = P.horner(pts)
    l2S = abs_sum_log2(a, pts)
    err = rel_err_vs(H, out["v"], out["e"], l2S)
    assert np.all(err <= TOL64), err.max()
    # large degree and large |z|: exponent tracking (cfg3 family, 16 points)
    a3 = workloads.coefficients(3, d=(1 << 16) - 1)
    p3 = workloads.points(3, 16) * np.array([1, 1e3, 1e-3, 7] * 4)
    poly3 = fpe.precondition(a3)
    P3 = oracle.OraclePoly(a3)
    out = gpu_eval(poly3, p3, horner=True)
    err = rel_err_vs(P3.horner(p3), out["v"], out["e"], abs_sum_log2(a3, p3))
    assert np.all(err <= TOL64), err.max()
    # real coefficients at real points (cfg2 family), and fp32 (cfg5 family), huge and tiny |z|
    for cfg, fp32, tol in ((2, False, TOL64), (5, True, TOL32)):
        ac = workloads.coefficients(cfg, d=(1 << 12) - 1)
        pc = workloads.points(cfg, 200)
        pc = np.concatenate([pc, pc[:20] * 1e6, pc[20:40] * 1e-6])
        if fp32:
            ac, pc = workloads.to_fp32(ac), workloads.to_fp32(pc)
        polyc = fpe.precondition(ac)
        Pc = oracle.OraclePoly(ac)
        out = gpu_eval(polyc, pc, horner=True)
        err = rel_err_vs(Pc.horner(pc), out["v"], out["e"], abs_sum_log2(ac, pc))
        assert np.all(err <= tol), (cfg, err.max())


@pytest.mark.parametrize("kind", ["c64", "r64", "c32", "long"])
def test_evaluate_host_matches_device(fpe, kind):
    """fpe_evaluate_host (pipelined host buffers, several chunks and kernel streams) gives the device
    path's bits, for complex / real / fp32 points and with tensor-core pieces (cfg3; the DMMA scratch
    does not overflow at this distribution, see fpe.h on the one exception)."""
    if kind == "long":   # cfg3's polynomial and point distribution: tensor-core pieces in every chunk
        a = workloads.coefficients(3)
        pts = workloads.points(3, (1 << 22) + (1 << 21) + 123)   # three chunks of the host pipeline
    else:
        a = workloads.coefficients(1)
        pts = workloads.points(1)
        if kind == "r64":
            a, pts = a.real.copy(), pts.real.copy()
        elif kind == "c32":
            a, pts = workloads.to_fp32(a), workloads.to_fp32(pts)
    poly = fpe.precondition(a)
    out = gpu_eval(poly, pts, diag=False)
    hv, he = poly.evaluate_host(pts)
    assert np.array_equal(hv, out["v"]) and np.array_equal(he, out["e"])


def test_determinism_permutation_and_batches(fpe):
    a = workloads.coefficients(3, d=(1 << 16) - 1)
    pts = workloads.points(3, 1 << 15)
    poly = fpe.precondition(a)
    base = gpu_eval(poly, pts, diag=False)
    perm = np.random.default_rng(9).permutation(len(pts))
    o = gpu_eval(poly, pts[perm], diag=False)
    assert np.array_equal(o["v"], base["v"][perm]) and np.array_equal(o["e"], base["e"][perm])
    parts = [gpu_eval(poly, pts[i:i + 5000], diag=False) for i in range(0, len(pts), 5000)]
    assert np.array_equal(np.concatenate([p["v"] for p in parts]), base["v"])


def test_buffer_roundtrip(fpe):
    a = workloads.coefficients(4, d=1 << 16)
    poly = fpe.precondition(a)
    ptr, nb = poly.device_buffer()
    poly2 = fpe.Poly.from_buffer(ptr, nb, device=0)
    host = fpe.precondition_buffer(a)
    poly3 = fpe.Poly.from_buffer(host.ctypes.data, len(host), device=0)
    pts = workloads.points(4, 4096)
    o1, o2, o3 = (gpu_eval(p, pts, diag=False) for p in (poly, poly2, poly3))
    assert np.array_equal(o1["v"], o2["v"]) and np.array_equal(o1["v"], o3["v"])
    with pytest.raises(fpe.FpeError):
        bad = np.zeros(512, np.uint8)
        fpe.Poly.from_buffer(bad.ctypes.data, len(bad), device=0)


def test_plain_float_output(fpe):
    a = workloads.coefficients(1, d=30)
    poly = fpe.precondition(a)
    pts = workloads.points(1, 1000)
    t = torch.from_numpy(pts).cuda()
    v1, e1 = poly.evaluate(t, exps=True)
    v2, _ = poly.evaluate(t, exps=False)
    v1, e1, v2 = v1.cpu().numpy(), e1.cpu().numpy(), v2.cpu().numpy()
    ref_re = np.ldexp(v1.real, np.clip(e1, -4000, 4000).astype(np.int32))
    ref_im = np.ldexp(v1.imag, np.clip(e1, -4000, 4000).astype(np.int32))
    assert np.array_equal(v2.real, ref_re) and np.array_equal(v2.imag, ref_im)


def test_diag_and_plain_paths_agree(fpe):
    """The classifier decides windows on an enclosure of log2|z| and falls back to the correctly rounded
    lambda only when undecided; with diagnostics on it also reports the rounded lambda.  Both runs must
    give bitwise-identical values (the windows, hence the arithmetic, are the same)."""
    for cfg, d in ((3, (1 << 18) - 1), (2, (1 << 16) - 1), (1, None)):
        a = workloads.coefficients(cfg, d=d)
        pts = workloads.points(cfg, 1 << 16, shard=3)
        poly = fpe.precondition(a)
        o1 = gpu_eval(poly, pts, diag=True)
        o2 = gpu_eval(poly, pts, diag=False)
        assert np.array_equal(o1["v"], o2["v"]) and np.array_equal(o1["e"], o2["e"]), cfg


def test_confidence_cancel_bits(fpe):
    """fpe_diag::cancel (eq:def_prec_loss): c = 0 if |P(z)| >= M, else s(M) - s(P(z)),
    M = max_k |a_k z^k|.  The library estimates s(M) by ceil(N_lambda) (log2 M in [N - 1, N)) and takes s of
    its own result; against the oracle's s(M) and s(P_ref) it may differ by 1 for each estimate.  The error
    bound err_exp must hold against the oracle's full Horner, and trusted = s(Q) - err_exp (clamped)."""
    cases = [(workloads.coefficients(1), workloads.points(1, 4096, shard=4))]
    # heavy cancellation: (z - 1)^40 near z = 1 loses many bits
    from math import comb
    a = np.array([comb(40, k) * (-1.0) ** (40 - k) for k in range(41)], dtype=np.complex128)
    zc = 1 + 2.0 ** -np.arange(1, 30) * np.exp(1j * np.linspace(0, 6, 29))
    cases.append((a, np.concatenate([zc, workloads.points(1, 500, shard=5)])))
    # a dominant term: |P(z)| >= M happens (c = 0 by the first case of eq:def_prec_loss)
    b = np.zeros(30, np.complex128); b[0] = 1.0; b[29] = 1e-3
    cases.append((b, workloads.points(1, 500, shard=6) * 0.5))
    for a, pts in cases:
        poly = fpe.precondition(a)
        P = oracle.OraclePoly(a)
        out = gpu_eval(poly, pts)
        c_gpu = out["diag"]["cancel"]
        H = P.horner(pts)
        sP = H.e + (np.abs(H.hi) >= 1.0)
        sM = 1 + np.floor(P.log2_maxterm(pts)).astype(np.int64)
        l2M = P.log2_maxterm(pts)
        absP_ge_M = (np.log2(np.abs(H.hi)) + H.e) >= l2M
        c_ref = np.where(absP_ge_M, 0, sM - sP)
        ok = np.isfinite(l2M) & (c_ref < 40)
        assert np.all(c_gpu[ok] >= 0)
        assert np.all(np.abs(c_gpu[ok] - c_ref[ok]) <= 2), (c_gpu[ok][:10], c_ref[ok][:10])
        assert np.any(c_ref[ok] > 10) or a.shape[0] != 41   # the (z-1)^40 case does exercise cancellation
        # the error bound holds: |P_gpu - P_ref| <= 2^err_exp (relative to 2^err_exp, exponents aligned)
        ee = out["diag"]["err_exp"].astype(np.int64)
        sh = np.clip(out["e"] - ee, -2000, 2000)
        g = np.ldexp(out["v"].real, sh) + 1j * np.ldexp(out["v"].imag, sh)
        diff = np.abs(g - H.scaled(ee))
        assert np.all(diff[ok] <= 1.0), diff[ok].max()
        sQ = out["e"] + (np.abs(out["v"]) >= 1.0)
        tr = out["diag"]["trusted"]
        assert np.all(tr == np.clip(sQ - ee, 0, 53))
        assert np.median(tr[ok & (c_ref == 0)]) >= 20 or a.shape[0] == 41


def test_newton_step_paper_example(fpe):
    """P(z) = z^64 + 1, p = 24 (FP32): P(10) and P'(10) overflow FP32, yet the Newton
    increment 10 - N_P(10) = 0.15625 (exact to 2e-65) comes out of the FP32 path."""
    a = np.zeros(65, dtype=np.float32)
    a[0] = 1.0
    a[64] = 1.0
    P = fpe.precondition(a)
    dP = fpe.precondition_derivative(a)
    z = torch.tensor([10.0], dtype=torch.float32, device="cuda")
    zn, inc = fpe.newton_step(P, dP, z, incr=True)
    assert inc.item() == 0.15625 and zn.item() == 10.0 - 0.15625


def test_newton_step_vs_oracle(fpe):
    """N_P(z) = z - P(z)/P'(z) (eq:newton) against binary128 full Horner of P and of P' (whose coefficients
    (j+1) a_{j+1} are formed with the same single fp64 rounding as the library's)."""
    a = workloads.coefficients(1, d=300)
    pts = workloads.points(1, 3000, shard=6)
    P = fpe.precondition(a)
    dP = fpe.precondition_derivative(a)
    zn, inc = fpe.newton_step(P, dP, torch.from_numpy(pts).cuda(), incr=True)
    inc = inc.cpu().numpy()
    da = (np.arange(1, len(a)) * a[1:].real) + 1j * (np.arange(1, len(a)) * a[1:].imag)
    H1 = oracle.OraclePoly(a).horner(pts)
    H2 = oracle.OraclePoly(da).horner(pts)
    ref = (H1.hi + H1.lo) / (H2.hi + H2.lo) * np.exp2((H1.e - H2.e).astype(np.float64))
    # condition: the library's values are within 2^-45 S of P and P'; compare where both are well away
    # from cancellation (|P| >= 2^-20 S_P and |P'| >= 2^-20 S_P')
    c1 = abs_sum_log2(a, pts) - (np.log2(np.abs(H1.hi)) + H1.e)
    c2 = abs_sum_log2(da, pts) - (np.log2(np.abs(H2.hi)) + H2.e)
    ok = (c1 < 20) & (c2 < 20) & np.isfinite(ref)
    assert ok.mean() > 0.9
    rel = np.abs(inc[ok] - ref[ok]) / np.abs(ref[ok])
    assert np.all(rel < 2.0 ** -40), rel.max()
    assert np.allclose(zn.cpu().numpy()[ok], pts[ok] - inc[ok], rtol=0, atol=0)


def test_half_circle_family(fpe):
    """Second workload: the half-circle family, the slowest family of
    the paper, d = 1000 (coefficients up to 2^500): indexing bit-exact and values within 2^-45 S."""
    d = 1000
    n = np.arange(d + 1)
    a = np.exp2(np.sqrt((n + 1.0) * (d + 1.0 - n))).astype(np.complex128)
    pts = workloads.sphere_points(1, 1 << 14, shard=11)
    poly = fpe.precondition(a)
    P = oracle.OraclePoly(a)
    out = gpu_eval(poly, pts)
    cls = check_indexing(P, pts, out["diag"])
    _values_ok(P, a, pts, out, np.arange(0, len(pts), 8), TOL64, cls)


def _many_vertex_coeffs(m, cplx, seed):
    """A concave cover with 2m + 1 vertices: edges (q, +1) for q = 1..m then (q, -1) for q = m..1
    (strictly decreasing slopes), the other terms 8 bits below it; scales span m bits."""
    ks, hs = [0], [-m]
    for q in list(range(1, m + 1)) + list(range(m, 0, -1)):
        ks.append(ks[-1] + q)
        hs.append(hs[-1] + (1 if len(ks) <= m + 1 else -1))
    kk = np.arange(ks[-1] + 1)
    sc = np.floor(np.interp(kk, ks, hs)).astype(np.int64) - 8
    sc[ks] = hs
    a = np.ldexp(1.5, sc - 1)   # scale(a_k) = sc_k (1.5 keeps it through the phase rounding)
    if cplx:
        a = a * np.exp(1j * np.random.default_rng(seed).uniform(0, 2 * np.pi, len(a)))
    return a


@pytest.mark.parametrize("cplx", [True, False])
def test_many_vertex_cover(fpe, cplx):
    """A cover of 1601 vertices: more than the classifier stages in shared memory (1536), so the
    bucketing classifier searches the cover in global memory (eval_tiled.cu k_classify_bucket)."""
    a = _many_vertex_coeffs(800, cplx, 5)
    poly = fpe.precondition(a)
    P = oracle.OraclePoly(a)
    assert len(P.hk) == 1601
    rng = np.random.default_rng(6)
    n = 4000
    r = np.exp2(rng.uniform(-1.2, 1.2, n))
    pts = r * np.exp(1j * rng.uniform(0, 2 * np.pi, n)) if cplx else r * rng.choice([-1.0, 1.0], n)
    pts = np.concatenate([pts, [0.5, 2.0, 1.0, -1.0, 2.0 ** (-1 / 3)]]).astype(pts.dtype)
    out = gpu_eval(poly, pts)
    cls = check_indexing(P, pts, out["diag"])
    _values_ok(P, a, pts, out, np.arange(0, len(pts), 16), TOL64, cls)


def test_sparse_many_terms(fpe):
    """Sparse handle with 20000 good terms (> the 8192 the sparse evaluator stages in shared
    memory, kernels.cu k_eval_sparse), d = 2^20: global-index path, indexing exact, values 2^-45 S."""
    rng = np.random.default_rng(12)
    d = 1 << 20
    a = np.zeros(d + 1, np.complex128)
    idx = np.unique(np.concatenate([[0, d], rng.integers(1, d, 20000)]))
    a[idx] = rng.uniform(-1, 1, len(idx)) + 1j * rng.uniform(-1, 1, len(idx))
    poly = fpe.precondition(a)
    P = oracle.OraclePoly(a)
    assert int(P.good.sum()) > 8192 and int(P.good.sum()) * 32 < d + 1
    pts = np.exp2(rng.uniform(-0.01, 0.01, 3000)) * np.exp(1j * rng.uniform(0, 2 * np.pi, 3000))
    out = gpu_eval(poly, pts)
    cls = check_indexing(P, pts, out["diag"])
    _values_ok(P, a, pts, out, np.arange(0, len(pts), 10), TOL64, cls)


def test_sparse_determinism_long_lists(fpe):
    """Sparse evaluator: points with long kept lists (K > 32: summed by the whole warp, strided partials
    and a fixed tree) mixed with short ones (flat round-robin list, summed per lane) -- bitwise the same
    results under a permutation of the batch and under batch slicing (a point's result must not depend
    on its warp-mates or on the work-queue order); values against the oracle on a sample."""
    rng = np.random.default_rng(13)
    d = 1 << 20
    a = np.zeros(d + 1, np.complex128)
    idx = np.unique(np.concatenate([[0, d], rng.integers(1, d, 20000)]))
    a[idx] = rng.uniform(-1, 1, len(idx)) + 1j * rng.uniform(-1, 1, len(idx))
    poly = fpe.precondition(a)
    P = oracle.OraclePoly(a)
    near = np.exp2(rng.uniform(-0.002, 0.002, 3000)) * np.exp(1j * rng.uniform(0, 2 * np.pi, 3000))
    pts = np.concatenate([near, workloads.points(3, 3000)])
    pts = pts[rng.permutation(len(pts))]
    base = gpu_eval(poly, pts)
    K = base["diag"]["kept"]
    assert (K > 32).sum() > 500 and (K <= 32).sum() > 500
    perm = rng.permutation(len(pts))
    o = gpu_eval(poly, pts[perm], diag=False)
    assert np.array_equal(o["v"], base["v"][perm]) and np.array_equal(o["e"], base["e"][perm])
    parts = [gpu_eval(poly, pts[i:i + 777], diag=False) for i in range(0, len(pts), 777)]
    assert np.array_equal(np.concatenate([q["v"] for q in parts]), base["v"])
    assert np.array_equal(np.concatenate([q["e"] for q in parts]), base["e"])
    cls = check_indexing(P, pts, base["diag"])
    _values_ok(P, a, pts, base, np.arange(0, len(pts), 12), TOL64, cls)


# ------------------------------------------------- device preconditioner ----
def _gpu_buffer(fpe, a):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    poly = fpe.precondition_gpu(t)
    out = np.zeros(poly.nbytes, np.uint8)
    poly.export(out.ctypes.data, len(out))
    torch.cuda.synchronize()
    return poly, out


def _precondition_cases(rng):
    d = 1 << 20
    sp = np.zeros(d + 1, np.complex128)
    idx = np.unique(np.concatenate([[0, d], rng.integers(1, d, 20000)]))
    sp[idx] = rng.uniform(-1, 1, len(idx)) + 1j * rng.uniform(-1, 1, len(idx))
    cases = [workloads.coefficients(1), workloads.coefficients(2), workloads.coefficients(3),
             workloads.coefficients(5), workloads.to_fp32(workloads.coefficients(5)),
             workloads.to_fp32(workloads.coefficients(2)), _many_vertex_coeffs(800, True, 5),
             _many_vertex_coeffs(800, False, 5), sp,
             np.array([0.0, 0.0, 3.0]), np.array([1.0, 1.0]), np.array([0, 0, 1 + 1j, 0, 0, 0, 2j, 0]),
             np.full(100, 0.5 + 0.5j), np.array([5e-324, 1.0, 1e300]), np.array([2.0 ** -1074 + 0j]),
             np.ldexp(1.0, np.floor(300 * np.sin(np.pi * np.arange(4001) / 4000)).astype(int))]
    for _ in range(30):
        n = int(rng.integers(1, 5000))
        a = rng.normal(size=n) * np.exp2(rng.integers(-60, 60, size=n))
        a[rng.random(n) < 0.4] = 0
        if not a.any():
            a[-1] = 1
        cases.append(a)
        cases.append(a * np.exp(1j * rng.uniform(0, 6.3, n)))
        cases.append(workloads.to_fp32(a * np.exp(1j * rng.uniform(0, 6.3, n))))
    return cases


def test_precondition_gpu_matches_host(fpe):
    """fpe_precondition_gpu (scales, chunked + merged monotone chains, G_p, scan) builds a flat buffer
    byte-identical to the host preconditioner's, which the oracle pins (test_abi_host.py)."""
    rng = np.random.default_rng(31)
    for ci, a in enumerate(_precondition_cases(rng)):
        try:
            host = fpe.precondition_buffer(a)
        except fpe.FpeError as e:
            with pytest.raises(fpe.FpeError) as e2:
                _gpu_buffer(fpe, a)
            assert e2.value.status == e.status
            continue
        try:
            poly, dev = _gpu_buffer(fpe, a)
        except fpe.FpeError as e:
            raise AssertionError(f"case {ci}: {a.dtype} n={len(a)} {a[:4]}: {e}")
        assert len(host) == len(dev) and np.array_equal(host, dev), (a.dtype, len(a))
        hk, hh = poly.hull()
        P = oracle.OraclePoly(a)
        assert np.array_equal(hk, P.hk) and np.array_equal(hh, P.hh)


def test_precondition_gpu_errors(fpe):
    for a, status in ((np.zeros(100), 2), (np.array([1.0, np.nan, 2.0]), 3),
                      (np.array([1.0, np.inf + 0j]), 3)):
        t = torch.from_numpy(a).cuda()
        with pytest.raises(fpe.FpeError) as e:
            fpe.precondition_gpu(t)
        assert e.value.status == status
        with pytest.raises(fpe.FpeError) as e2:
            fpe.precondition(a)
        assert e2.value.status == status


def test_partial_preprocessing(fpe):
    """Remark rem:partialpreproc: one cover (lines 2-3), finished for several p
    (line 4) in O(d); every finished buffer equals the host preconditioner's at that p, byte for byte."""
    rng = np.random.default_rng(41)
    cases = [workloads.coefficients(3), workloads.to_fp32(workloads.coefficients(5)), _many_vertex_coeffs(300, True, 2)]
    a = rng.normal(size=3000) * np.exp2(rng.integers(-40, 40, 3000))
    a[rng.random(3000) < 0.5] = 0
    cases.append(a)
    for a in cases:
        cover = fpe.Cover(torch.from_numpy(np.ascontiguousarray(a)).cuda())
        for p in (0, 53, 30, 12, 4):
            try:
                host = fpe.precondition_buffer(a, p=p or None)
            except fpe.FpeError as e:
                with pytest.raises(fpe.FpeError) as e2:
                    cover.finish(p=p or None)
                assert e2.value.status == e.status
                continue
            poly = cover.finish(p=p or None)
            dev = np.zeros(poly.nbytes, np.uint8)
            poly.export(dev.ctypes.data, len(dev))
            torch.cuda.synchronize()
            assert np.array_equal(host, dev), (a.dtype, len(a), p)
        cover.close()


def test_analyse_intervals(fpe, worked):
    """-analyse: the lambda intervals of constant (i*, l, r) tile [lo, hi], neighbours
    differ, and every interval's triple (and kept count) is the oracle's at points inside it; on the
    paper's worked example the intervals through lambda = 0 and -3 carry the printed bands."""
    s = np.array(worked["scales"])
    wa = np.ldexp(1.0, s - 1).astype(np.complex128)
    rng = np.random.default_rng(51)
    b = rng.normal(size=600) * np.exp2(rng.integers(-30, 30, 600))
    b[rng.random(600) < 0.6] = 0
    cases = [(wa, 6), (wa, None), (workloads.coefficients(1, d=200), None), (b, None),
             (_many_vertex_coeffs(40, True, 3), None)]
    for a, drop in cases:
        poly = fpe.precondition(a, p=6 if drop else None, drop=drop)
        P = oracle.OraclePoly(a, p=6 if drop else None, drop=drop)
        iv = poly.analyse(-12.0, 12.0)
        assert iv[0]["lam_lo"] == -12.0 and iv[-1]["lam_hi"] == 12.0
        assert np.all(iv["lam_hi"][:-1] == iv["lam_lo"][1:])
        trip = np.stack([iv["region"], iv["l"], iv["r"]], 1)
        assert np.all(np.any(trip[1:] != trip[:-1], axis=1))
        for f in (0.5, 0.01, 0.99):
            lam = iv["lam_lo"] + f * (iv["lam_hi"] - iv["lam_lo"])
            ist, l, r = P.search(lam)
            assert np.array_equal(ist, iv["region"]) and np.array_equal(l, iv["l"]) and np.array_equal(r, iv["r"])
            K = P.good_prefix[r + 1] - P.good_prefix[l]
            assert np.array_equal(K, iv["kept"])
        if drop == 6:
            band = worked["derived_not_printed"]["band_drop6"]
            for lam, key in ((0.0, "lambda0"), (-3.0, "lambda_m3")):
                j = np.flatnonzero((iv["lam_lo"] < lam) & (lam < iv["lam_hi"]))
                if len(j):
                    assert [iv["l"][j[0]], iv["r"][j[0]]] == band[key]


@pytest.mark.parametrize("real_points", [False, True])
def test_tensor_core_pieces_and_overflow(fpe, real_points):
    """Points near |z| = 1 on cfg3's polynomial have windows of 10^5 coefficients: most pieces are covered
    whole and go to k_eval_mma; 400 points (4 groups) request more DMMA items than the small batch's
    scratch holds (64), so some groups run them in-warp (k_eval_overflow).  Indexing exact, values within
    2^-45 S, against the oracle; complex and real points."""
    a = workloads.coefficients(3)
    P = oracle.OraclePoly(a)
    rng = np.random.default_rng(61)
    n = 400
    r = np.exp2(rng.uniform(-2.0 ** -12, 2.0 ** -12, n))
    pts = r * rng.choice([-1.0, 1.0], n) if real_points else r * np.exp(1j * rng.uniform(0, 2 * np.pi, n))
    poly = fpe.precondition(a)
    out = gpu_eval(poly, pts)
    cls = check_indexing(P, pts, out["diag"])
    assert np.median(cls["K"]) > 3 * 16384   # long windows: several whole pieces per point
    _values_ok(P, a, pts, out, np.arange(0, n, 8), TOL64, cls)


@pytest.mark.parametrize("coef_kind,pt_kind", [("r", "r"), ("r", "c"), ("c", "r"), ("c", "c")])
@pytest.mark.parametrize("fp32", [False, True])
def test_dtype_combinations(fpe, coef_kind, pt_kind, fp32):
    """Every (coefficient, point) dtype pair the evaluator instantiates (real/complex x real/complex, fp64
    and fp32): indexing exact, values within the dtype's tolerance, on a polynomial with zero
    coefficients and a 2^+-40 dynamic range and points spanning |z| in [2^-6, 2^6] with a cluster at 1."""
    rng = np.random.default_rng(81 + 2 * fp32)
    d = 3000
    a = rng.normal(size=d + 1) * np.exp2(rng.uniform(-40, 0, d + 1))
    a[rng.random(d + 1) < 0.3] = 0.0
    if coef_kind == "c":
        a = a * np.exp(1j * rng.uniform(0, 2 * np.pi, d + 1))
    n = 4000
    r = np.concatenate([np.exp2(rng.uniform(-6, 6, n // 2)), np.exp2(rng.uniform(-2.0 ** -8, 2.0 ** -8, n // 2))])
    pts = r * (np.exp(1j * rng.uniform(0, 2 * np.pi, n)) if pt_kind == "c" else rng.choice([-1.0, 1.0], n))
    if fp32:
        a, pts = workloads.to_fp32(a), workloads.to_fp32(pts)
    poly = fpe.precondition(a)
    P = oracle.OraclePoly(a)
    out = gpu_eval(poly, pts)
    cls = check_indexing(P, pts, out["diag"])
    _values_ok(P, a, pts, out, np.arange(0, n, 4), TOL32 if fp32 else TOL64, cls)


def test_special_points_fp32(fpe):
    """Single-precision points at the edges of their format (subnormal, near FLT_MAX, exact powers of two,
    within one ulp of |z| = 1, zero, NaN/inf): indexing exact, values within 2^-16 S, z = 0 gives a_0."""
    a = workloads.to_fp32(workloads.coefficients(1, d=200))
    poly = fpe.precondition(a)
    P = oracle.OraclePoly(a)
    f = np.float32
    one_up, one_dn = np.nextafter(f(1), f(2)), np.nextafter(f(1), f(0))
    sp = [0, 1, -1, 1j, -1j, 2, 0.5j, np.finfo(f).tiny, f(1e-45), np.finfo(f).max / 2, complex(3e38, 3e38),
          complex(one_up, 0), complex(one_dn, 0), complex(one_dn, f(1e-4)), complex(0.6, 0.8), complex(1e-38, 1e-40)]
    rng = np.random.default_rng(91)
    for _ in range(300):
        t = rng.uniform(0, 2 * np.pi)
        sp.append(np.exp(1j * t) * (1 + rng.choice([-1, 1]) * 2.0 ** -rng.integers(1, 24)))
    pts = np.array(sp, dtype=np.complex64)
    out = gpu_eval(poly, pts)
    cls = check_indexing(P, pts, out["diag"])
    nz = np.flatnonzero(pts != 0)
    _values_ok(P, a, pts, out, nz, TOL32, cls)
    assert out["v"][0] * 2.0 ** out["e"][0] == a[0]
    nanpts = np.array([complex(np.nan, 0), complex(np.inf, 1)], dtype=np.complex64)
    o2 = gpu_eval(poly, nanpts)
    assert np.all(np.isnan(o2["v"].real)) and np.all(o2["diag"]["region"] == -1)


def test_tensor_core_pieces_with_k_min(fpe):
    """Long windows on a polynomial whose first 1000 coefficients are zero (k_min = 1000; pieces and
    chunks are relative to k_min): indexing exact, values within 2^-45 S."""
    a = np.concatenate([np.zeros(1000, np.complex128), workloads.coefficients(3)[: (1 << 18)]])
    P = oracle.OraclePoly(a)
    assert P.k_min == 1000
    rng = np.random.default_rng(62)
    n = 1000
    pts = np.exp2(rng.uniform(-2.0 ** -14, 2.0 ** -14, n)) * np.exp(1j * rng.uniform(0, 2 * np.pi, n))
    poly = fpe.precondition(a)
    out = gpu_eval(poly, pts)
    cls = check_indexing(P, pts, out["diag"])
    assert np.median(cls["K"]) > 2 * 16384
    _values_ok(P, a, pts, out, np.arange(0, n, 10), TOL64, cls)


def test_batch_slicing_above_2_28(fpe):
    """fpe_evaluate slices batches above 2^28 points (the bucketing's index range): 2^28 + 4097 points,
    the ones around the slice boundary and a random sample checked against the oracle, and the slice
    boundary invisible in the results (the same points evaluated alone give the same bits)."""
    a = workloads.coefficients(1)
    P = oracle.OraclePoly(a)
    poly = fpe.precondition(a)
    n = (1 << 28) + 4097
    g = torch.Generator(device="cuda").manual_seed(5)
    t = torch.complex(torch.randn(n, device="cuda", dtype=torch.float64, generator=g),
                      torch.randn(n, device="cuda", dtype=torch.float64, generator=g))
    v, e, dg = poly.evaluate(t, exps=True, diag=True)
    idx = np.concatenate([np.arange((1 << 28) - 64, (1 << 28) + 64), np.arange(n - 8, n),
                          workloads.sample_indices(n, 2048, salt=7)])
    idx = np.unique(idx)
    it = torch.from_numpy(idx).cuda()
    pts = t[it].cpu().numpy()
    D = {k: x[it].cpu().numpy() for k, x in fpe.diag_fields(dg).items()}
    out = {"v": v[it].cpu().numpy(), "e": e[it].cpu().numpy()}
    del v, e, dg
    torch.cuda.empty_cache()
    cls = check_indexing(P, pts, D)
    _values_ok(P, a, pts, out, np.arange(len(idx)), TOL64, cls)
    alone = gpu_eval(poly, pts)
    assert np.array_equal(alone["v"], out["v"]) and np.array_equal(alone["e"], out["e"])


@pytest.mark.parametrize("fp32", [False, True])
def test_coherent_long_windows(fpe, fp32):
    """Coherent terms (a_k = 1, d = 2^20 - 1) at z within 2^-14 of 1 with small argument, complex and real:
    every term has nearly the same phase, so the Horner rounding errors of a 16384-coefficient piece add up
    like sum_j u |b_j| instead of cancelling at random -- the hardest case for the window evaluator's
    accuracy, against the oracle's full binary128 Horner (the plain definition), tolerance 2^-45 S (fp64) /
    2^-16 S (fp32).  Complex points take the tensor-core pieces (k_eval_mma) in fp64."""
    d = (1 << 20) - 1
    a = np.ones(d + 1, np.complex128)
    rng = np.random.default_rng(71)
    m = 24
    eps = rng.uniform(-2.0 ** -14, 2.0 ** -14, m)
    th = rng.uniform(-2.0 ** -14, 2.0 ** -14, m)
    zc = (1 + eps) * np.exp(1j * th)
    zc[:4] = [1.0, 1 + 2.0 ** -14, 1 - 2.0 ** -14, np.exp(1j * 2.0 ** -14)]
    zr = 1 + rng.uniform(-2.0 ** -14, 2.0 ** -14, m)
    tol = TOL32 if fp32 else TOL64
    worst = {}
    for kind, pts, coef in (("complex", zc, a), ("real", zr, a.real.copy())):
        if fp32:
            coef, pts = workloads.to_fp32(coef), workloads.to_fp32(pts)
        poly = fpe.precondition(coef)
        P = oracle.OraclePoly(coef)
        out = gpu_eval(poly, pts)
        check_indexing(P, pts, out["diag"])
        H = P.horner_dd(pts)
        l2S = abs_sum_log2(coef, pts)
        err = rel_err_vs(H, out["v"], out["e"], l2S)
        worst[kind] = float(np.log2(max(err.max(), 2.0 ** -200)))
        assert np.all(err <= tol), (kind, err.max())
    print(f"\ncoherent a_k = 1, d = 2^20 - 1, {'fp32' if fp32 else 'fp64'}: max err/S = 2^{worst}")


def test_cfg5_fp32_near_unit_circle(fpe):
    """cfg5-fp32 (d = 2^22 - 1, the longest fp32 windows: ~4 10^5 terms) at points within 2^-12 of
    |z| = 1: values against the oracle's full Horner within 2^-16 S."""
    a = workloads.to_fp32(workloads.coefficients(5))
    rng = np.random.default_rng(72)
    m = 48
    pts = workloads.to_fp32(np.exp2(rng.uniform(-2.0 ** -12, 2.0 ** -12, m)) * np.exp(1j * rng.uniform(0, 2 * np.pi, m)))
    poly = fpe.precondition(a)
    P = oracle.OraclePoly(a)
    out = gpu_eval(poly, pts)
    cls = check_indexing(P, pts, out["diag"])
    assert np.median(cls["K"]) > 1e5
    H = P.horner_dd(pts)
    err = rel_err_vs(H, out["v"], out["e"], abs_sum_log2(a, pts))
    print(f"\ncfg5-fp32 near |z| = 1: median K = {int(np.median(cls['K']))}, max err/S = 2^{np.log2(err.max()):.1f}")
    assert np.all(err <= TOL32), err.max()


def test_replicate_and_evaluate_shard_nccl_world1(fpe):
    """dist.replicate (export + NCCL broadcast + fpe_poly_from_device_buffer) and dist.evaluate_shard through
    a real NCCL process group (world size 1 on the one GPU of this box): the imported handle evaluates
    bitwise like the source, and from a host precondition_buffer as well."""
    import socket

    import torch.distributed as dist

    from paper_2211_06320_b200 import dist as fdist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        a = workloads.coefficients(3, d=(1 << 16) - 1)
        poly = fpe.precondition(a)
        pts = workloads.points(3, 1 << 15)
        (lo, hi), v, e = fdist.evaluate_shard(poly, pts)
        assert (lo, hi) == (0, len(pts))
        rep = fdist.replicate(fpe.precondition_buffer(a), src=0, device=0)
        v2, e2 = rep.evaluate(torch.from_numpy(pts).cuda(), exps=True)
        assert torch.equal(v, v2) and torch.equal(e, e2)
        assert torch.equal(fdist.gather_shards(v, len(pts)), v)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fp32", [False, True])
def test_wide_dynamic_range(fpe, fp32):
    """Coefficient scales spanning more than one common shift holds (fp64: 2^-950 .. 2^950 with random
    exponents in between; fp32: a 200-bit span) give "wide" handles, evaluated by the exponent-rescaled
    Horner (k_eval_wide): indexing exact, values within 2^-45 S (fp64) / 2^-16 S (fp32) against the oracle's
    Q_lambda and its full Horner, complex and real, including long multi-piece windows."""
    rng = np.random.default_rng(91 + fp32)
    tol = TOL32 if fp32 else TOL64
    cases = []
    if fp32:
        d = 3000
        k = np.arange(d + 1)
        a = rng.normal(size=d + 1) * np.exp2(np.round(200 * k / d - 100 + rng.normal(0, 3, d + 1)))
        cases.append(a)
        # a gentle 100-bit ramp over 40000 terms: long windows near |z| = 2^(-100/40000)
        d2 = 40000
        k2 = np.arange(d2 + 1)
        cases.append(rng.uniform(0.5, 1, d2 + 1) * np.exp2(np.floor(-60 + 160 * k2 / d2)))
    else:
        d = 2000
        a = rng.normal(size=d + 1) * np.exp2(rng.integers(-900, 900, size=d + 1).astype(float))
        a[0], a[-1] = 2.0 ** -950, 3 * 2.0 ** 950
        cases.append(a)
        d2 = 60000   # a 1900-bit ramp: slope ~ 1/32 bit per index, windows of ~10^4 terms near |z| = 2^(-1/32)
        k2 = np.arange(d2 + 1)
        cases.append(rng.uniform(0.5, 1, d2 + 1) * np.exp2(np.floor(-950 + 1900 * k2 / d2)))
    for ci, base in enumerate(cases):
        for cplx in (True, False):
            a = base * np.exp(1j * rng.uniform(0, 2 * np.pi, len(base))) if cplx else base.copy()
            n = 1500
            if ci == 0:
                r = np.exp2(rng.uniform(-3, 3, n))
            else:   # around |z| = 2^(-slope): long windows, several pieces
                sl = (160 / 40000) if fp32 else (1900 / 60000)
                r = np.exp2(-sl + rng.uniform(-sl / 8, sl / 8, n))
            pts = r * (np.exp(1j * rng.uniform(0, 2 * np.pi, n)) if cplx else rng.choice([-1.0, 1.0], n))
            if fp32:
                a, pts = workloads.to_fp32(a), workloads.to_fp32(pts)
            buf = fpe.precondition_buffer(a)
            assert fpe.header_fields(buf)["wide"] == 1
            poly = fpe.precondition(a)
            P = oracle.OraclePoly(a)
            out = gpu_eval(poly, pts)
            cls = check_indexing(P, pts, out["diag"])
            if ci == 1:
                assert np.median(cls["K"]) > 16384 if not fp32 else np.median(cls["K"]) > 5000
            err = _values_ok(P, a, pts, out, np.arange(0, n, 3), tol, cls)
            sub = np.arange(0, n, 50)
            H = P.horner_dd(pts[sub])
            e2 = rel_err_vs(H, out["v"][sub], out["e"][sub], abs_sum_log2(a, pts[sub]))
            assert np.all(e2 <= tol), e2.max()
            # the pipelined host entry point gives the same bits
            hv, he = poly.evaluate_host(pts)
            assert np.array_equal(hv, out["v"]) and np.array_equal(he, out["e"])
            print(f"\nwide {'fp32' if fp32 else 'fp64'} case {ci} {'complex' if cplx else 'real'}: "
                  f"median K {int(np.median(cls['K']))}, max err/S 2^{np.log2(max(err.max(), 1e-300)):.1f}")


@pytest.mark.parametrize("pset", ["rbar", "disk"])
def test_second_point_sets(fpe, pset):
    """points uniform on R-bar (real polynomial, the Cauchy law; eq:compAlgoRe) and on
    the unit disk (complex polynomial; rmk:case_disk) -- on the cfg2 / cfg1 families and the half-circle
    family: indexing bit-exact, values within 2^-45 S against the oracle, mean band below the paper's bound
    (1.7673 / 2.3141)."""
    d = 1000
    nn = np.arange(d + 1)
    half = np.exp2(np.sqrt((nn + 1.0) * (d + 1.0 - nn)))
    if pset == "rbar":
        cases = [(workloads.coefficients(2, d=(1 << 16) - 1), workloads.rbar_points(2, 1 << 14)),
                 (half, workloads.rbar_points(2, 1 << 14, shard=1))]
        C = 1.7673
    else:
        cases = [(workloads.coefficients(1), workloads.disk_points(1, 1 << 14)),
                 (workloads.coefficients(5, d=(1 << 16) - 1), workloads.disk_points(5, 1 << 14)),
                 (half.astype(np.complex128), workloads.disk_points(1, 1 << 14, shard=1))]
        C = 2.3141
    for a, pts in cases:
        poly = fpe.precondition(a)
        P = oracle.OraclePoly(a)
        out = gpu_eval(poly, pts)
        cls = check_indexing(P, pts, out["diag"])
        width = cls["r"] - cls["l"] + 1
        assert width.mean() < 1 + C * math.sqrt(P.d_eff * P.drop)
        _values_ok(P, a, pts, out, np.arange(0, len(pts), 4), TOL64, cls)


def test_full_horner_tensor_cores(fpe):
    """fpe_horner with complex fp64 coefficients runs on the FP64 tensor cores (k_horner_mma: every piece of
    the range, per-chunk power-of-two rescaling for |z| > 1, piece partials folded with z^16384) and sends
    points outside 2^-4 <= |z| < 2^3.99, zero and non-finite points to the vector full Horner: values
    against the oracle's full double-double Horner within 2^-45 S, complex and real points, on cfg3's
    family at d = 2^18 - 1 (16 pieces) and a polynomial with k_min > 0."""
    rng = np.random.default_rng(101)
    a = workloads.coefficients(3, d=(1 << 18) - 1)
    m = 300
    r = np.concatenate([np.exp2(rng.uniform(-4.5, 4.5, m)), np.exp2(rng.uniform(-2.0 ** -10, 2.0 ** -10, m)),
                        [2.0 ** -4, 15.87, 15.88, 16.0, 1.0, np.nextafter(2.0 ** -4, 1), np.nextafter(2.0 ** -4, 0)]])
    th = rng.uniform(0, 2 * np.pi, len(r))
    for pts in (r * np.exp(1j * th), r * np.where(rng.random(len(r)) < 0.5, -1.0, 1.0)):
        for coef in (a, np.concatenate([np.zeros(777, np.complex128), a[: (1 << 17)]])):
            poly = fpe.precondition(coef)
            P = oracle.OraclePoly(coef)
            out = gpu_eval(poly, pts, horner=True)
            H = P.horner_dd(pts)
            err = rel_err_vs(H, out["v"], out["e"], abs_sum_log2(coef, pts))
            r2 = np.abs(pts) ** 2
            tc = (r2 >= 2.0 ** -8) & (r2 < 252.0)   # tensor-core path (2^-4 <= |z| < 2^3.99): pieces of 16384
            assert np.all(err[tc] <= TOL64), (err[tc].max(), pts[tc][np.argmax(err[tc])])
            # the others take one plain Horner pass over all 2^18 coefficients, whose rounding error grows
            # like sqrt(d) u (gamma_2d S in the worst case): 2^-40 S
            assert np.all(err[~tc] <= 2.0 ** -40), err[~tc].max()
    z0 = gpu_eval(fpe.precondition(a), np.array([0j, complex(np.nan, 0)]), horner=True)
    assert z0["v"][0] * 2.0 ** z0["e"][0] == a[0] and np.isnan(z0["v"][1].real)
