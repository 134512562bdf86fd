"""Pins for the oracle's evaluation phase: lambda, k_lambda / N / [l, r], Q_lambda.

Expected values: the paper's worked example (tests/golden/worked_example.json),
mpmath at 300 bits, exact-rational linear scans (tests/brute.py), closed
forms ((z-1)^d, geometric series, Chebyshev T_n(cos x) = cos(n x), monomials,
1 + z), and the paper's theorems (truncation bound T3, kept-term averages T1,
worst case T2).
"""
import math

import mpmath as mp
import numpy as np
import pytest

import oracle
import workloads
from brute import classify_brute

mp.mp.prec = 300


def mp_round_lambda(z) -> float:
    v = mp.log(abs(mp.mpc(z.real, z.imag)), 2)
    return float(v)   # mpmath rounds to nearest on conversion


# ---------------------------------------------------------------- lambda ---

def test_lambda_exact_powers_of_two():
    for n in range(-1074, 1024, 13):
        assert oracle.lam(math.ldexp(1.0, n)) == (float(n), 0)
        assert oracle.lam(complex(0, math.ldexp(-1.0, n))) == (float(n), 0)
    # |z|^2 = 2^(2n+1): lambda = n + 1/2 exactly
    for n in range(-500, 500, 7):
        z = complex(math.ldexp(1.0, n), math.ldexp(1.0, n))
        assert oracle.lam(z) == (n + 0.5, 0)
    assert oracle.lam(0j)[0] == -math.inf
    assert math.isnan(oracle.lam(complex(math.nan, 0))[0])


def test_lambda_vs_mpmath():
    rng = np.random.default_rng(11)
    zs = []
    for _ in range(3000):
        zs.append(complex(*rng.normal(size=2)) * 2.0 ** rng.integers(-60, 60))
    # near |z| = 1 (log1p path) -- relative accuracy matters, SURVEY G4
    for _ in range(1500):
        t = rng.uniform(0, 2 * math.pi)
        eps = 2.0 ** -rng.integers(1, 60) * rng.choice([-1, 1])
        zs.append(complex(math.cos(t), math.sin(t)) * (1 + eps))
    zs += [complex(1.0, 2.0 ** -30), complex(1.0, 1e-200), complex(1 - 2 ** -53, 2 ** -26),
           complex(math.nextafter(1.0, 2.0), 0.0), complex(math.nextafter(1.0, 0.0), 0.0)]
    for z in zs:
        l, hard = oracle.lam(z)
        assert hard == 0
        assert l == mp_round_lambda(z), z
    # real points
    for _ in range(2000):
        x = float(rng.choice([-1, 1]) * 2.0 ** rng.uniform(-8, 8))
        l, hard = oracle.lam(x)
        assert hard == 0 and l == mp_round_lambda(complex(x, 0)), x


# ------------------------------------------------------------- searches ---

def _example_poly(worked, drop=None):
    s = np.array(worked["scales"], dtype=np.int32)
    a = np.ldexp(1.0, s - 1).astype(np.complex128)
    return oracle.OraclePoly(a, p=6, drop=drop)


def test_classify_worked_example(worked):
    exp = worked["derived_not_printed"]
    pts = np.array([1.0 + 0j, 0.125 + 0j])   # lambda = 0 and lambda = -3
    for drop, tag in ((6, "drop6"), (None, "drop13")):
        P = _example_poly(worked, drop)
        c = P.classify(pts)
        assert c["lam"].tolist() == [0.0, -3.0]
        # k_lambda: at lambda=0 the argmax is {8, 9} -> smallest, k=8;
        # at lambda=-3 it is k=6
        assert P.hk[c["istar"]].tolist() == [8, worked["k_lambda_m3"]]
        band = exp["band_" + tag]
        assert [int(c["l"][0]), int(c["r"][0])] == band["lambda0"]
        assert [int(c["l"][1]), int(c["r"][1])] == band["lambda_m3"]
        W = [sorted(k for k in range(int(c["l"][i]), int(c["r"][i]) + 1) if P.good[k]) for i in range(2)]
        assert W[0] == exp["W_" + tag]["lambda0"] and W[1] == exp["W_" + tag]["lambda_m3"]
        assert c["K"].tolist() == [len(W[0]), len(W[1])]
    # the paper's own kept sets: Q_0 exactly, Q_{-3} as a subset
    P = _example_poly(worked, 6)
    c = P.classify(pts)
    W0 = [k for k in range(c["l"][0], c["r"][0] + 1) if P.good[k]]
    Wm3 = [k for k in range(c["l"][1], c["r"][1] + 1) if P.good[k]]
    assert W0 == worked["Q0_indices_paper"]
    assert set(worked["Qm3_indices_paper"]) <= set(Wm3)
    # N_lambda values printed in the paper: 30 at lambda=0, 9 at lambda=-3
    for lam, N in ((0.0, worked["N_lambda0"]), (-3.0, worked["N_lambda_m3"])):
        i, l, r, Nb = classify_brute(P.hk, P.hh, 6, lam)
        assert Nb == N


def test_classify_vs_linear_scan():
    rng = np.random.default_rng(12)
    for trial in range(300):
        d = int(rng.integers(1, 48))
        s = rng.integers(-40, 40, size=d + 1)
        zero = rng.random(d + 1) < 0.1
        a = np.where(zero, 0.0, np.ldexp(1.0, s)).astype(np.float64)
        if np.count_nonzero(a) == 0:
            a[0] = 1.0
        drop = int(rng.integers(1, 30))
        P = oracle.OraclePoly(a, p=53, drop=drop)
        # lambdas: random, hull slopes exactly (ties), +-1 ulp around them, extremes
        lams = list(rng.uniform(-50, 50, size=8))
        dk = np.diff(P.hk); dh = np.diff(P.hh)
        for j in range(len(dk)):
            sl = -dh[j] / dk[j]
            lams.append(float(sl))   # exact when dk is a power of two: ties
            lams += [math.nextafter(float(sl), math.inf), math.nextafter(float(sl), -math.inf)]
        lams += [0.0, 1e-300, -1e-300, 5e-324, 1000.0, -1000.0, 2.0 ** -40, -(2.0 ** -40)]
        ist, l, r = P.search(np.array(lams))
        for q, lam in enumerate(lams):
            i, lb, rb, _ = classify_brute(P.hk, P.hh, drop, lam)
            assert (int(ist[q]), int(l[q]), int(r[q])) == (i, lb, rb), (lam, i, lb, rb)
        # non-integer lambdas through actual points
        xs = np.ldexp(rng.uniform(0.5, 1.0, size=12), rng.integers(-40, 40, size=12))
        c = P.classify(xs)
        for q, x in enumerate(xs):
            i, l, r, _ = classify_brute(P.hk, P.hh, drop, float(c["lam"][q]))
            assert (int(c["istar"][q]), int(c["l"][q]), int(c["r"][q])) == (i, l, r)


def test_classify_special_points():
    a = workloads.coefficients(1, d=63)
    P = oracle.OraclePoly(a)
    c = P.classify(np.array([0j, complex(math.inf, 0), complex(math.nan, 1)]))
    assert c["istar"].tolist() == [0, -1, -1]
    assert c["l"][0] == P.k_min and c["r"][0] == P.k_min


# ---------------------------------------------------------------- values ---

def _to_mpc(x: oracle.oracle.XVal, i):
    return (mp.mpc(x.hi[i].real, x.hi[i].imag) + mp.mpc(x.lo[i].real, x.lo[i].imag)) * mp.mpf(2) ** int(x.e[i])


def _S(P, z):
    return sum(abs(mp.mpc(complex(c))) * abs(mp.mpc(complex(z))) ** k for k, c in enumerate(P.coeffs))


@pytest.mark.parametrize("method,tol", [("horner", 2.0 ** -100), ("horner_dd", 2.0 ** -90)])
def test_values_closed_forms(method, tol):
    """P_ref (binary128 Horner, and the double-double Horner used at full size) against closed forms."""
    tol = mp.mpf(tol)
    rng = np.random.default_rng(13)
    zs = [complex(*rng.normal(size=2)) * 2.0 ** rng.integers(-3, 3) for _ in range(12)] + [1j, -1.0, 2.0, 0.5j]
    # geometric series sum_{k<=d} z^k = (z^(d+1) - 1)/(z - 1), exact coefficients
    for d in (1, 7, 100, 513):
        P = oracle.OraclePoly(np.ones(d + 1, dtype=np.complex128))
        H = getattr(P, method)(np.array(zs))
        for i, z in enumerate(zs):
            zz = mp.mpc(z.real, z.imag)
            ref = (zz ** (d + 1) - 1) / (zz - 1) if z != 1 else mp.mpf(d + 1)
            S = sum(abs(zz) ** k for k in range(d + 1))
            assert abs(_to_mpc(H, i) - ref) <= tol * S
    # (z - 1)^d with binomial coefficients rounded to fp64 (error <= 2^-53 S)
    for d in (5, 60, 300, 1023):
        c = np.array([float(mp.binomial(d, k)) * (-1) ** (d - k) for k in range(d + 1)])
        P = oracle.OraclePoly(c.astype(np.complex128))
        H = getattr(P, method)(np.array(zs))
        for i, z in enumerate(zs):
            zz = mp.mpc(z.real, z.imag)
            S = (1 + abs(zz)) ** d
            assert abs(_to_mpc(H, i) - (zz - 1) ** d) <= (mp.mpf(2) ** -53 + tol) * S
    # Chebyshev T_n(cos x) = cos(n x), integer coefficients exact in fp64 (n <= 40)
    for n in (3, 17, 40):
        T = [mp.mpf(0)] * (n + 1)
        t0, t1 = [1], [0, 1]
        for _ in range(n - 1):
            t2 = [0] + t1
            t2 = [2 * v for v in t2]
            for k, v in enumerate(t0):
                t2[k] -= v
            t0, t1 = t1, t2
        coef = np.array(t1 if n >= 1 else t0, dtype=np.float64)
        P = oracle.OraclePoly(coef)
        xs = np.cos(rng.uniform(0, math.pi, size=20))
        H = getattr(P, method)(xs)
        for i, x in enumerate(xs):
            ref = mp.cos(n * mp.acos(mp.mpf(x)))
            assert abs(_to_mpc(H, i).real - ref) <= mp.mpf(2) ** -95 * sum(abs(v) for v in coef)
    # monomial a z^n and 1 + z
    P = oracle.OraclePoly(np.array([0] * 1000 + [0.75 - 0.5j]))
    H = getattr(P, method)(np.array([1.5 + 0.25j]))
    ref = mp.mpc(0.75, -0.5) * mp.mpc(1.5, 0.25) ** 1000
    assert abs(_to_mpc(H, 0) - ref) <= tol * abs(ref)


def test_horner_vs_mpmath_bruteforce():
    """Both full-Horner references and the direct sum against mpmath at 300 bits (d <= 32)."""
    rng = np.random.default_rng(14)
    for _ in range(60):
        d = int(rng.integers(1, 33))
        a = (rng.uniform(-1, 1, d + 1) + 1j * rng.uniform(-1, 1, d + 1)) * 2.0 ** rng.integers(-20, 20, d + 1)
        P = oracle.OraclePoly(a)
        zs = np.array([complex(*rng.normal(size=2)) * 2.0 ** rng.integers(-6, 6) for _ in range(4)])
        H = P.horner(zs)
        H2 = P.horner_dd(zs)
        D = P.direct_sum(zs)
        for i, z in enumerate(zs):
            zz = mp.mpc(z.real, z.imag)
            ref = sum(mp.mpc(c.real, c.imag) * zz ** k for k, c in enumerate(a))
            S = _S(P, z)
            assert abs(_to_mpc(H, i) - ref) <= mp.mpf(2) ** -100 * S
            assert abs(_to_mpc(H2, i) - ref) <= mp.mpf(2) ** -98 * S
            assert abs(_to_mpc(D, i) - ref) <= mp.mpf(2) ** -100 * S
    # real polynomial at real points, zeros at both ends (k_min > 0), huge and tiny |z| (exponent counter)
    a = np.array([0.0, 0.0, 3.0, -1.5, 0.0, 2.0 ** -600, 7.0, 0.0])
    P = oracle.OraclePoly(a)
    xs = np.array([0.75, -2.0 ** 300, 2.0 ** -400, -1.25])
    H2 = P.horner_dd(xs)
    for i, x in enumerate(xs):
        ref = sum(mp.mpf(c) * mp.mpf(x) ** k for k, c in enumerate(a))
        S = sum(abs(mp.mpf(c)) * abs(mp.mpf(x)) ** k for k, c in enumerate(a))
        assert abs(_to_mpc(H2, i) - ref) <= mp.mpf(2) ** -98 * S


def test_abs_sum():
    rng = np.random.default_rng(15)
    a = rng.normal(size=50) + 1j * rng.normal(size=50)
    P = oracle.OraclePoly(a)
    zs = np.array([0.3 + 0.4j, 2.0 - 1j, -7j])
    m, e = P.abs_sum(zs)
    for i, z in enumerate(zs):
        ref = _S(P, z)
        assert abs(mp.mpf(m[i]) * mp.mpf(2) ** int(e[i]) - ref) <= mp.mpf(2) ** -50 * ref


def test_log2_maxterm_vs_mpmath_and_cover():
    """M(z) = max_k |a_k z^k| (eq:def_prec_loss), which scales the T3 self-check and the confidence test:
    (1) against mpmath at 300 bits on random polynomials with zeros, ties and a wide dynamic range;
    (2) against the cover: log2|a_k| lies in [s_k - 1, s_k) (eq:sigma), so log2 M lies in [N - 1, N) with
    N = hh_i* + lambda hk_i* the sheared cover's top (eq:defN) -- a dropped or shifted
    term, a wrong sign of k lambda or an index off by one in or_log2_maxterm fails one of them."""
    rng = np.random.default_rng(19)
    for fam in range(8):
        d = int(rng.integers(5, 60))
        a = rng.normal(size=d + 1) * np.exp2(rng.integers(-40, 40, d + 1).astype(float))
        if fam % 2:
            a = a * np.exp(1j * rng.uniform(0, 2 * np.pi, d + 1))
        a[rng.random(d + 1) < 0.2] = 0
        a[-1] = a[-1] or 3.0
        P = oracle.OraclePoly(a)
        r = np.exp2(rng.uniform(-6, 6, 40))
        pts = r * np.exp(1j * rng.uniform(0, 2 * np.pi, 40)) if fam % 2 else r * rng.choice([-1.0, 1.0], 40)
        got = P.log2_maxterm(pts)
        for i, z in enumerate(pts):
            zz = mp.mpc(complex(z).real, complex(z).imag)
            ref = max(mp.log(abs(mp.mpc(complex(c).real, complex(c).imag)) * abs(zz) ** k, 2)
                      for k, c in enumerate(a) if c != 0)
            assert abs(got[i] - float(ref)) <= 2.0 ** -40 * max(1.0, abs(float(ref))), (fam, i)
        c = P.classify(pts)
        N = P.hh[c["istar"]] + c["lam"] * P.hk[c["istar"]]
        assert np.all(got >= N - 1 - 1e-9) and np.all(got < N + 1e-9)
    # cfg1 and cfg3 samples: the cover bound at full degree
    for cfg in (1, 3):
        a = workloads.coefficients(cfg) if cfg == 1 else workloads.coefficients(3, d=(1 << 14) - 1)
        P = oracle.OraclePoly(a)
        pts = workloads.points(cfg, 300, shard=2)
        got = P.log2_maxterm(pts)
        c = P.classify(pts)
        N = P.hh[c["istar"]] + c["lam"] * P.hk[c["istar"]]
        assert np.all(got >= N - 1 - 1e-6) and np.all(got < N + 1e-6)
    # a monomial a z^k: log2 M = log2|a| + k log2|z| exactly
    P = oracle.OraclePoly(np.array([0.0] * 7 + [5.0]))
    assert np.allclose(P.log2_maxterm(np.array([2.0, 0.5, 3.0])), [math.log2(5) + 7, math.log2(5) - 7,
                                                                  math.log2(5) + 7 * math.log2(3)], rtol=0, atol=1e-12)


def _truncation_check(P, pts, slack=2.0 ** -20):
    """T3 (eq:target / equ:err), normalised:
    |P(z) - Q_lambda(z)| < 2^(-p-2) max_j |a_j z^j|."""
    c = P.classify(pts)
    Q = P.fpe_eval(pts, c)
    H = P.horner(pts)
    l2M = P.log2_maxterm(pts)
    ok = c["l"] >= 0
    e_ref = np.round(l2M).astype(np.int64)
    diff = np.abs(H.scaled(e_ref) - Q.scaled(e_ref))
    bound = np.exp2(l2M - e_ref) * 2.0 ** (-P.p - 2) * (1 + slack)
    assert np.all(diff[ok] < bound[ok]), np.max(diff[ok] / bound[ok])
    return c


def test_truncation_theorem_cfg1_sample():
    a = workloads.coefficients(1)
    P = oracle.OraclePoly(a)
    assert P.drop == 66
    pts = workloads.points(1, 4096)
    c = _truncation_check(P, pts)
    # T2 worst case: K <= d_eff + 1 ; T1 average over the sphere: mean #[l,r] < 1 + 1.9046 sqrt(d D)
    width = c["r"] - c["l"] + 1
    assert np.all(c["K"] <= P.d_eff + 1)
    assert width.mean() < 1 + 1.9046 * math.sqrt(P.d_eff * P.drop)
    assert np.all(c["hard"] == 0)


def test_truncation_theorem_random_families():
    rng = np.random.default_rng(16)
    for fam in range(12):
        d = int(rng.integers(30, 400))
        k = np.arange(d + 1)
        prof = rng.choice([0, 30, 120]) * np.sin(np.pi * k / d) + rng.normal(0, rng.choice([0.5, 4]), d + 1)
        a = np.exp2(prof) * np.exp(1j * rng.uniform(0, 2 * np.pi, d + 1))
        a[rng.random(d + 1) < 0.05] = 0
        a[0] = a[0] or 1.0
        for p in (24, 53):
            P = oracle.OraclePoly(a, p=p)
            pts = workloads.sphere_points(1, 300) * (1 + 1e-3 * fam)
            _truncation_check(P, pts)


def test_fpe_eval_worked_example_structure(worked):
    # P(z) with the example's scales, evaluated on |z|=1 and |z|=1/8: Q equals the sum over W exactly
    P = _example_poly(worked, 6)
    zs = np.array([np.exp(0.7j), 0.125 * np.exp(-2.1j)])
    c = P.classify(zs)
    Q = P.fpe_eval(zs, c)
    for i, z in enumerate(zs):
        zz = mp.mpc(z.real, z.imag)
        W = [k for k in range(c["l"][i], c["r"][i] + 1) if P.good[k]]
        ref = sum(mp.mpc(P.coeffs[k].real, P.coeffs[k].imag) * zz ** k for k in W)
        assert abs(_to_mpc(Q, i) - ref) <= mp.mpf(2) ** -100 * abs(ref)


def test_half_circle_family_complexity():
    """The half-circle family (eq:halfcirclepoly), a_n = 2^sqrt((n+1)(d+1-n)), nearly
    saturates the complexity bound: on the Riemann sphere the mean band width / sqrt(d (p + s(d) + 3))
    stays below Theorem thm:equivAlgo's 1.9046 and approaches C_3(0) = 1.32178 from below as d
    grows (C_3(delta) increases to C_3(0) as delta -> 0)."""
    ratios = []
    for d in (250, 1000, 2000):
        n = np.arange(d + 1)
        a = np.exp2(np.sqrt((n + 1.0) * (d + 1.0 - n))).astype(np.complex128)
        P = oracle.OraclePoly(a)
        c = P.classify(workloads.sphere_points(1, 60000, shard=9))
        ratios.append((c["r"] - c["l"] + 1).mean() / math.sqrt(P.d_eff * P.drop))
    assert all(r < 1.9046 for r in ratios)
    assert ratios[0] < ratios[1] < ratios[2] < 1.32178
    assert ratios[2] > 1.25


def test_second_point_sets_average_window():
    """Theorem thm:algo / eq:compAlgoRe and remark rmk:case_disk: the mean
    band width #[l, r] is below 1 + C sqrt(d_eff D) with C = 1.7673 for a real polynomial at points uniform on
    R-bar (the Cauchy law) and C = 2.3141 for a complex polynomial at points uniform on the unit disk --
    for any polynomial, so also for the half-circle family (the paper's slowest)."""
    import workloads
    d = 1000
    nn = np.arange(d + 1)
    half = np.exp2(np.sqrt((nn + 1.0) * (d + 1.0 - nn)))
    for a, pts, C in (
            (workloads.coefficients(2, d=4095), workloads.rbar_points(2, 1 << 15), 1.7673),
            (half, workloads.rbar_points(2, 1 << 15, shard=1), 1.7673),
            (workloads.coefficients(1), workloads.disk_points(1, 1 << 15), 2.3141),
            (half.astype(np.complex128), workloads.disk_points(1, 1 << 15, shard=1), 2.3141)):
        P = oracle.OraclePoly(a)
        c = P.classify(pts)
        width = (c["r"] - c["l"] + 1).astype(float)
        bound = 1 + C * math.sqrt(P.d_eff * P.drop)
        assert width.mean() < bound, (width.mean(), bound)
        assert np.all(c["K"] <= width)
    # the generators' laws: Cauchy quartiles at +-1, disk radii with P(r < 1/2) = 1/4
    x = workloads.rbar_points(3, 1 << 16)
    assert abs(np.mean(np.abs(x) < 1) - 0.5) < 0.01
    z = workloads.disk_points(3, 1 << 16)
    assert np.all(np.abs(z) < 1) and abs(np.mean(np.abs(z) < 0.5) - 0.25) < 0.01
