"""CPU checks of the library's host/device math (fpe_math.cuh, fpe_polar.cuh), compiled as
host code by tests/native/devmath_host.cu.

* lambda_fast (quick table-driven log2 + Ziv test, fallback lambda_cr) must equal the
  oracle's correctly rounded lambda bit for bit (G4);
* log2abs_quick / atan2_turns accuracy against mpmath;
* lambda_enclosure (the classifier's fast path: every window decision is taken on an fp64 enclosure
  [lo, hi] of log2|z| and must equal the decision at the correctly rounded lambda, so the enclosure
  must contain it) on 10^6 adversarial points against the oracle's correctly rounded lambda;
* the work bucketing (eval_tiled.cu): every point's correctly rounded lambda lies inside its bucket's range
  of lambda estimates widened by 2^-44 (1 + |lambda|) -- the range k_bucket_windows classifies at both ends to
  bound the windows of the bucket's points -- at every bucket count; the key is monotone in lambda;
* z^n by the polar route (the library's z^l) within 2^-50 + n 2^-76
  relative of mpmath at 200 bits (2^-49.6 at n = 2^24, the largest degree of the configs).
"""
import ctypes as C
import math
import os
import subprocess

import mpmath as mp
import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "native", "devmath_host.cu")
SO = os.path.join(HERE, "native", "libdevmath_host.so")
DEPS = [SRC] + [os.path.join(HERE, "..", "paper_2211_06320_b200", "csrc", f)
                for f in ("fpe_math.cuh", "fpe_polar.cuh", "fpe_hd.cuh", "log_table.h")]


@pytest.fixture(scope="module")
def dm():
    if not os.path.exists(SO) or any(os.path.getmtime(d) > os.path.getmtime(SO) for d in DEPS):
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-O2", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
                        "-shared", "-o", SO, SRC], check=True)
    L = C.CDLL(SO)
    P = C.c_void_p
    for f in ("dm_lambda_fast", "dm_lambda_cr", "dm_log2abs"):
        getattr(L, f).argtypes = [P, C.c_longlong, C.c_int, P] + ([P] if f != "dm_log2abs" else [])
    L.dm_atan2_turns.argtypes = [P, C.c_longlong, P]
    L.dm_pow_polar.argtypes = [P, P, C.c_longlong, C.c_int, P, P]
    L.dm_lambda_enclosure.argtypes = [P, C.c_longlong, C.c_int, P]
    L.dm_bucket_key.argtypes = [P, C.c_longlong, C.c_int, P]
    L.dm_bucket_estimates.argtypes = [P, C.c_longlong, C.c_int, P]
    return L


def _xy(z):
    z = np.asarray(z, dtype=np.complex128)
    return np.ascontiguousarray(np.stack([z.real, z.imag], 1)), len(z)


def _points(rng, n):
    zs = [complex(*rng.normal(size=2)) * 2.0 ** rng.integers(-80, 80) for _ in range(n)]
    for _ in range(n):
        t = rng.uniform(0, 2 * math.pi)
        eps = 2.0 ** -rng.integers(1, 62) * rng.choice([-1, 1])
        zs.append(complex(math.cos(t), math.sin(t)) * (1 + eps))
    for _ in range(n // 4):   # near the axes and the diagonal, tiny / huge moduli
        a = 2.0 ** rng.uniform(-1070, 1020)
        zs += [complex(a, a * 2.0 ** -rng.integers(1, 80)), complex(a * 2.0 ** -rng.integers(1, 80), -a),
               complex(-a, a * (1 + 2.0 ** -rng.integers(1, 50)))]
    zs += [complex(1.0, 2.0 ** -30), complex(1.0, 1e-200), complex(1 - 2 ** -53, 2 ** -26), complex(0.6, 0.8),
           complex(math.nextafter(1.0, 2.0), 0.0), complex(math.nextafter(1.0, 0.0), 0.0), complex(2.0 ** -1074, 0),
           complex(1e308, 1e308), complex(-3.0, 4.0), complex(5e-324, 5e-324)]
    return np.array(zs)


def test_lambda_fast_equals_oracle_cr(dm):
    rng = np.random.default_rng(5)
    z = _points(rng, 20000)
    for cplx in (1, 0):
        zz = z if cplx else z.real.astype(np.complex128)
        zz = zz[zz != 0]
        xy, n = _xy(zz)
        lam = np.empty(n); hard = np.zeros(n, np.int32)
        dm.dm_lambda_fast(xy.ctypes.data, n, cplx, lam.ctypes.data, hard.ctypes.data)
        ref = np.array([oracle.lam(complex(v) if cplx else float(v.real))[0] for v in zz])
        assert np.array_equal(lam, ref), np.flatnonzero(lam != ref)[:5]
        assert hard.sum() == 0


def test_log2abs_quick_accuracy(dm):
    mp.mp.prec = 200
    rng = np.random.default_rng(6)
    z = _points(rng, 1500)
    xy, n = _xy(z)
    hl = np.empty(2 * n)
    dm.dm_log2abs(xy.ctypes.data, n, 1, hl.ctypes.data)
    worst = 0.0
    for i, v in enumerate(z):
        ref = mp.log(mp.sqrt(mp.mpf(v.real) ** 2 + mp.mpf(v.imag) ** 2), 2)
        # the bound lambda_fast's Ziv test relies on: 2^-80 relative + 2^-102 absolute
        err = abs(mp.mpf(hl[2 * i]) + mp.mpf(hl[2 * i + 1]) - ref) / (abs(ref) * mp.mpf(2) ** -80 + mp.mpf(2) ** -102)
        worst = max(worst, float(err))
    assert worst < 2.0 ** -6, math.log2(worst)


def test_atan2_turns_accuracy(dm):
    mp.mp.prec = 200
    rng = np.random.default_rng(7)
    z = _points(rng, 1500)
    z = np.concatenate([z, [1, -1, 1j, -1j, 1 + 1j, -1 - 1j, complex(1, -0.0), complex(-1, 0.0)]])
    xy, n = _xy(z)
    hl = np.empty(2 * n)
    dm.dm_atan2_turns(xy.ctypes.data, n, hl.ctypes.data)
    worst = 0.0
    for i, v in enumerate(z):
        ref = mp.atan2(mp.mpf(v.imag), mp.mpf(v.real)) / (2 * mp.pi)
        err = abs(mp.mpf(hl[2 * i]) + mp.mpf(hl[2 * i + 1]) - ref)
        worst = max(worst, float(err))
    assert worst < 2.0 ** -78, math.log2(worst)   # n tau error < 2^-51 for n <= 2^24


@pytest.mark.parametrize("cplx", [1, 0])
def test_pow_polar_accuracy(dm, cplx):
    mp.mp.prec = 200
    rng = np.random.default_rng(8 + cplx)
    m = 600
    r = np.exp2(rng.uniform(-3, 3, m)) * np.where(rng.random(m) < 0.3, 1 + 2.0 ** -rng.integers(10, 40, m), 1.0)
    z = r * np.exp(1j * rng.uniform(-math.pi, math.pi, m))
    if not cplx:
        z = (z.real + 0j)
    e = rng.integers(0, 31, m)
    p = (2.0 ** e * rng.uniform(1, 2, m)).astype(np.int64)
    p[:20] = np.arange(20)
    p = np.clip(p, 0, 2 ** 31 - 1)
    xy, n = _xy(z)
    out = np.empty(2 * n); E = np.empty(n, np.int64)
    dm.dm_pow_polar(xy.ctypes.data, p.ctypes.data, n, cplx, out.ctypes.data, E.ctypes.data)
    worst = 0.0
    for i in range(n):
        zz = mp.mpc(z[i].real, z[i].imag) if cplx else mp.mpf(z[i].real)
        ref = zz ** int(p[i])
        got = mp.mpc(out[2 * i], out[2 * i + 1]) * mp.mpf(2) ** int(E[i])
        # exp2 / sincospi rounding plus n times the 2^-78 accuracy of lambda and tau
        err = abs(got - ref) / abs(ref) / (2.0 ** -50 + float(p[i]) * 2.0 ** -76)
        worst = max(worst, float(err))
    assert worst < 1.0, worst


def _adversarial(rng, n):
    """Points where log2|z| is hardest to bracket: |z| within 2^-1..2^-62 of a power of two (any binade,
    incl. 1), subnormal and near-overflow moduli, near the axes and the diagonal, and random moduli."""
    q = n // 6
    k = rng.integers(-1070, 1020, q).astype(float)
    eps = rng.choice([-1.0, 1.0], q) * np.exp2(-rng.integers(1, 63, q).astype(float))
    near_pow2 = np.exp2(k) * (1 + eps)
    near_one = 1 + rng.choice([-1.0, 1.0], q) * np.exp2(-rng.uniform(1, 62, q))
    sub = rng.integers(1, 1 << 40, q).astype(float) * 2.0 ** -1074
    big = np.exp2(rng.choice([-1.0, 1.0], q) * 1000 + rng.uniform(-40, 23, q))
    rnd = np.exp2(rng.uniform(-1074, 1023, q))
    mods = np.concatenate([near_pow2, near_one, sub, big, rnd])
    th = rng.uniform(0, 2 * np.pi, len(mods))
    z = mods * np.exp(1j * th)
    m = len(mods)
    # axes and diagonal: one coordinate tiny relative to the other, or |x| = |y| (1 + tiny)
    a = np.exp2(rng.uniform(-1070, 1020, q))
    axis = a + 1j * a * np.exp2(-rng.integers(1, 80, q).astype(float)) * rng.choice([-1, 1], q)
    diag = a * (1 + 1j * (1 + rng.choice([-1, 1], q) * np.exp2(-rng.integers(1, 60, q).astype(float))))
    z = np.concatenate([z, axis, diag])
    z = z[np.isfinite(z) & (z != 0)]
    return z, mods[np.isfinite(mods) & (mods > 0)] * rng.choice([-1.0, 1.0], int(np.sum(np.isfinite(mods) & (mods > 0))))


def test_lambda_enclosure_contains_rounded_lambda(dm):
    rng = np.random.default_rng(17)
    zc, xr = _adversarial(rng, 1_000_000)
    for pts, cplx in ((zc, 1), (xr, 0)):
        xy, n = _xy(pts if cplx else pts.astype(np.complex128))
        lmh = np.empty(3 * n)
        dm.dm_lambda_enclosure(xy.ctypes.data, n, cplx, lmh.ctypes.data)
        lo, hi, mid = lmh[0::3], lmh[1::3], lmh[2::3]
        P = oracle.OraclePoly(np.array([1.0, 1.0]))
        lam = P.classify(pts)["lam"]          # correctly rounded log2|z| (binary128, G4)
        bad = ~((lo <= lam) & (lam <= hi))
        assert not bad.any(), (int(bad.sum()), pts[bad][:3], lam[bad][:3], lo[bad][:3], hi[bad][:3])
        # the error the enclosure is built on (fpe_math.cuh): |mid - log2|z|| < 2^-50 + 2^-53 |lambda| (+ ulp)
        err = np.abs(mid - lam) / (2.0 ** -50 + 2.0 ** -52 * np.abs(lam))
        assert err.max() < 1.0, err.max()
        assert n > 700_000 if cplx else n > 500_000


def test_bucket_key_ranges_contain_lambda(dm):
    """k_plan bounds a group's union window by [l at the low end, r at the high end] of its buckets' lambda
    ranges (k_bucket_windows); that is a valid bound only if every point's correctly rounded lambda lies in
    its bucket's range of estimates widened by eps = 2^-44 (1 + |lambda|) -- checked here on 2 * 10^6
    adversarial points at bucket counts 2^10 .. 2^15 -- and the key must be monotone in lambda (points
    whose lambdas differ by more than the estimate's error are ordered by their keys)."""
    rng = np.random.default_rng(29)
    zc, xr = _adversarial(rng, 1_000_000)
    P = oracle.OraclePoly(np.array([1.0, 1.0]))
    for pts, cplx in ((zc, 1), (xr, 0)):
        xy, n = _xy(pts if cplx else pts.astype(np.complex128))
        key = np.empty(n, np.uint32)
        dm.dm_bucket_key(xy.ctypes.data, n, cplx, key.ctypes.data)
        lam = P.classify(pts)["lam"]
        assert np.all(key > 0) and np.all(key < 2 ** 23)
        for cb in (10, 12, 15):
            b = np.ascontiguousarray(key >> (23 - cb))
            lohi = np.empty(2 * n)
            dm.dm_bucket_estimates(b.ctypes.data, n, cb, lohi.ctypes.data)
            lo, hi = lohi[0::2], lohi[1::2]
            la = lo - 2.0 ** -44 * (1 + np.abs(lo))
            lb = hi + 2.0 ** -44 * (1 + np.abs(hi))
            bad = ~((la <= lam) & (lam <= lb))
            assert not bad.any(), (cb, int(bad.sum()), lam[bad][:3], lo[bad][:3], hi[bad][:3])
            assert np.all(lo <= hi)
        o = np.argsort(lam, kind="stable")
        ls, ks = lam[o], key[o].astype(np.int64)
        # for lambdas more than the estimate error apart, the keys do not decrease
        sep = np.diff(ls) > 2.0 ** -48 * (1 + np.abs(ls[1:]))
        run_max = np.maximum.accumulate(ks)
        assert np.all(ks[1:][sep] >= run_max[:-1][sep]), "key not monotone in lambda"
