"""Pins for the oracle's preconditioning steps (scales, cover, G_p).

Every expected value here comes from the paper's printed example, a closed
form, or the brute-force definitions in tests/brute.py -- never from the
oracle itself.
"""
import math

import numpy as np
import pytest

import oracle
from brute import good_brute, hull_brute, scale_exact

NEG = oracle.NEG_INF_SCALE


# ---------------------------------------------------------------- scales ---

def test_scale_paper_examples():
    # "s(3+2i)=2=s(3) and s(3+3i)=3=s(3)+1"
    assert oracle.scale(3 + 2j) == 2
    assert oracle.scale(3.0) == 2
    assert oracle.scale(3 + 3j) == 3
    assert oracle.scale(0.0) == NEG and oracle.scale(0j) == NEG   # s(0) = -inf


def test_scale_boundaries():
    # |a| = 2^n gives n+1 (eq:sigma with equality on the left); smallest subnormal
    for n in range(-1074, 1024, 37):
        assert oracle.scale(math.ldexp(1.0, n)) == n + 1
        assert oracle.scale(complex(0.0, -math.ldexp(1.0, n))) == n + 1
    assert oracle.scale(5e-324) == -1073
    # exact s = 0 where hypot() rounds to 1
    x = 1.0 - 2.0 ** -53
    y = 2.0 ** -26 * (1.0 - 2.0 ** -52)
    assert scale_exact(x, y) == 0
    assert oracle.scale(complex(x, y)) == 0


def test_scale_random_vs_fraction():
    rng = np.random.default_rng(1)
    for _ in range(3000):
        e1, e2 = rng.integers(-1070, 1020, size=2)
        re = math.ldexp(rng.uniform(-1, 1), int(e1))
        im = math.ldexp(rng.uniform(-1, 1), int(e2 if rng.random() < 0.5 else e1))
        assert oracle.scale(complex(re, im)) == scale_exact(re, im)
        assert oracle.scale(re) == scale_exact(re)
    # near |z| = 2^n boundaries: x^2 + y^2 straddling 4^n
    for _ in range(2000):
        t = rng.uniform(0, math.pi / 2)
        n = int(rng.integers(-50, 50))
        re, im = math.ldexp(math.cos(t), n), math.ldexp(math.sin(t), n)
        for dre in (-1, 0, 1):
            r2 = np.nextafter(re, np.inf) if dre > 0 else (np.nextafter(re, -np.inf) if dre < 0 else re)
            assert oracle.scale(complex(r2, im)) == scale_exact(r2, im)


def test_scale_lemma_invariants():
    # s(zz') - s(z) - s(z') in {-1, 0}; s(z +- z') <= max + 1
    rng = np.random.default_rng(2)
    for _ in range(2000):
        z = complex(*rng.normal(size=2)) * 2.0 ** rng.integers(-30, 30)
        w = complex(*rng.normal(size=2)) * 2.0 ** rng.integers(-30, 30)
        sz, sw = oracle.scale(z), oracle.scale(w)
        assert oracle.scale(z * w) - sz - sw in (-1, 0) or abs(z * w) == 0
        assert oracle.scale(z + w) <= max(sz, sw) + 1
        # equ:sz: s(z) in max{s(Re z), s(Im z)} + {0, 1}
        assert oracle.scale(z) - max(oracle.scale(z.real), oracle.scale(z.imag)) in (0, 1)


# ------------------------------------------------------------------ hull ---

def test_hull_worked_example(worked):
    s = np.array(worked["scales"], dtype=np.int32)
    hk, hh = oracle.hull(s)
    exp = worked["derived_not_printed"]
    assert hk.tolist() == exp["hull_k"] and hh.tolist() == exp["hull_h"]
    bk, bh = hull_brute([int(v) for v in s])
    assert hk.tolist() == bk.tolist() and hh.tolist() == bh.tolist()


def _rand_scales(rng, d):
    kind = rng.integers(0, 4)
    if kind == 0:
        s = rng.integers(-8, 9, size=d + 1)            # many ties
    elif kind == 1:
        s = rng.integers(-300, 300, size=d + 1)
    elif kind == 2:
        k = np.arange(d + 1)
        s = np.floor(40 * np.sin(np.pi * k / max(d, 1)) + rng.normal(0, 3, d + 1)).astype(np.int64)
    else:
        s = np.cumsum(rng.integers(-3, 4, size=d + 1))   # random walk
    s = [int(v) for v in s]
    # interior zeros (s = -inf), sometimes at the ends too
    for k in range(d + 1):
        if rng.random() < 0.15:
            s[k] = None
    if all(v is None for v in s):
        s[int(rng.integers(0, d + 1))] = 0
    return s


def test_hull_vs_bruteforce_random():
    rng = np.random.default_rng(3)
    for _ in range(1500):
        d = int(rng.integers(0, 64))
        s = _rand_scales(rng, d)
        arr = np.array([NEG if v is None else v for v in s], dtype=np.int32)
        hk, hh = oracle.hull(arr)
        bk, bh = hull_brute(s)
        assert hk.tolist() == bk.tolist(), (s, hk, bk)
        assert hh.tolist() == bh.tolist()


def test_hull_closed_forms():
    # constant scales: two vertices (SPEC-style closed form)
    hk, hh = oracle.hull(np.full(100, 7, dtype=np.int32))
    assert hk.tolist() == [0, 99] and hh.tolist() == [7, 7]
    # strictly concave integer data is its own cover: -k^2
    s = np.array([-(k * k) for k in range(40)], dtype=np.int32)
    hk, hh = oracle.hull(s)
    assert hk.tolist() == list(range(40))
    # monotone profile -- exercises the insertion sentinel: s = (0, 1, 5)
    hk, hh = oracle.hull(np.array([0, 1, 5], dtype=np.int32))
    assert hk.tolist() == [0, 2] and hh.tolist() == [0, 5]


def test_hull_invariants_large():
    rng = np.random.default_rng(4)
    d = 200000
    k = np.arange(d + 1)
    s = np.floor(1000 * np.sin(np.pi * k / d)).astype(np.int32) + 1   # SURVEY 8(d) stress profile
    s[rng.random(d + 1) < 0.01] = NEG
    s[0] = 1; s[-1] = 1
    hk, hh = oracle.hull(s)
    assert len(hk) > 300
    dk = np.diff(hk.astype(np.int64)); dh = np.diff(hh.astype(np.int64))
    # strictly decreasing slopes
    assert np.all(dh[:-1] * dk[1:] > dh[1:] * dk[:-1])
    # majorant, touching at the vertices
    nz = np.flatnonzero(s != NEG)
    j = np.searchsorted(hk, nz, side="right") - 1
    j = np.minimum(j, len(hk) - 2)
    lhs = (s[nz].astype(np.int64) - hh[j]) * dk[j]
    rhs = dh[j] * (nz - hk[j])
    assert np.all(lhs <= rhs)
    assert np.all(s[hk] == hh)


# ------------------------------------------------------------------- G_p ---

def test_good_worked_example(worked):
    s = np.array(worked["scales"], dtype=np.int32)
    a = np.ldexp(1.0, s - 1).astype(np.complex128)   # |a_k| = 2^(s_k - 1) exactly
    assert oracle.scales(a).tolist() == worked["scales"]
    exp = worked["derived_not_printed"]
    P6 = oracle.OraclePoly(a, p=6, drop=6)
    assert np.flatnonzero(P6.good).tolist() == exp["G_drop6"]
    # drop = p + s(d) + 3 = 6 + 4 + 3 = 13; SPEC S:254 prints the same set
    P13 = oracle.OraclePoly(a, p=6)
    assert P13.drop == 13
    assert np.flatnonzero(P13.good).tolist() == exp["G_drop13"]


def test_good_simple_and_random():
    # P = 1 + z: G_p = {0, 1} for every p
    for p in (1, 6, 24, 53):
        P = oracle.OraclePoly(np.array([1.0, 1.0]), p=p)
        assert np.flatnonzero(P.good).tolist() == [0, 1]
        assert P.drop == p + 1 + 3
    rng = np.random.default_rng(5)
    for _ in range(400):
        d = int(rng.integers(1, 64))
        s = _rand_scales(rng, d)
        if sum(v is not None for v in s) < 2:
            continue
        arr = np.array([NEG if v is None else v for v in s], dtype=np.int32)
        a = np.where(arr == NEG, 0.0, np.ldexp(1.0, np.where(arr == NEG, 0, arr) - 1))
        drop = int(rng.integers(1, 40))
        P = oracle.OraclePoly(a, p=53, drop=drop)
        assert np.flatnonzero(P.good).tolist() == good_brute(s, drop)
        # hull vertices are always good
        assert set(P.hk.tolist()) <= set(np.flatnonzero(P.good).tolist())


def test_drop_formula():
    # D = p + s(d_eff) + 3 (eq:threshold); s(d) = 1 + floor(log2 d)
    assert oracle.drop_for(53, 1023) == 53 + 10 + 3
    assert oracle.drop_for(53, (1 << 20) - 1) == 53 + 20 + 3
    assert oracle.drop_for(53, (1 << 22) - 1) == 78
    assert oracle.drop_for(24, (1 << 22) - 1) == 49
    assert oracle.drop_for(53, 1 << 20) == 53 + 21 + 3
