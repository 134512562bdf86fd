"""CPU tests of the product library: it loads, exports every symbol of include/fpe.h,
and its host preconditioner agrees bit-exactly with the oracle (cover, D, G_p, layout).
No compute call touches a GPU here.
"""
import os
import re

import numpy as np
import pytest

import oracle
import workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def fpe():
    from paper_2211_06320_b200 import build
    build.build()
    import paper_2211_06320_b200 as m
    return m


def test_exports_every_declared_symbol(fpe):
    from paper_2211_06320_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "fpe.h")).read()
    names = set(re.findall(r"^\s*(?:fpe_status|void|const char\*)\s+(fpe_\w+)\s*\(", hdr, re.M))
    assert len(names) >= 14, names
    L = _lib.lib()
    for n in names:
        assert hasattr(L, n), n
    assert names <= set(_lib.SIGNATURES), names - set(_lib.SIGNATURES)


def _ldexp(v, sh):
    if np.iscomplexobj(v):
        return np.ldexp(v.real, sh) + 1j * np.ldexp(v.imag, sh)
    return np.ldexp(v, sh)


def _check_against_oracle(fpe, a, p=None, drop=None):
    buf = fpe.precondition_buffer(a, p=p, drop=drop)
    h = fpe.header_fields(buf)
    P = oracle.OraclePoly(a, p=p, drop=drop)
    assert h["magic"] == 0x4650453230304232
    assert h["hk"].tolist() == P.hk.tolist()
    assert h["hh"].tolist() == P.hh.tolist()
    assert (h["k_min"], h["k_max"], h["drop"]) == (P.k_min, P.k_max, P.drop)
    good = np.flatnonzero(P.good)
    assert h["n_good"] == len(good)
    sh = h["shift"]
    if h["sparse"]:
        assert h["sidx"].tolist() == good.tolist()
        np.testing.assert_array_equal(h["coef"], _ldexp(P.coeffs[good], -sh).astype(h["coef"].dtype))
    else:
        dense = np.zeros(P.k_max - P.k_min + 1, dtype=P.coeffs.dtype)
        sel = good - P.k_min
        dense[sel] = P.coeffs[good]
        np.testing.assert_array_equal(h["coef"], _ldexp(dense, -sh).astype(h["coef"].dtype))
        if "prefix" in h:
            np.testing.assert_array_equal(h["prefix"], np.concatenate([[0], np.cumsum(P.good[P.k_min:P.k_max + 1])]))
        else:
            assert h["all_good"] == 1 and len(good) == P.k_max - P.k_min + 1
    return h, P


def test_worked_example_layout(fpe, worked):
    s = np.array(worked["scales"])
    a = np.ldexp(1.0, s - 1).astype(np.complex128)
    h, P = _check_against_oracle(fpe, a, p=6, drop=6)
    assert np.flatnonzero(P.good).tolist() == worked["derived_not_printed"]["G_drop6"]
    _check_against_oracle(fpe, a, p=6)


@pytest.mark.parametrize("cfg,d", [(1, None), (2, (1 << 14) - 1), (3, (1 << 16) - 1), (5, (1 << 12) - 1)])
def test_configs_match_oracle(fpe, cfg, d):
    a = workloads.coefficients(cfg, d)
    _check_against_oracle(fpe, a)
    if cfg == 5:
        _check_against_oracle(fpe, workloads.to_fp32(a))


def test_sparse_config_matches_oracle(fpe):
    a = workloads.coefficients(4, d=1 << 18)
    h, P = _check_against_oracle(fpe, a)
    assert h["sparse"] == 1


def test_full_size_cfg3_cover(fpe):
    a = workloads.coefficients(3)
    h, P = _check_against_oracle(fpe, a)
    assert 25 <= len(h["hk"]) <= 60     # SURVEY 8(d) estimated 41-43 vertices with approximate scales
    assert h["all_good"] == 1


def test_degenerate_polys(fpe):
    rng = np.random.default_rng(7)
    cases = [
        np.array([0.0, 0.0, 3.0]),                         # monomial 3 z^2
        np.array([1.0, 1.0]),                              # 1 + z
        np.array([0, 0, 1 + 1j, 0, 0, 0, 2j, 0]),          # leading/trailing zeros
        np.full(100, 0.5 + 0.5j),                          # all equal scales
        np.array([5e-324, 1.0, 1e300]),                    # subnormal and huge
        np.ldexp(1.0, np.floor(300 * np.sin(np.pi * np.arange(2001) / 2000)).astype(int)),
    ]
    for _ in range(40):
        d = int(rng.integers(1, 300))
        a = rng.normal(size=d + 1) * np.exp2(rng.integers(-200, 200, size=d + 1))
        a[rng.random(d + 1) < 0.3] = 0
        if not a.any():
            a[0] = 1
        cases.append(a)
        cases.append(a * np.exp(1j * rng.uniform(0, 6.3, d + 1)))
    for cplx in (False, True):   # coefficients at 2^+-900: wide handles
        a = rng.normal(size=501) * np.exp2(rng.integers(-900, 900, size=501))
        a[0], a[-1] = 2.0 ** -950, 3 * 2.0 ** 950        # cover endpoints 1900 bits apart
        cases.append(a * np.exp(1j * rng.uniform(0, 6.3, 501)) if cplx else a)
    n_wide = 0
    for a in cases:
        h, P = _check_against_oracle(fpe, a)
        g = P.s[P.good.astype(bool)]
        # scales of G_p spanning more than 1000 bits: a "wide" handle (raw coefficients, exponent-tracked
        # evaluation); otherwise one common shift maps the cover's top to 2^0
        assert h["wide"] == int(g.max() - g.min() > 1000)
        assert h["shift"] == (0 if h["wide"] else P.hh.max())
        n_wide += h["wide"]
    assert n_wide >= 3
    # single precision: spans beyond 100 bits are wide (the fp32 working range)
    a = (rng.normal(size=300) * np.exp2(rng.integers(-100, 100, size=300))).astype(np.float32)
    h, P = _check_against_oracle(fpe, a)
    g = P.s[P.good.astype(bool)]
    assert h["wide"] == int(g.max() - g.min() > 100) == 1 and h["shift"] == 0


def test_errors(fpe):
    with pytest.raises(fpe.FpeError) as e:
        fpe.precondition_buffer(np.zeros(10))
    assert e.value.status == 2
    with pytest.raises(fpe.FpeError) as e:
        fpe.precondition_buffer(np.array([1.0, np.nan]))
    assert e.value.status == 3
    with pytest.raises(TypeError):
        fpe.precondition_buffer(np.arange(5))   # int64 is not a supported dtype
