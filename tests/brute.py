"""Brute-force references used to pin the oracle (tests only).

Exact rational arithmetic (``fractions.Fraction``) and numpy integer
cross-multiplication, straight from the definitions:

* scale s(z): the integer sigma with 2^(sigma-1) <= |z| < 2^sigma;
* concave cover: the minimal concave majorant of the points (k, s_k)
   -- a point is a canonical vertex iff it lies strictly
  above every chord over it;
* G_p, k_lambda, N_lambda, [l, r]: linear scans of Algorithm FPE_p lines 4-8
   over every integer k.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

NEG = None  # s(0) = -inf


def scale_exact(re: float, im: float = 0.0):
    """s(z) from |z|^2 as an exact rational."""
    v = Fraction(re) ** 2 + Fraction(im) ** 2
    if v == 0:
        return NEG
    # find sigma with 4^(sigma-1) <= v < 4^sigma
    sig = (v.numerator.bit_length() - v.denominator.bit_length()) // 2
    while Fraction(4) ** (sig - 1) > v:
        sig -= 1
    while Fraction(4) ** sig <= v:
        sig += 1
    return sig


def hull_brute(s):
    """Canonical upper hull vertices of {(k, s_k) : s_k is not None}, O(d^3) numpy."""
    ks = np.array([k for k, v in enumerate(s) if v is not None], dtype=np.int64)
    hs = np.array([s[k] for k in ks], dtype=np.int64)
    n = len(ks)
    keep = []
    for t in range(n):
        if t == 0 or t == n - 1:
            keep.append(t)
            continue
        i = np.arange(t)[:, None]
        j = np.arange(t + 1, n)[None, :]
        # point t strictly above chord (i, j):  (h_t - h_i)(k_j - k_i) > (h_j - h_i)(k_t - k_i)
        above = (hs[t] - hs[i]) * (ks[j] - ks[i]) > (hs[j] - hs[i]) * (ks[t] - ks[i])
        if above.all():
            keep.append(t)
    return ks[keep].astype(np.int32), hs[keep].astype(np.int32)


def cover_value(hk, hh, k) -> Fraction:
    """cover(k) as an exact rational by linear interpolation on the vertex list."""
    hk = [int(x) for x in hk]
    hh = [int(x) for x in hh]
    if len(hk) == 1:
        return Fraction(hh[0])
    for j in range(len(hk) - 1):
        if hk[j] <= k <= hk[j + 1]:
            return Fraction(hh[j]) + Fraction(hh[j + 1] - hh[j], hk[j + 1] - hk[j]) * (k - hk[j])
    raise ValueError(k)


def good_brute(s, drop):
    """G_p by the chord characterisation: s_k + drop >= every chord value over k."""
    ks = [k for k, v in enumerate(s) if v is not None]
    hk, hh = hull_brute(s)
    out = []
    for k in ks:
        if cover_value(hk, hh, k) - drop <= s[k]:
            out.append(k)
    return out


def classify_brute(hk, hh, drop, lam: float):
    """(i*, l, r) by linear scans with exact rationals (lam is an exact dyadic)."""
    L = Fraction(lam)
    vals = [Fraction(int(h)) + L * int(k) for k, h in zip(hk, hh)]
    N = max(vals)
    istar = vals.index(N)  # smallest maximiser
    kmin, kmax = int(hk[0]), int(hk[-1])
    inside = [k for k in range(kmin, kmax + 1) if cover_value(hk, hh, k) + L * k >= N - drop]
    return istar, min(inside), max(inside), N
