// fpe_math.cuh -- device arithmetic of the FPE hot path (sm_100a).
//
//  * double-double (dd) error-free transformations (Dekker/Knuth TwoSum/TwoProd);
//  * lambda = log2|z| correctly rounded to fp64 (R4; PAPER.md:1131 eq:defLambda)
//    from a dd logarithm with a Ziv rounding test;
//  * exact sign of lambda*I + J for integers I, J (all classification decisions,
//    DESIGN.md R14);
//  * z^n in extended range with compensated (dd-accurate) binary powering
//    ("compute z^l in 2 log2 l steps").
//
// All exactness-critical products/sums use fpe_mul/fpe_add so that nvcc's
// FMA contraction cannot change them.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "log_table.h"
#include "fpe_hd.cuh"

namespace fpe {

struct dd_t { double hi, lo; };

FPE_HD dd_t two_sum(double a, double b) {
  double s = fpe_add(a, b);
  double bb = fpe_sub(s, a);
  double e = fpe_add(fpe_sub(a, fpe_sub(s, bb)), fpe_sub(b, bb));
  return {s, e};
}
FPE_HD dd_t fast_two_sum(double a, double b) {  // |a| >= |b| or a == 0
  double s = fpe_add(a, b);
  return {s, fpe_sub(b, fpe_sub(s, a))};
}
FPE_HD dd_t two_prod(double a, double b) {
  double p = fpe_mul(a, b);
  return {p, fpe_fma(a, b, -p)};
}
FPE_HD dd_t dd_add(dd_t a, dd_t b) {
  dd_t s = two_sum(a.hi, b.hi);
  dd_t t = two_sum(a.lo, b.lo);
  s.lo = fpe_add(s.lo, t.hi);
  s = fast_two_sum(s.hi, s.lo);
  s.lo = fpe_add(s.lo, t.lo);
  return fast_two_sum(s.hi, s.lo);
}
FPE_HD dd_t dd_mul(dd_t a, dd_t b) {
  dd_t p = two_prod(a.hi, b.hi);
  p.lo = fpe_fma(a.hi, b.lo, fpe_fma(a.lo, b.hi, p.lo));
  return fast_two_sum(p.hi, p.lo);
}
FPE_HD dd_t dd_mul_d(dd_t a, double b) {
  dd_t p = two_prod(a.hi, b);
  p.lo = fpe_fma(a.lo, b, p.lo);
  return fast_two_sum(p.hi, p.lo);
}
FPE_HD dd_t dd_div(dd_t a, dd_t b) {
  double q1 = fpe_div(a.hi, b.hi);
  dd_t r = dd_add(a, dd_mul_d(b, -q1));
  double q2 = fpe_div(r.hi, b.hi);
  r = dd_add(r, dd_mul_d(b, -q2));
  double q3 = fpe_div(r.hi, b.hi);
  dd_t q = fast_two_sum(q1, q2);
  return dd_add(q, dd_t{q3, 0.0});
}

// 2^e as a double for -1022 <= e <= 1023.
FPE_HD double pow2i(int e) {
  return fpe_bits2d((long long)(e + 1023) << 52);
}
// x 2^e, exact when the scale factor is a normal double (one multiplication), else ldexp.
FPE_HD double ldexp_fast(double x, int e) {
  return (e >= -1022 && e <= 1023) ? fpe_mul(x, pow2i(e)) : ldexp(x, e);
}
// Exponent e with |x| = m 2^e, m in [1/2, 1), for finite nonzero normal or subnormal x.
FPE_HD int frexp_exp(double x) {
  const long long b = fpe_d2bits(x);
  const int be = (int)((b >> 52) & 0x7ff);
  if (be != 0 && be != 0x7ff) return be - 1022;   // normal: read the exponent field
  int e;
  (void)frexp(x, &e);                              // zero, subnormal, inf, NaN
  return e;
}

// dd constants (hi, lo): 1/ln2, 1/(2 ln2), 1/3, 1/5
#define FPE_INV_LN2_HI 0x1.71547652b82fep+0
#define FPE_INV_LN2_LO 0x1.777d0ffda0d24p-56
#define FPE_THIRD_HI 0x1.5555555555555p-2
#define FPE_THIRD_LO 0x1.5555555555555p-56
#define FPE_FIFTH_HI 0x1.999999999999ap-3
#define FPE_FIFTH_LO -0x1.999999999999ap-57

// log1p(u) for |u| <= 2^-7.9, relative error ~2^-104:
// log1p(u) = 2 atanh(s), s = u/(2+u) = 2s (1 + s^2/3 + s^4/5 + ... + s^12/13).
FPE_HD dd_t log1p_small(dd_t u) {
  if (u.hi == 0.0) return dd_t{0.0, 0.0};
  dd_t s = dd_div(u, dd_add(dd_t{2.0, 0.0}, u));
  dd_t s2 = dd_mul(s, s);
  double x = s2.hi;
  double b7 = fpe_fma(x, fpe_fma(x, fpe_fma(x, 1.0 / 13.0, 1.0 / 11.0), 1.0 / 9.0), 1.0 / 7.0);
  dd_t b5 = dd_add(dd_t{FPE_FIFTH_HI, FPE_FIFTH_LO}, dd_mul_d(s2, b7));
  dd_t b3 = dd_add(dd_t{FPE_THIRD_HI, FPE_THIRD_LO}, dd_mul(s2, b5));
  dd_t R = dd_mul(s2, b3);
  dd_t r = dd_add(s, dd_mul(s, R));
  return dd_t{r.hi * 2.0, r.lo * 2.0};
}

// log2 of w = (whi + wlo), w in (0, inf) finite; returns (j, frac) with
// log2 w = j + frac*(1/ln2) where frac = ln f is returned as dd and f = w 2^-j in [0.703, 1.414).
// Table-driven: f r_i = 1 + u, ln f = log1p(u) - ln r_i.
FPE_HD dd_t ln_reduced(double whi, double wlo, int* j_out) {
  int j = frexp_exp(whi);
  double f = ldexp(whi, -j);                 // [1/2, 1)
  if (f < FPE_LOGTAB_F0) { f *= 2.0; j -= 1; }
  double flo = ldexp(wlo, -j);
  int i = fpe_d2i_rn((f - FPE_LOGTAB_F0) * 256.0);
  i = max(0, min(i, FPE_LOGTAB_N - 1));
  double r = fpe_logtab(i, 0);
  dd_t L0 = dd_t{fpe_logtab(i, 1), fpe_logtab(i, 2)};
  dd_t p = two_prod(f, r);
  dd_t u = fast_two_sum(fpe_sub(p.hi, 1.0), fpe_fma(flo, r, p.lo));  // p.hi - 1 exact (Sterbenz)
  *j_out = j;
  return dd_add(log1p_small(u), L0);
}

// Exact sum of five doubles as a dd (grow-expansion then compression).
FPE_HD dd_t exact_sum5(double t0, double t1, double t2, double t3, double t4) {
  double h[5];
  h[0] = t0;
  double in[4] = {t1, t2, t3, t4};
#pragma unroll
  for (int m = 1; m <= 4; ++m) {   // add in[m-1] to expansion h[0..m-1]
    double Q = in[m - 1];
#pragma unroll
    for (int i = 0; i < m; ++i) {
      dd_t s = two_sum(Q, h[i]);
      Q = s.hi;
      h[i] = s.lo;
    }
    h[m] = Q;
  }
  double hi = h[4], lo = 0.0;
#pragma unroll
  for (int i = 3; i >= 0; --i) {
    dd_t s = two_sum(hi, h[i]);
    hi = s.hi;
    lo = fpe_add(lo, s.lo);
  }
  return fast_two_sum(hi, lo);
}

// Round hi+lo (a normalised dd, |lo| <= ulp(hi)/2) to fp64; flag when within tol of a
// rounding boundary (midpoint between consecutive doubles).
FPE_HD double round_checked(dd_t v, double tol, int* hard) {
  double h = v.hi;
  if (h == 0.0) return v.lo;  // only arises when the value is exactly representable
  int e = frexp_exp(h);              // |h| in [2^(e-1), 2^e)
  double ulp = ldexp(1.0, e - 53);   // spacing above |h| (normal range)
  double half = 0.5 * ulp;
  bool pow2 = (fabs(h) == ldexp(1.0, e - 1));
  // boundary below |h| is at distance ulp/4 when |h| is a power of two
  bool toward_zero = (v.lo != 0.0) && ((v.lo < 0.0) == (h > 0.0));
  double dist = (pow2 && toward_zero) ? 0.25 * ulp : half;
  if (fabs(dist - fabs(v.lo)) <= tol) *hard = 1;
  return h;
}

// lambda = RN64(log2|z|) for z = x + iy (complex) or x (real, y ignored).
// Returns -inf for z = 0 and NaN for non-finite z; *hard set on a Ziv failure
// (|true - boundary| < 2^-96 |lambda|; expected never, R4).
FPE_HD double lambda_cr(double x, double y, bool cplx, int* hard) {
  *hard = 0;
  if (!cplx) y = 0.0;
  if (!isfinite(x) || !isfinite(y)) return fpe_bits2d(0x7ff8000000000000LL);
  double ax = fabs(x), ay = fabs(y);
  if (ay > ax) { double t = ax; ax = ay; ay = t; }
  if (ax == 0.0) return -INFINITY;
  const dd_t INV_LN2 = {FPE_INV_LN2_HI, FPE_INV_LN2_LO};
  dd_t lam;
  if (ay == 0.0) {                                   // |z| = ax
    double t = fpe_sub(ax, 1.0);
    if (ax >= 0.5 && ax <= 2.0 && fabs(t) <= 0x1p-8) {   // t exact (Sterbenz); relative accuracy near 1
      lam = dd_mul(log1p_small(dd_t{t, 0.0}), INV_LN2);
    } else {
      int j;
      dd_t L = ln_reduced(ax, 0.0, &j);
      lam = dd_add(dd_t{(double)j, 0.0}, dd_mul(L, INV_LN2));
    }
  } else {
    double v = fpe_fma(ax, ax, ay * ay);
    if (v >= 0.5 && v <= 2.0) {                      // near |z| = 1: t = x^2 + y^2 - 1 exactly
      if (ay < 0x1p-480) {
        if (ax == 1.0) {
          // t = ay^2 < 2^-960: lambda = t/(2 ln 2) (1 - t/2 + ...), relative term < 2^-960.
          int k = frexp_exp(ay);
          double ys = ldexp(ay, -k);                  // [1/2, 1)
          dd_t t = two_prod(ys, ys);                  // t = ts 2^(2k)
          dd_t L = dd_mul(t, INV_LN2);
          L.hi *= 0.5; L.lo *= 0.5;
          // result = L 2^(2k): round with a quantum of 2^-1074 (subnormal) or exactly (normal)
          int sc = 2 * k;
          int eL = frexp_exp(L.hi);
          if (eL + sc > -1021) {
            double r = round_checked(L, fabs(L.hi) * 0x1p-96, hard);
            return ldexp(r, sc);
          }
          double A = ldexp(L.hi, 1074 + sc), B = ldexp(L.lo, 1074 + sc);
          double n = rint(A);
          double fr = fpe_add(fpe_sub(A, n), B);
          if (fr > 0.5) n += 1.0; else if (fr < -0.5) n -= 1.0;
          if (fabs(fabs(fr) - 0.5) < 0x1p-40) *hard = 1;
          return ldexp(n, -1074);
        }
        ay = 0.0;   // |x^2 - 1| >= 2^-106 dominates y^2 < 2^-960 beyond any rounding margin
      }
      dd_t p = two_prod(ax, ax);
      dd_t a = two_sum(p.hi, -1.0);
      dd_t q = two_prod(ay, ay);
      dd_t t = exact_sum5(a.hi, a.lo, p.lo, q.hi, q.lo);
      if (fabs(t.hi) <= 0x1p-8) {
        lam = dd_mul(log1p_small(t), INV_LN2);
      } else {
        dd_t w = dd_add(dd_t{1.0, 0.0}, t);
        int j;
        dd_t L = ln_reduced(w.hi, w.lo, &j);
        lam = dd_add(dd_t{(double)j, 0.0}, dd_mul(L, INV_LN2));
      }
      lam.hi *= 0.5; lam.lo *= 0.5;
    } else {                                         // far from |z| = 1: lambda = e + log2(v')/2
      int e = frexp_exp(ax);
      double xs = ldexp(ax, -e), ys = ldexp(ay, -e);
      dd_t vv = dd_add(two_prod(xs, xs), two_prod(ys, ys));   // [1/4, 2)
      int j;
      dd_t L = ln_reduced(vv.hi, vv.lo, &j);
      dd_t h = dd_mul(L, INV_LN2);
      h = dd_add(dd_t{(double)j, 0.0}, h);
      h.hi *= 0.5; h.lo *= 0.5;
      lam = dd_add(dd_t{(double)e, 0.0}, h);
    }
  }
  return round_checked(lam, fabs(lam.hi) * 0x1p-96, hard);
}

// Exact sign of lambda*I + J for integers |I|, |J| < 2^53 (R14): I and J are exact
// doubles and the fused multiply-add evaluates lambda*I + J exactly before its single rounding,
// and rounding to nearest preserves the sign; it cannot underflow to zero because a nonzero
// lambda*I + J is a multiple of min(1, ulp(lambda)) >= 2^-1074.
FPE_HD int sign_lin(double lam, long long I, long long J) {
  double t = fpe_fma(lam, (double)I, (double)J);
  return (t > 0.0) - (t < 0.0);
}

// ---------------------------------------------------------------------------------
// Extended-range complex value (h + e) 2^E: h the fp64 approximation, e its error term.
struct xc_t { double hr, hi, er, ei; long long E; };

FPE_HD void xc_renorm(xc_t& v) {
  dd_t r = two_sum(v.hr, v.er), i = two_sum(v.hi, v.ei);   // keep |e| <= ulp(h)/2
  v.hr = r.hi; v.er = r.lo; v.hi = i.hi; v.ei = i.lo;
  double m = fmax(fabs(v.hr), fabs(v.hi));
  if (m == 0.0) return;
  int e = frexp_exp(m);
  double s = pow2i(-e);
  v.hr *= s; v.hi *= s; v.er *= s; v.ei *= s;
  v.E += e;
}

// (h+e)^2 with the products of h exact (TwoProd) and the error propagated to first order.
FPE_HD void xc_sqr(xc_t& v) {
  double a = v.hr, b = v.hi, c = v.er, d = v.ei;
  dd_t p1 = two_prod(a, a), p2 = two_prod(b, b);
  dd_t sr = two_sum(p1.hi, -p2.hi);
  double re_err = sr.lo + (p1.lo - p2.lo);
  double a2 = a + a;
  dd_t p3 = two_prod(a2, b);
  double xr = 2.0 * fpe_fma(a, c, -b * d);
  double xi = 2.0 * fpe_fma(a, d, b * c);
  v.hr = sr.hi; v.hi = p3.hi;
  v.er = re_err + xr; v.ei = p3.lo + xi;
  v.E *= 2;                               // (h 2^E)^2 = h^2 2^(2E)
}

// (h+e) * w for an exact w = u + iv.
FPE_HD void xc_mul_exact(xc_t& v, double u, double w) {
  double a = v.hr, b = v.hi, c = v.er, d = v.ei;
  dd_t p1 = two_prod(a, u), p2 = two_prod(b, w);
  dd_t sr = two_sum(p1.hi, -p2.hi);
  dd_t p3 = two_prod(a, w), p4 = two_prod(b, u);
  dd_t si = two_sum(p3.hi, p4.hi);
  v.hr = sr.hi; v.hi = si.hi;
  v.er = sr.lo + (p1.lo - p2.lo) + fpe_fma(c, u, -d * w);
  v.ei = si.lo + (p3.lo + p4.lo) + fpe_fma(c, w, d * u);
}

// z^n (n >= 0) for finite nonzero z = x + iy, relative error ~ n 2^-104 + 2^-53.
// Left-to-right binary powering on w = z 2^-ez (|w| in [1/2, sqrt 2)).
FPE_HD xc_t xc_pow(double x, double y, long long n) {
  xc_t v;
  v.hr = 1.0; v.hi = 0.0; v.er = 0.0; v.ei = 0.0; v.E = 0;
  if (n <= 0) return v;
  int ez = frexp_exp(fmax(fabs(x), fabs(y)));
  double u = ldexp(x, -ez), w = ldexp(y, -ez);
  v.hr = u; v.hi = w;
  int top = 63 - fpe_clzll(n);
  for (int b = top - 1; b >= 0; --b) {
    xc_sqr(v);
    if ((n >> b) & 1) xc_mul_exact(v, u, w);
    xc_renorm(v);
  }
  v.E += n * (long long)ez;
  return v;
}

// Real version: x^n for finite nonzero real x.
struct xr_t { double h, e; long long E; };
FPE_HD xr_t xr_pow(double x, long long n) {
  xr_t v{1.0, 0.0, 0};
  if (n <= 0) return v;
  int ex = frexp_exp(x);
  double u = ldexp(x, -ex);
  v.h = u;
  int top = 63 - fpe_clzll(n);
  for (int b = top - 1; b >= 0; --b) {
    dd_t p = two_prod(v.h, v.h);
    double e = p.lo + 2.0 * v.h * v.e;
    v.h = p.hi; v.e = e; v.E *= 2;
    if ((n >> b) & 1) {
      dd_t q = two_prod(v.h, u);
      v.e = q.lo + v.e * u;
      v.h = q.hi;
    }
    dd_t f = fast_two_sum(v.h, v.e);
    v.h = f.hi; v.e = f.lo;
    int k = frexp_exp(v.h);
    double s = pow2i(-k);
    v.h *= s; v.e *= s; v.E += k;
  }
  v.E += n * (long long)ex;
  return v;
}

// ------------------------------------------------------------------------------------------
// The classifier's enclosure of log2|z| (k_classify_bucket fast path; host-tested by
// tests/test_devmath_host.py against the oracle's correctly rounded lambda).
// log2 v for v in [1/4, 2) (normal): v = f 2^j, f in [F0, 1.41) by bit manipulation, f r_i = 1 + u with the
// table of fpe_logtab (|u| < 2^-8.5), ln(1 + u) to u^5 in fp64 (truncation u^6/6 < 2^-53):
// |error| < 2^-51 absolute.
FPE_HD double log2_fast(double v) {
  const long long b = fpe_d2bits(v);
  int j = (int)((b >> 52) & 0x7ff) - 1022;
  double f = fpe_bits2d((b & 0x000fffffffffffffLL) | 0x3fe0000000000000LL);   // [1/2, 1)
  if (f < FPE_LOGTAB_F0) { f *= 2.0; j -= 1; }
  int i = fpe_d2i_rn((f - FPE_LOGTAB_F0) * 256.0);
  i = (i < 0 ? 0 : (i > FPE_LOGTAB_N - 1 ? FPE_LOGTAB_N - 1 : i));
  const double r = fpe_logtab(i, 0), L0 = fpe_logtab(i, 1);
  const double u = fpe_fma(f, r, -1.0);
  double p = fpe_fma(u, 0.2, -0.25);
  p = fpe_fma(u, p, 1.0 / 3.0);
  p = fpe_fma(u, p, -0.5);
  p = fpe_fma(u, p, 1.0);
  return fpe_fma(fpe_fma(u, p, L0), FPE_INV_LN2_HI, (double)j);
}

// An enclosure of log2|z| from plain fp64 (finite nonzero z): |z|^2 4^-e in [1/4, 2) to 2^-52 relative,
// log2_fast to 2^-51, so |error| < 2^-50 + 2^-53 |lambda|; the enclosure is widened to
// 2^-48 + 2^-50 |lambda|.  Powers of two are taken from the exponent bits (subnormal |z| via frexp).
FPE_HD void lambda_enclosure(double x, double y, bool cplx, double& lo, double& hi, double& mid) {
  double ax = fabs(x), ay = cplx ? fabs(y) : 0.0;
  if (ay > ax) { const double t = ax; ax = ay; ay = t; }
  int e;
  double xs, ys;
  if (ax >= 0x1p-1000 && ax < 0x1p1000) {
    e = (int)((fpe_d2bits(ax) >> 52) & 0x7ff) - 1022;                 // ax = xs 2^e, xs in [1/2, 1)
    const double sc = fpe_bits2d((long long)(1023 - e) << 52);       // 2^-e, exact
    xs = ax * sc;
    ys = ay * sc;
  } else {
    e = frexp_exp(ax);
    xs = ldexp(ax, -e);
    ys = ldexp(ay, -e);
  }
  const double v = fpe_fma(xs, xs, ys * ys);
  mid = (double)e + 0.5 * log2_fast(v);
  const double w = fpe_fma(fabs(mid), 0x1p-50, 0x1p-48);
  lo = mid - w;
  hi = mid + w;
}

// ------------------------------------------------------------------------------------------
// The work bucketing's sort key (eval_tiled.cu k_bucket_hist / k_classify_bucket; host-tested by
// tests/test_devmath_host.py).  The key only decides which points share a warp: every point's arithmetic
// depends on its own window alone, so any deterministic function of z gives bitwise the same results.  It is
// the bits of an fp64 estimate of log2|z| (lambda_enclosure's midpoint, within 2^-50 + 2^-53 |lambda| of
// lambda): |lambda| = (1.m) 2^E gives mag = (E + 53) << 16 | the top 16 bits of m, monotone in
// |lambda| >= 2^-52, and the sign of lambda on top -- 23 bits, monotone in |z|.  l and r are non-decreasing in
// lambda (d/dlambda of cover(k) + lambda k - N is k - k_lambda), so points with close keys have nested, nearly
// equal windows.  z = 0 and non-finite z take key 0.  Both kernels call these functions on the same points.
constexpr int kKeyBits = 23;
FPE_HD bool key_point(double x, double y, bool cplx) {
  return isfinite(x) && isfinite(y) && (x != 0.0 || (cplx && y != 0.0));
}
// lam: lambda_enclosure's midpoint for a key_point (finite nonzero z)
FPE_HD uint32_t key_of_estimate(double lam) {
  const unsigned long long b = (unsigned long long)fpe_d2bits(fabs(lam));
  const int E = (int)(b >> 52) - 1023;
  uint32_t mag = 0;
  if (E >= -52) mag = ((uint32_t)(E + 53) << 16) | (uint32_t)((b >> 36) & 0xffff);
  return (lam >= 0.0) ? (1u << 22) + mag : (1u << 22) - 1u - mag;
}
FPE_HD uint32_t bucket_key(double x, double y, bool cplx) {
  if (!key_point(x, y, cplx)) return 0u;
  double lo, hi, lam;
  lambda_enclosure(x, y, cplx, lo, hi, lam);
  return key_of_estimate(lam);
}
// The lambda estimates whose keys fall in bucket b of 2^cb (keys [b 2^s, (b + 1) 2^s), s = kKeyBits - cb): a
// superset [lo, hi] (mag values no estimate produces -- exponent field 0 -- are read as |lambda| < 2^-52).
FPE_HD double key_mag_lo(uint32_t mag) {   // the least |lambda| with this mag
  return (mag >> 16) == 0 ? 0.0 : ldexp(1.0 + (mag & 0xffff) * 0x1p-16, (int)(mag >> 16) - 53);
}
FPE_HD double key_mag_hi(uint32_t mag) {   // above every |lambda| with this mag
  return (mag >> 16) == 0 ? 0x1p-52 : ldexp(1.0 + ((mag & 0xffff) + 1) * 0x1p-16, (int)(mag >> 16) - 53);
}
FPE_HD void bucket_estimates(uint32_t b, int cb, double& lo, double& hi) {
  const int s = kKeyBits - cb;
  const uint32_t k0 = b << s, k1 = ((b + 1) << s) - 1;
  if (k0 >= (1u << 22)) { lo = key_mag_lo(k0 - (1u << 22)); hi = key_mag_hi(k1 - (1u << 22)); }
  else { lo = -key_mag_hi((1u << 22) - 1 - k0); hi = -key_mag_lo((1u << 22) - 1 - k1); }
}

}  // namespace fpe
