// fpe_polar.cuh -- fast log2|z|, arg z and z^n in polar form (host/device).
//
//  * log2abs_quick: log2|z| as a double-double with relative error ~2^-95 (table-driven
//    reduction, fpe_logtab, plus a degree-11 log1p series), ~70 fp64 operations.
//  * lambda_fast:   lambda = RN64(log2|z|) (reading G4; PAPER.md:1131 eq:defLambda):
//    the quick value is rounded and checked with a Ziv test at 2^-80 relative; the rare
//    points that fail it go through the slower fully double-double lambda_cr (fpe_math.cuh).
//  * atan2_turns:   arg z / (2 pi) as a double-double (fpe_atantab + atan series).
//  * pow_polar:     z^n = 2^(n lambda) e^(2 pi i n tau) with n lambda and n tau formed exactly
//    enough that the result has relative error ~2^-50 for n < 2^31 (PAPER.md:1621-1622 computes
//    z^l by 2 log2 l multiplications; plain fp64 powering loses 0.29 l ulp, so
//    the library evaluates the same power through the logarithm instead).
#pragma once
#include "fpe_math.cuh"

namespace fpe {

#define FPE_INV_2PI_HI 0x1.45f306dc9c883p-3
#define FPE_INV_2PI_LO -0x1.6b01ec5417056p-57

// ln(1 + u) for a double-double u with |u| <= 2^-8: u - u^2/2 + u^3/3 - u^4/4 + u^5/5 + u^6 R(u)
// with the first five terms as double-doubles (an fp64 rounding of a term T costs 2^-53 T, which
// must stay below 2^-90 |u|) and R to u^6 in fp64 (truncation u^13/13 < 2^-99 |u|).
FPE_HD dd_t ln1p_series(dd_t u) {
  const double uh = u.hi, ul = u.lo;
  dd_t u2 = two_prod(uh, uh);
  u2.lo = fpe_fma(2.0 * uh, ul, u2.lo);
  dd_t u3 = two_prod(u2.hi, uh);
  u3.lo = fpe_fma(u2.lo, uh, fpe_fma(u2.hi, ul, u3.lo));
  dd_t t3 = two_prod(u3.hi, FPE_THIRD_HI);                 // u^3 / 3
  t3.lo = fpe_fma(u3.lo, FPE_THIRD_HI, fpe_fma(u3.hi, FPE_THIRD_LO, t3.lo));
  dd_t u4 = two_prod(u2.hi, u2.hi);
  u4.lo = fpe_fma(2.0 * u2.hi, u2.lo, u4.lo);
  dd_t u5 = two_prod(u4.hi, uh);
  u5.lo = fpe_fma(u4.lo, uh, u5.lo);
  dd_t t5 = two_prod(u5.hi, FPE_FIFTH_HI);                 // u^5 / 5
  t5.lo = fpe_fma(u5.lo, FPE_FIFTH_HI, fpe_fma(u5.hi, FPE_FIFTH_LO, t5.lo));
  double R = -1.0 / 12.0;
  R = fpe_fma(R, uh, 1.0 / 11.0);
  R = fpe_fma(R, uh, -1.0 / 10.0);
  R = fpe_fma(R, uh, 1.0 / 9.0);
  R = fpe_fma(R, uh, -1.0 / 8.0);
  R = fpe_fma(R, uh, 1.0 / 7.0);
  R = fpe_fma(R, uh, -1.0 / 6.0);
  const double u6R = fpe_mul(fpe_mul(u5.hi, uh), R);
  dd_t s = fast_two_sum(uh, -0.5 * u2.hi);
  dd_t s2 = fast_two_sum(s.hi, t3.hi);
  dd_t s3 = fast_two_sum(s2.hi, -0.25 * u4.hi);
  dd_t s4 = fast_two_sum(s3.hi, t5.hi);
  double lo = fpe_add(fpe_add(s.lo, s2.lo), fpe_add(s3.lo, s4.lo));
  lo = fpe_add(lo, fpe_add(fpe_add(ul, -0.5 * u2.lo), fpe_add(t3.lo, -0.25 * u4.lo)));
  lo = fpe_add(lo, fpe_add(t5.lo, u6R));
  return fast_two_sum(s4.hi, lo);
}

// ln f for f = fh + fl in [FPE_LOGTAB_F0, 1.4141): f r_i = 1 + u, ln f = ln1p(u) - ln r_i.
FPE_HD dd_t ln_table(double fh, double fl) {
  int i = fpe_d2i_rn((fh - FPE_LOGTAB_F0) * 256.0);
  i = i < 0 ? 0 : (i > FPE_LOGTAB_N - 1 ? FPE_LOGTAB_N - 1 : i);
  const double r = fpe_logtab(i, 0);
  dd_t p = two_prod(fh, r);
  const double uh = fpe_sub(p.hi, 1.0);          // exact: p.hi in [1/2, 2] (Sterbenz)
  dd_t u = fast_two_sum(uh, fpe_fma(fl, r, p.lo));
  dd_t L = ln1p_series(u);
  dd_t s = two_sum(fpe_logtab(i, 1), L.hi);
  return fast_two_sum(s.hi, fpe_add(s.lo, fpe_add(fpe_logtab(i, 2), L.lo)));
}

FPE_HD dd_t dd_times_inv_ln2(dd_t a) {
  return dd_mul(a, dd_t{FPE_INV_LN2_HI, FPE_INV_LN2_LO});
}

// log2 of a double-double v = vh + vl > 0 (vh normal): j + log2(v 2^-j).
FPE_HD dd_t log2_dd(double vh, double vl) {
  int j = frexp_exp(vh);
  double f = ldexp_fast(vh, -j), fl = ldexp_fast(vl, -j);
  if (f < FPE_LOGTAB_F0) { f *= 2.0; fl *= 2.0; j -= 1; }
  dd_t L = dd_times_inv_ln2(ln_table(f, fl));
  dd_t s = two_sum((double)j, L.hi);
  return fast_two_sum(s.hi, fpe_add(s.lo, L.lo));
}

// log2|z| as a double-double for finite nonzero z (x + iy, or x when !cplx).
FPE_HD dd_t log2abs_quick(double x, double y, bool cplx) {
  double ax = fabs(x), ay = cplx ? fabs(y) : 0.0;
  if (ay > ax) { double t = ax; ax = ay; ay = t; }
  if (ay == 0.0) {
    const double t = fpe_sub(ax, 1.0);           // exact for ax in [1/2, 2]
    if (ax >= 0.5 && ax <= 2.0 && fabs(t) <= 0x1p-8) return dd_times_inv_ln2(ln1p_series(dd_t{t, 0.0}));
    return log2_dd(ax, 0.0);
  }
  // near |z| = 1 the relative accuracy of lambda needs t = x^2 + y^2 - 1 formed directly
  const double v0 = fpe_fma(ax, ax, fpe_mul(ay, ay));
  if (v0 >= 0.98 && v0 <= 1.02) {
    dd_t p = two_prod(ax, ax), q = two_prod(ay, ay);
    dd_t a = two_sum(p.hi, -1.0);                // p.hi may be below 1/2: not Sterbenz-exact
    dd_t s = two_sum(a.hi, q.hi);
    dd_t t = two_sum(s.hi, fpe_add(fpe_add(s.lo, a.lo), fpe_add(p.lo, q.lo)));
    if (fabs(t.hi) <= 0x1p-8) {
      dd_t L = dd_times_inv_ln2(ln1p_series(t));
      return dd_t{0.5 * L.hi, 0.5 * L.lo};
    }
  }
  const int e = frexp_exp(ax);
  const double xs = ldexp_fast(ax, -e), ys = ldexp_fast(ay, -e);   // xs in [1/2, 1)
  dd_t p = two_prod(xs, xs), q = two_prod(ys, ys);
  dd_t s = two_sum(p.hi, q.hi);
  dd_t v = fast_two_sum(s.hi, fpe_add(s.lo, fpe_add(p.lo, q.lo)));   // |z|^2 4^-e in [1/4, 2)
  dd_t L = log2_dd(v.hi, v.lo);
  dd_t h = two_sum((double)e, 0.5 * L.hi);
  return fast_two_sum(h.hi, fpe_add(h.lo, 0.5 * L.lo));
}

// lambda = RN64(log2|z|); -inf for z = 0, NaN for non-finite z; *hard as lambda_cr.
FPE_HD double lambda_fast(double x, double y, bool cplx, int* hard) {
  *hard = 0;
  if (!cplx) y = 0.0;
  if (!isfinite(x) || !isfinite(y)) return fpe_bits2d(0x7ff8000000000000LL);
  if (x == 0.0 && y == 0.0) return -INFINITY;
  dd_t L = log2abs_quick(x, y, cplx);
  // error bound: 2^-80 relative (series, tables) plus 2^-102 absolute (|z|^2 - 1 near |z| = 1)
  int fail = 0;
  double r = round_checked(L, fpe_fma(fabs(L.hi), 0x1p-80, 0x1p-102), &fail);
  if (!fail && r != 0.0) return r;
  return lambda_cr(x, y, cplx, hard);
}

// arg(z) / (2 pi) in (-1/2, 1/2] as a double-double, z finite and nonzero.
FPE_HD dd_t atan2_turns(double x, double y) {
  double ax = fabs(x), ay = fabs(y);
  const bool sw = ay > ax;
  if (sw) { double t = ax; ax = ay; ay = t; }
  {  // scale to ax in [1/2, 1) so that TwoProd stays exact for subnormal / huge inputs
    const int e = frexp_exp(ax);
    ax = ldexp_fast(ax, -e);
    ay = ldexp_fast(ay, -e);
  }
  // table index round(128 ay/ax): only needs to be nearly right (|u| stays ~2^-8, far inside the series'
  // range), so one fp32 division on the device instead of an fp64 one
#ifdef __CUDA_ARCH__
  const int j = min(128, __float2int_rn(__fdividef((float)ay, (float)ax) * 128.0f));
#else
  const int j = fpe_d2i_rn(fpe_div(ay, ax) * 128.0);        // 0..128
#endif
  const double c = (double)j * 0.0078125;
  // u = (ay - c ax) / (ax + c ay), atan(ay/ax) = atan(c) + atan(u), |u| <= 2^-8
  dd_t pc = two_prod(c, ax);
  dd_t num = two_sum(fpe_sub(ay, pc.hi), -pc.lo);          // ay - pc.hi exact (Sterbenz, j >= 1)
  dd_t qc = two_prod(c, ay);
  dd_t den = two_sum(ax, qc.hi);
  den = fast_two_sum(den.hi, fpe_add(den.lo, qc.lo));
  // u = num / den as uh + ul: uh from a reciprocal good to ~2^-46 (device: fp32 rcp + one Newton step),
  // the exact remainder, and ul = remainder / den at the same accuracy -- |uh + ul - u| ~ 2^-92 |u|
#ifdef __CUDA_ARCH__
  const double rd0 = (double)__frcp_rn((float)den.hi);
  const double rd = fpe_fma(rd0, fpe_fma(-den.hi, rd0, 1.0), rd0);
  const double uh = fpe_mul(num.hi, rd);
#else
  const double rd = fpe_div(1.0, den.hi);
  const double uh = fpe_div(num.hi, den.hi);
#endif
  double rr = fpe_fma(-uh, den.hi, num.hi);                 // exact remainder
  rr = fpe_add(rr, fpe_fma(-uh, den.lo, num.lo));
  const double ul = fpe_mul(rr, rd);
  const double s = fpe_mul(uh, uh);
  double R = -1.0 / 11.0;
  R = fpe_fma(R, s, 1.0 / 9.0);
  R = fpe_fma(R, s, -1.0 / 7.0);
  R = fpe_fma(R, s, 1.0 / 5.0);
  R = fpe_fma(R, s, -1.0 / 3.0);
  dd_t at = fast_two_sum(uh, fpe_fma(fpe_mul(uh, s), R, ul));
  dd_t tu = dd_mul(at, dd_t{FPE_INV_2PI_HI, FPE_INV_2PI_LO});
  dd_t a = two_sum(fpe_atantab(j, 0), tu.hi);
  tu = fast_two_sum(a.hi, fpe_add(a.lo, fpe_add(fpe_atantab(j, 1), tu.lo)));   // [0, 1/8]
  if (sw) { dd_t b = two_sum(0.25, -tu.hi); tu = fast_two_sum(b.hi, fpe_sub(b.lo, tu.lo)); }
  if (x < 0.0) { dd_t b = two_sum(0.5, -tu.hi); tu = fast_two_sum(b.hi, fpe_sub(b.lo, tu.lo)); }
  if (y < 0.0) { tu.hi = -tu.hi; tu.lo = -tu.lo; }
  return tu;
}

// 2^g e^(2 pi i f) pieces: both g and f in about [-1/2, 1/2].
FPE_HD void exp2_cis(double g, double f, double& c, double& s, double& m) {
#ifdef __CUDA_ARCH__
  m = exp2(g);
  sincospi(2.0 * f, &s, &c);
#else
  m = std::exp2(g);
  const long double ang = 2.0L * 3.14159265358979323846264338327950288L * (long double)f;
  s = (double)sinl(ang);
  c = (double)cosl(ang);
#endif
}

// z^n (n >= 0) for z = 2^lambda e^(2 pi i tau): (hr + i hi) 2^E, hr/hi within ~2^-50 relative.
FPE_HD xc_t pow_polar(dd_t lam, dd_t tau, long long n) {
  xc_t v;
  v.hr = 1.0; v.hi = 0.0; v.er = 0.0; v.ei = 0.0; v.E = 0;
  if (n <= 0) return v;
  const double dn = (double)n;
  dd_t m = two_prod(dn, lam.hi);
  const double E = rint(m.hi);
  const double g = fpe_add(fpe_sub(m.hi, E), fpe_fma(dn, lam.lo, m.lo));
  dd_t a = two_prod(dn, tau.hi);
  const double k = rint(a.hi);
  const double f = fpe_add(fpe_sub(a.hi, k), fpe_fma(dn, tau.lo, a.lo));
  double c, s, mod;
  exp2_cis(g, f, c, s, mod);
  v.hr = fpe_mul(c, mod);
  v.hi = fpe_mul(s, mod);
  v.E = (long long)E;
  return v;
}

// Real z = sign 2^lambda: z^n = (+-1) 2^(n lambda).
FPE_HD xr_t pow_polar_real(dd_t lam, bool negative, long long n) {
  xr_t v{1.0, 0.0, 0};
  if (n <= 0) return v;
  const double dn = (double)n;
  dd_t m = two_prod(dn, lam.hi);
  const double E = rint(m.hi);
  const double g = fpe_add(fpe_sub(m.hi, E), fpe_fma(dn, lam.lo, m.lo));
#ifdef __CUDA_ARCH__
  const double mod = exp2(g);
#else
  const double mod = std::exp2(g);
#endif
  v.h = (negative && (n & 1)) ? -mod : mod;
  v.E = (long long)E;
  return v;
}

// Per-point polar data for repeated powers.
struct polar_t { dd_t lam, tau; bool neg; };

template <bool CPLX>
FPE_HD polar_t polar_of(double x, double y) {
  polar_t p;
  p.lam = log2abs_quick(x, y, CPLX);
  p.neg = x < 0.0;
  if constexpr (CPLX) p.tau = atan2_turns(x, y);
  else p.tau = dd_t{0.0, 0.0};
  return p;
}

}  // namespace fpe
