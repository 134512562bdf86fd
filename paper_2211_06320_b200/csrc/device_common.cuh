// device_common.cuh -- device helpers shared by the FPE kernels (point/coefficient access,
// exact classification searches, extended-range output).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>
#include "fpe_internal.h"
#include "fpe_math.cuh"

namespace fpe {

// ------------------------------------------------------------------------------------------
// point / coefficient access
template <int PK> struct PtTraits;
template <> struct PtTraits<FPE_R64> { static constexpr bool cplx = false; static constexpr bool f32 = false; };
template <> struct PtTraits<FPE_C64> { static constexpr bool cplx = true; static constexpr bool f32 = false; };
template <> struct PtTraits<FPE_R32> { static constexpr bool cplx = false; static constexpr bool f32 = true; };
template <> struct PtTraits<FPE_C32> { static constexpr bool cplx = true; static constexpr bool f32 = true; };

template <int PK>
__device__ __forceinline__ void load_point(const void* __restrict__ p, long long i, double& x, double& y) {
  if constexpr (PK == FPE_R64) { x = __ldg(static_cast<const double*>(p) + i); y = 0.0; }
  else if constexpr (PK == FPE_C64) { double2 v = __ldg(static_cast<const double2*>(p) + i); x = v.x; y = v.y; }
  else if constexpr (PK == FPE_R32) { x = (double)__ldg(static_cast<const float*>(p) + i); y = 0.0; }
  else { float2 v = __ldg(static_cast<const float2*>(p) + i); x = (double)v.x; y = (double)v.y; }
}

// ------------------------------------------------------------------------------------------
// classification: exact searches on the cover (fpe_math.cuh sign_lin).
//
// f(k) = cover(k) + lambda k - (N - D),  N = hh_i* + lambda hk_i*  (eq:defN, def:LRN).
// At a vertex j:      f >= 0  <=>  lambda (hk_j - hk_i*) + (hh_j - hh_i* + D) >= 0
// Inside segment s:   f >= 0  <=>  lambda (k - hk_i*) dk_s + (hh_s - hh_i* + D) dk_s + dh_s (k - hk_s) >= 0
__device__ __forceinline__ bool band_vertex(const int2* hull, int j, int2 vs, int drop, double lam) {
  int2 v = hull[j];
  return sign_lin(lam, (long long)v.x - vs.x, (long long)v.y - vs.y + drop) >= 0;
}
// lambda policies for the searches.  LamExact: the correctly rounded lambda, every predicate is the exact
// sign of lambda I + J.  LamIv: an enclosure [lo, hi] of the exact log2|z| (and so of its rounding);
// lambda I + J is monotone in lambda, so a predicate is decided for every lambda of the enclosure when
// both ends agree -- otherwise `amb` is set and the caller redoes the search with the rounded lambda.
struct LamExact {
  double l;
  __device__ __forceinline__ double mid() const { return l; }
  __device__ __forceinline__ bool ge0(double I, double J) const { return __fma_rn(l, I, J) >= 0.0; }
  __device__ __forceinline__ bool le0(double I, double J) const { return __fma_rn(l, I, J) <= 0.0; }
};
struct LamIv {
  double lo, hi;
  bool* amb;
  __device__ __forceinline__ double mid() const { return 0.5 * (lo + hi); }
  __device__ __forceinline__ bool ge0(double I, double J) const {
    const bool a = __fma_rn(lo, I, J) >= 0.0, b = __fma_rn(hi, I, J) >= 0.0;
    if (a != b) *amb = true;
    return a;
  }
  __device__ __forceinline__ bool le0(double I, double J) const {
    const bool a = __fma_rn(lo, I, J) <= 0.0, b = __fma_rn(hi, I, J) <= 0.0;
    if (a != b) *amb = true;
    return a;
  }
};

// The same predicate in doubles: exact when every |I|, |J| < 2^53 (PolyDev::dbl_ok, checked per polynomial):
// the products are exact integers and the fused multiply-add rounds lambda I + J once.
template <typename L>
__device__ __forceinline__ bool band_seg_dp(int2 a, int2 b, int2 vs, int drop, const L& pl, long long k) {
  const double dk = (double)(b.x - a.x), dh = (double)(b.y - a.y);
  const double J = __fma_rn(dh, (double)(k - a.x), (double)(a.y - vs.y + drop) * dk);
  const double I = (double)(k - vs.x) * dk;
  return pl.ge0(I, J);
}
__device__ __forceinline__ bool band_seg_d(int2 a, int2 b, int2 vs, int drop, double lam, long long k) {
  return band_seg_dp(a, b, vs, drop, LamExact{lam}, k);
}
__device__ __forceinline__ bool band_seg(int2 a, int2 b, int2 vs, int drop, double lam, long long k) {
  long long dk = (long long)b.x - a.x, dh = (long long)b.y - a.y;
  long long J = ((long long)a.y - vs.y + drop) * dk + dh * (k - a.x);
  long long I = (k - vs.x) * dk;
  return sign_lin(lam, I, J) >= 0;
}

// 1/c for the boundary estimates below: the fp32 reciprocal refined by one Newton step in fp64 (relative
// error ~2^-46; an IEEE division costs a subroutine of ~40 instructions).  The estimate only seeds the
// exact predicate tests, which correct any error (and fall back to bisection), so the result is exact
// whatever the estimate.
__device__ __forceinline__ double rcp_est(double c) {
  const double r = (double)__frcp_rn((float)c);
  return fma(r, fma(-c, r, 1.0), r);
}

// Least k in [lo, hi] with band_seg(A, B, ...) true, given that it holds at hi and the predicate
// is monotone on the segment (left branch: increasing).  The sheared cover is affine on the
// segment, F(k) = c0 + c1 k, so the crossing is estimated in fp64 and then verified exactly.
template <bool DBL = false>
__device__ __forceinline__ long long seg_first_true(int2 A, int2 B, int2 vs, int drop, double lam,
                                                    long long lo, long long hi) {
  // F(A.x + t) = dk g + t c1,  g = (A.y - vs.y + D) + lambda (A.x - vs.x),  c1 = dh + lambda dk
  const double dk = (double)(B.x - A.x), dh = (double)(B.y - A.y);
  const double c1 = __fma_rn(lam, dk, dh);                       // > 0 on the left branch
  const double g = __fma_rn(lam, (double)(A.x - vs.x), (double)(A.y - vs.y + drop));
  long long k = hi;
  if (c1 > 0.0) {
    double e = (double)A.x + ceil(-(g * dk) * rcp_est(c1));
    if (e >= (double)lo && e <= (double)hi) k = (long long)e;
    else if (e < (double)lo) k = lo;
  }
  // exact adjustment; a bounded number of steps, else bisection
  for (int it = 0; it < 4; ++it) {
    const bool t = (DBL ? band_seg_d(A, B, vs, drop, lam, k) : band_seg(A, B, vs, drop, lam, k));
    if (t) {
      if (k == lo || !(DBL ? band_seg_d(A, B, vs, drop, lam, k - 1) : band_seg(A, B, vs, drop, lam, k - 1))) return k;
      --k;
    } else {
      ++k;
    }
  }
  long long a = lo, b = hi;
  while (a < b) { long long m = (a + b) >> 1; if ((DBL ? band_seg_d(A, B, vs, drop, lam, m) : band_seg(A, B, vs, drop, lam, m))) b = m; else a = m + 1; }
  return a;
}
// Greatest k in [lo, hi] with the predicate true, given that it holds at lo (right branch: decreasing).
template <bool DBL = false>
__device__ __forceinline__ long long seg_last_true(int2 A, int2 B, int2 vs, int drop, double lam,
                                                   long long lo, long long hi) {
  const double dk = (double)(B.x - A.x), dh = (double)(B.y - A.y);
  const double c1 = __fma_rn(lam, dk, dh);                       // < 0 on the right branch
  const double g = __fma_rn(lam, (double)(A.x - vs.x), (double)(A.y - vs.y + drop));
  long long k = lo;
  if (c1 < 0.0) {
    double e = (double)A.x + floor(-(g * dk) * rcp_est(c1));
    if (e >= (double)lo && e <= (double)hi) k = (long long)e;
    else if (e > (double)hi) k = hi;
  }
  for (int it = 0; it < 4; ++it) {
    const bool t = (DBL ? band_seg_d(A, B, vs, drop, lam, k) : band_seg(A, B, vs, drop, lam, k));
    if (t) {
      if (k == hi || !(DBL ? band_seg_d(A, B, vs, drop, lam, k + 1) : band_seg(A, B, vs, drop, lam, k + 1))) return k;
      ++k;
    } else {
      --k;
    }
  }
  long long a = lo, b = hi;
  while (a < b) { long long m = (a + b + 1) >> 1; if ((DBL ? band_seg_d(A, B, vs, drop, lam, m) : band_seg(A, B, vs, drop, lam, m))) a = m; else b = m - 1; }
  return a;
}

// seg_first_true / seg_last_true for a lambda policy (predicates in exact doubles: PolyDev::dbl_ok).
template <typename L>
__device__ __forceinline__ long long seg_first_true_p(int2 A, int2 B, int2 vs, int drop, const L& pl,
                                                      long long lo, long long hi) {
  const double lam = pl.mid();
  const double dk = (double)(B.x - A.x), dh = (double)(B.y - A.y);
  const double c1 = __fma_rn(lam, dk, dh);
  const double g = __fma_rn(lam, (double)(A.x - vs.x), (double)(A.y - vs.y + drop));
  long long k = hi;
  if (c1 > 0.0) {
    double e = (double)A.x + ceil(-(g * dk) * rcp_est(c1));
    if (e >= (double)lo && e <= (double)hi) k = (long long)e;
    else if (e < (double)lo) k = lo;
  }
  for (int it = 0; it < 4; ++it) {
    if (band_seg_dp(A, B, vs, drop, pl, k)) {
      if (k == lo || !band_seg_dp(A, B, vs, drop, pl, k - 1)) return k;
      --k;
    } else {
      ++k;
    }
  }
  long long a = lo, b = hi;
  while (a < b) { long long m = (a + b) >> 1; if (band_seg_dp(A, B, vs, drop, pl, m)) b = m; else a = m + 1; }
  return a;
}
template <typename L>
__device__ __forceinline__ long long seg_last_true_p(int2 A, int2 B, int2 vs, int drop, const L& pl,
                                                     long long lo, long long hi) {
  const double lam = pl.mid();
  const double dk = (double)(B.x - A.x), dh = (double)(B.y - A.y);
  const double c1 = __fma_rn(lam, dk, dh);
  const double g = __fma_rn(lam, (double)(A.x - vs.x), (double)(A.y - vs.y + drop));
  long long k = lo;
  if (c1 < 0.0) {
    double e = (double)A.x + floor(-(g * dk) * rcp_est(c1));
    if (e >= (double)lo && e <= (double)hi) k = (long long)e;
    else if (e > (double)hi) k = hi;
  }
  for (int it = 0; it < 4; ++it) {
    if (band_seg_dp(A, B, vs, drop, pl, k)) {
      if (k == hi || !band_seg_dp(A, B, vs, drop, pl, k + 1)) return k;
      ++k;
    } else {
      --k;
    }
  }
  long long a = lo, b = hi;
  while (a < b) { long long m = (a + b + 1) >> 1; if (band_seg_dp(A, B, vs, drop, pl, m)) a = m; else b = m - 1; }
  return a;
}

__device__ __forceinline__ void classify_lambda(const int2* hull, int nv, int drop, double lam,
                                                int& istar, int& l, int& r) {
  if (isnan(lam)) { istar = -1; l = 0; r = -1; return; }
  if (lam == -INFINITY) { istar = 0; l = r = hull[0].x; return; }
  const int m = nv - 1;
  // k_lambda: least i in [0, m) with lambda dk_i + dh_i <= 0 (slopes decreasing), else m.
  int a = 0, b = m;
  while (a < b) {
    int i = (a + b) >> 1;
    int2 v0 = hull[i], v1 = hull[i + 1];
    if (sign_lin(lam, (long long)v1.x - v0.x, (long long)v1.y - v0.y) <= 0) b = i; else a = i + 1;
  }
  istar = a;
  const int2 vs = hull[a];
  // l: least vertex in [0, i*] inside the band, then the least integer in the segment before it.
  a = 0; b = istar;
  while (a < b) { int j = (a + b) >> 1; if (band_vertex(hull, j, vs, drop, lam)) b = j; else a = j + 1; }
  if (a == 0) {
    l = hull[0].x;
  } else {
    int2 A = hull[a - 1], B = hull[a];   // f(A) < 0 <= f(B)
    l = (int)seg_first_true(A, B, vs, drop, lam, (long long)A.x + 1, (long long)B.x);
  }
  // r: greatest vertex in [i*, m] inside the band, then the greatest integer in the segment after it.
  a = istar; b = m;
  while (a < b) { int j = (a + b + 1) >> 1; if (band_vertex(hull, j, vs, drop, lam)) a = j; else b = j - 1; }
  if (a == m) {
    r = hull[m].x;
  } else {
    int2 A = hull[a], B = hull[a + 1];   // f(A) >= 0 > f(B)
    r = (int)seg_last_true(A, B, vs, drop, lam, (long long)A.x, (long long)B.x - 1);
  }
}

// The same searches with the cover vertices also staged as doubles hv[i] = (hk_i, hh_i): every vertex
// predicate is then one fused multiply-add on exactly representable operands (|hk|, |hh| < 2^31), whose
// single rounding preserves the sign of lambda I + J -- no integer products or conversions in the loops.
template <bool DBL>
__device__ __forceinline__ void classify_lambda_v(const int2* hull, const double2* hv, int nv, int drop, double lam,
                                                  int& istar, int& l, int& r) {
  if (isnan(lam)) { istar = -1; l = 0; r = -1; return; }
  if (lam == -INFINITY) { istar = 0; l = r = hull[0].x; return; }
  const int m = nv - 1;
  int a = 0, b = m;
  while (a < b) {
    const int i = (a + b) >> 1;
    const double2 v0 = hv[i], v1 = hv[i + 1];
    if (__fma_rn(lam, v1.x - v0.x, v1.y - v0.y) <= 0.0) b = i; else a = i + 1;
  }
  istar = a;
  const double2 vs = hv[a];
  const double Dd = (double)drop;
  a = 0; b = istar;
  while (a < b) {
    const int j = (a + b) >> 1;
    const double2 v = hv[j];
    if (__fma_rn(lam, v.x - vs.x, (v.y - vs.y) + Dd) >= 0.0) b = j; else a = j + 1;
  }
  const int2 vsi = hull[istar];
  if (a == 0) {
    l = hull[0].x;
  } else {
    const int2 A = hull[a - 1], B = hull[a];
    l = (int)seg_first_true<DBL>(A, B, vsi, drop, lam, (long long)A.x + 1, (long long)B.x);
  }
  a = istar; b = m;
  while (a < b) {
    const int j = (a + b + 1) >> 1;
    const double2 v = hv[j];
    if (__fma_rn(lam, v.x - vs.x, (v.y - vs.y) + Dd) >= 0.0) a = j; else b = j - 1;
  }
  if (a == m) {
    r = hull[m].x;
  } else {
    const int2 A = hull[a], B = hull[a + 1];
    r = (int)seg_last_true<DBL>(A, B, vsi, drop, lam, (long long)A.x, (long long)B.x - 1);
  }
}

// The vertex searches of classify_lambda_v for a lambda policy (finite lambda; predicates in doubles).
// Most points lie beyond the extreme cover slopes and have narrow bands, so k_lambda tests the two end
// slopes before bisecting, and the band's end vertices are found by galloping outward from i*
// (1, 2, 4, ... vertices, then bisection inside the last step): a narrow band costs one test per side.
template <typename L>
__device__ __forceinline__ void classify_lambda_vp(const int2* hull, const double2* hv, int nv, int drop, const L& pl,
                                                   int& istar, int& l, int& r) {
  const int m = nv - 1;
  int a = 0, b = m;   // least i in [0, m) with lambda dk_i + dh_i <= 0, else m
  if (m > 0) {
    const double2 v0 = hv[0], v1 = hv[1];
    if (pl.le0(v1.x - v0.x, v1.y - v0.y)) {
      b = 0;
    } else {
      a = 1;
      if (m > 1) {
        const double2 w0 = hv[m - 1], w1 = hv[m];
        if (pl.le0(w1.x - w0.x, w1.y - w0.y)) b = m - 1; else a = m;
      }
    }
  }
  while (a < b) {
    const int i = (a + b) >> 1;
    const double2 v0 = hv[i], v1 = hv[i + 1];
    if (pl.le0(v1.x - v0.x, v1.y - v0.y)) b = i; else a = i + 1;
  }
  istar = a;
  const double2 vs = hv[a];
  const double Dd = (double)drop;
  auto band = [&](int j) { const double2 v = hv[j]; return pl.ge0(v.x - vs.x, (v.y - vs.y) + Dd); };
  int t = istar, f = -1;   // least vertex in the band: band(t) true, band(f) false (f = -1: none)
  for (int st = 1;; st <<= 1) {
    const int j = istar - st;
    if (j < 0) break;
    if (band(j)) t = j; else { f = j; break; }
  }
  while (t - f > 1) { const int mid = (f + t) >> 1; if (band(mid)) t = mid; else f = mid; }
  a = t;
  const int2 vsi = hull[istar];
  if (a == 0) {
    l = hull[0].x;
  } else {
    const int2 A = hull[a - 1], B = hull[a];
    l = (int)seg_first_true_p(A, B, vsi, drop, pl, (long long)A.x + 1, (long long)B.x);
  }
  t = istar; f = m + 1;    // greatest vertex in the band
  for (int st = 1;; st <<= 1) {
    const int j = istar + st;
    if (j > m) break;
    if (band(j)) t = j; else { f = j; break; }
  }
  while (f - t > 1) { const int mid = (t + f) >> 1; if (band(mid)) t = mid; else f = mid; }
  a = t;
  if (a == m) {
    r = hull[m].x;
  } else {
    const int2 A = hull[a], B = hull[a + 1];
    r = (int)seg_last_true_p(A, B, vsi, drop, pl, (long long)A.x, (long long)B.x - 1);
  }
}

__device__ __forceinline__ int lower_bound_i32(const int32_t* __restrict__ a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) { int m = (lo + hi) >> 1; if (__ldg(a + m) < key) lo = m + 1; else hi = m; }
  return lo;
}

__device__ __forceinline__ int kept_count(const PolyDev& P, int l, int r) {
  if (r < l) return 0;
  if (P.sparse) return lower_bound_i32(P.sidx, (int)P.n_good, r + 1) - lower_bound_i32(P.sidx, (int)P.n_good, l);
  if (P.all_good) return r - l + 1;
  return __ldg(P.prefix + (r + 1 - P.k_min)) - __ldg(P.prefix + (l - P.k_min));
}

// ------------------------------------------------------------------------------------------
// output: mantissa normalised to max(|re|,|im|) in [1/2, 1), exponent int64
template <int OK>   // output kind = fpe_dtype of the values
__device__ __forceinline__ void store_value(void* __restrict__ vals, long long* __restrict__ exps, long long i,
                                            double re, double im, long long E) {
  double m = fmax(fabs(re), fabs(im));
  if (m == 0.0 || !isfinite(m)) {
    E = 0;
  } else {
    int e = frexp_exp(m);
    re = ldexp_fast(re, -e); im = ldexp_fast(im, -e);
    E += e;
  }
  if (!exps) {   // plain floats: value * 2^E, saturating
    int Ec = (int)max(-4000ll, min(4000ll, E));
    re = ldexp(re, Ec); im = ldexp(im, Ec);
  } else {
    exps[i] = E;
  }
  if constexpr (OK == FPE_R64) static_cast<double*>(vals)[i] = re;
  else if constexpr (OK == FPE_C64) static_cast<double2*>(vals)[i] = make_double2(re, im);
  else if constexpr (OK == FPE_R32) static_cast<float*>(vals)[i] = (float)re;
  else static_cast<float2*>(vals)[i] = make_float2((float)re, (float)im);
}

template <int CK> struct Coef;
template <int CK> __device__ void a0_value(const PolyDev& P, double& re, double& im);
template <> struct Coef<FPE_C64> {
  using T = double2;
  __device__ static void get(const void* c, long long k, double& re, double& im) {
    double2 v = __ldg(static_cast<const double2*>(c) + k); re = v.x; im = v.y;
  }
};
template <> struct Coef<FPE_R64> {
  using T = double;
  __device__ static void get(const void* c, long long k, double& re, double& im) {
    re = __ldg(static_cast<const double*>(c) + k); im = 0.0;
  }
};
template <> struct Coef<FPE_C32> {
  using T = float2;
  __device__ static void get(const void* c, long long k, float& re, float& im) {
    float2 v = __ldg(static_cast<const float2*>(c) + k); re = v.x; im = v.y;
  }
};
template <> struct Coef<FPE_R32> {
  using T = float;
  __device__ static void get(const void* c, long long k, float& re, float& im) {
    re = __ldg(static_cast<const float*>(c) + k); im = 0.0f;
  }
};

// a_0 2^-shift (0 if a_0 = 0): the value at z = 0 (the lambda -> -inf limit).
template <int CK> __device__ void a0_value(const PolyDev& P, double& re, double& im) {
  re = 0.0; im = 0.0;
  if (P.k_min != 0) return;
  if (P.sparse && __ldg(P.sidx) != 0) return;
  if constexpr (PtTraits<CK>::f32) { float a, b; Coef<CK>::get(P.coef, 0, a, b); re = a; im = b; }
  else Coef<CK>::get(P.coef, 0, re, im);
}

// Q = b * z^n with b in the working precision and z^n extended (fpe_math.cuh xc_pow).
template <bool CPLX>
__device__ __forceinline__ void times_zpow(double br, double bi, double x, double y, long long n,
                                           double& qr, double& qi, long long& E) {
  if constexpr (CPLX) {
    xc_t zp = xc_pow(x, y, n);
    qr = __fma_rn(br, zp.hr, __fma_rn(-bi, zp.hi, __fma_rn(br, zp.er, -bi * zp.ei)));
    qi = __fma_rn(br, zp.hi, __fma_rn(bi, zp.hr, __fma_rn(br, zp.ei, bi * zp.er)));
    E = zp.E;
  } else {
    xr_t zp = xr_pow(x, n);
    qr = __fma_rn(br, zp.h, br * zp.e);
    qi = 0.0;
    E = zp.E;
  }
}

}  // namespace fpe
