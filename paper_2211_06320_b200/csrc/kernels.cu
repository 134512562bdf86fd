// kernels.cu -- sm_100a kernels of the FPE hot path.
//
//   k_classify     lines 5-8 of Algorithm FPE_p: lambda = log2|z| (correctly
//                  rounded, fpe_math.cuh), k_lambda by binary search over the cover slopes staged in
//                  shared memory, [l, r] by binary searches with exact predicates.
//   k_eval_point   line 9: Q_lambda(z) = z^l * Horner over G_p cap [l, r]
//                  (PAPER.md:1621-1622), one thread per point; the reference path of the tiled
//                  evaluator and the path for sparse handles.
//   k_horner_full  Horner's scheme over the whole coefficient range with
//                  in-loop exponent rescaling -- the context baseline.
#include <cuda_runtime.h>
#include <cstdint>
#include "fpe_internal.h"
#include "fpe_math.cuh"
#include "kernels.cuh"

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
__device__ __forceinline__ bool band_seg(int2 a, int2 b, int2 vs, int drop, double lam, long long k) {
  long long dk = (long long)b.x - a.x, dh = (long long)b.y - a.y;
  long long J = ((long long)a.y - vs.y + drop) * dk + dh * (k - a.x);
  long long I = (k - vs.x) * dk;
  return sign_lin(lam, I, J) >= 0;
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
    int2 A = hull[a - 1], B = hull[a];
    long long lo = A.x + 1, hi = B.x;   // f(A) < 0 <= f(B)
    while (lo < hi) { long long k = (lo + hi) >> 1; if (band_seg(A, B, vs, drop, lam, k)) hi = k; else lo = k + 1; }
    l = (int)lo;
  }
  // r: greatest vertex in [i*, m] inside the band, then the greatest integer in the segment after it.
  a = istar; b = m;
  while (a < b) { int j = (a + b + 1) >> 1; if (band_vertex(hull, j, vs, drop, lam)) a = j; else b = j - 1; }
  if (a == m) {
    r = hull[m].x;
  } else {
    int2 A = hull[a], B = hull[a + 1];
    long long lo = A.x, hi = B.x - 1;   // f(A) >= 0 > f(B)
    while (lo < hi) { long long k = (lo + hi + 1) >> 1; if (band_seg(A, B, vs, drop, lam, k)) lo = k; else hi = k - 1; }
    r = (int)lo;
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

template <int PK>
__global__ void __launch_bounds__(256) k_classify(const void* __restrict__ pts, long long n, PolyDev P,
                                                  int2* __restrict__ lr, fpe_diag* __restrict__ diag,
                                                  unsigned long long* __restrict__ hard_ctr) {
  extern __shared__ int2 s_hull[];
  const int2* hull = P.hull;
  if (P.nv <= kSmemHullMax) {
    for (int i = threadIdx.x; i < P.nv; i += blockDim.x) s_hull[i] = P.hull[i];
    __syncthreads();
    hull = s_hull;
  }
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double x, y;
    load_point<PK>(pts, i, x, y);
    int hard;
    double lam = lambda_cr(x, y, PtTraits<PK>::cplx, &hard);
    int istar, l, r;
    classify_lambda(hull, P.nv, P.drop, lam, istar, l, r);
    lr[i] = make_int2(l, r);
    if (diag) {
      fpe_diag d;
      d.lambda = lam; d.region = istar; d.l = l; d.r = r;
      d.kept = kept_count(P, l, r); d.hard = hard; d.pad = 0;
      diag[i] = d;
    }
    if (hard) atomicAdd(hard_ctr, 1ull);
  }
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
    re = ldexp(re, -e); im = ldexp(im, -e);
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

// One thread per point: Q_lambda(z) = z^l sum_{k in G_p cap [l,r]} a_k z^(k-l).
template <int PK, int CK, int OK>
__global__ void __launch_bounds__(128) k_eval_point(const void* __restrict__ pts, long long n, PolyDev P,
                                                    const int2* __restrict__ lr, void* __restrict__ vals,
                                                    long long* __restrict__ exps) {
  constexpr bool CPLX = PtTraits<OK>::cplx;
  constexpr bool F32 = PtTraits<CK>::f32;
  using W = typename std::conditional<F32, float, double>::type;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double x, y;
    load_point<PK>(pts, i, x, y);
    int2 w = lr[i];
    if (w.y < w.x) {   // non-finite point
      double nan = __longlong_as_double(0x7ff8000000000000LL);
      store_value<OK>(vals, exps, i, nan, CPLX ? nan : 0.0, 0);
      continue;
    }
    if (x == 0.0 && y == 0.0) {   // z = 0: P(0) = a_0
      double cr, ci;
      a0_value<CK>(P, cr, ci);
      store_value<OK>(vals, exps, i, cr, ci, cr == 0 && ci == 0 ? 0 : P.shift);
      continue;
    }
    const W zr = (W)x, zi = (W)y;
    W br = 0, bi = 0;
    long long base;   // Q = b * z^base
    if (!P.sparse) {
      const long long off = P.k_min;
      for (long long k = w.y; k >= w.x; --k) {
        W cr, ci;
        Coef<CK>::get(P.coef, k - off, cr, ci);
        if constexpr (CPLX) {
          W t = fma(br, zr, fma(-bi, zi, cr));
          bi = fma(br, zi, fma(bi, zr, ci));
          br = t;
        } else {
          br = fma(br, zr, cr);
        }
      }
      base = w.x;
    } else {
      // Horner over the compact good list with gap powers z^(k_{j+1} - k_j)
      int jlo = lower_bound_i32(P.sidx, (int)P.n_good, w.x);
      int jhi = lower_bound_i32(P.sidx, (int)P.n_good, w.y + 1) - 1;
      base = w.x;
      if (jlo <= jhi) {
        Coef<CK>::get(P.coef, jhi, br, bi);
        for (int j = jhi - 1; j >= jlo; --j) {
          long long gap = (long long)__ldg(P.sidx + j + 1) - __ldg(P.sidx + j);
          double gr, gi;
          long long gE;
          times_zpow<CPLX>((double)br, (double)bi, x, y, gap, gr, gi, gE);
          // b_{j+1} z^gap = b_j - c_j is bounded by K 2^D (cover argument)
          int sc = (int)max(-3000ll, min(3000ll, gE));
          W cr, ci;
          Coef<CK>::get(P.coef, j, cr, ci);
          br = (W)ldexp(gr, sc) + cr;
          bi = (W)ldexp(gi, sc) + ci;
        }
        base = __ldg(P.sidx + jlo);
      }
    }
    double qr, qi;
    long long E;
    times_zpow<CPLX>((double)br, (double)bi, x, y, base, qr, qi, E);
    store_value<OK>(vals, exps, i, qr, qi, E + P.shift);
  }
}

// ------------------------------------------------------------------------------------------
// Full Horner with exponent tracking: value = b 2^E; z = w 2^ez with |w| in [1/2, sqrt 2).
template <int PK, int CK, int OK>
__global__ void __launch_bounds__(128) k_horner_full(const void* __restrict__ pts, long long n, PolyDev P,
                                                     void* __restrict__ vals, long long* __restrict__ exps) {
  constexpr bool CPLX = PtTraits<OK>::cplx;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double x, y;
    load_point<PK>(pts, i, x, y);
    if (!isfinite(x) || !isfinite(y)) {
      double nan = __longlong_as_double(0x7ff8000000000000LL);
      store_value<OK>(vals, exps, i, nan, CPLX ? nan : 0.0, 0);
      continue;
    }
    if (x == 0.0 && y == 0.0) {
      double cr, ci;
      a0_value<CK>(P, cr, ci);
      store_value<OK>(vals, exps, i, cr, ci, (cr == 0 && ci == 0) ? 0 : P.shift);
      continue;
    }
    const int ez = frexp_exp(fmax(fabs(x), fabs(y)));
    const double wr = ldexp(x, -ez), wi = ldexp(y, -ez);
    double br = 0.0, bi = 0.0;
    long long E = 0;
    const long long kmin = P.k_min;
    const long long cnt = P.sparse ? P.n_good : (P.k_max - P.k_min + 1);
    long long prevk = P.k_max;
    for (long long t = cnt - 1; t >= 0; --t) {
      long long k = P.sparse ? (long long)__ldg(P.sidx + t) : kmin + t;
      long long steps = prevk - k;   // multiply by z^(prevk - k) (1 for dense)
      prevk = k;
      if (steps == 1) {
        E += ez;
        double t2 = __fma_rn(br, wr, -bi * wi);
        bi = __fma_rn(br, wi, bi * wr);
        br = t2;
      } else if (steps > 1) {
        double qr, qi; long long qE;
        times_zpow<CPLX>(br, bi, x, y, steps, qr, qi, qE);
        br = qr; bi = qi; E += qE;
      }
      double cr, ci;
      if constexpr (PtTraits<CK>::f32) { float a, b; Coef<CK>::get(P.coef, t, a, b); cr = a; ci = b; }
      else Coef<CK>::get(P.coef, t, cr, ci);
      if (cr != 0.0 || ci != 0.0) {
        if (br == 0.0 && bi == 0.0) { E = 0; }
        if (-E > 1000) { br = ldexp(br, (int)max(E, -3000ll)); bi = ldexp(bi, (int)max(E, -3000ll)); E = 0; }
        if (-E >= -1000) { double f = ldexp(1.0, (int)-E); br = __fma_rn(cr, f, br); bi = __fma_rn(ci, f, bi); }
      }
      double m = fmax(fabs(br), fabs(bi));
      if (m != 0.0) { int e = frexp_exp(m); double s = pow2i(-e); br *= s; bi *= s; E += e; }
      else E = 0;
    }
    double qr, qi; long long qE;
    times_zpow<CPLX>(br, bi, x, y, kmin, qr, qi, qE);
    store_value<OK>(vals, exps, i, qr, qi, E + qE + P.shift);
  }
}

// ------------------------------------------------------------------------------------------
// launchers
static int grid_for(long long n, int block) {
  long long g = (n + block - 1) / block;
  if (g > 148LL * 64) g = 148LL * 64;
  return (int)(g < 1 ? 1 : g);
}

template <int PK>
static void launch_classify_t(const void* pts, long long n, const PolyDev& P, int2* lr, fpe_diag* diag,
                              unsigned long long* hard, cudaStream_t s) {
  size_t smem = P.nv <= kSmemHullMax ? P.nv * sizeof(int2) : 0;
  k_classify<PK><<<grid_for(n, 256), 256, smem, s>>>(pts, n, P, lr, diag, hard);
}

void launch_classify(int pk, const void* pts, long long n, const PolyDev& P, int2* lr, fpe_diag* diag,
                     unsigned long long* hard, cudaStream_t s) {
  switch (pk) {
    case FPE_R64: launch_classify_t<FPE_R64>(pts, n, P, lr, diag, hard, s); break;
    case FPE_C64: launch_classify_t<FPE_C64>(pts, n, P, lr, diag, hard, s); break;
    case FPE_R32: launch_classify_t<FPE_R32>(pts, n, P, lr, diag, hard, s); break;
    default: launch_classify_t<FPE_C32>(pts, n, P, lr, diag, hard, s); break;
  }
}

template <int PK, int CK>
static void launch_eval_point_t(const void* pts, long long n, const PolyDev& P, const int2* lr, void* vals,
                                long long* exps, cudaStream_t s) {
  constexpr bool cplx = PtTraits<PK>::cplx || PtTraits<CK>::cplx;
  constexpr int OK = PtTraits<CK>::f32 ? (cplx ? FPE_C32 : FPE_R32) : (cplx ? FPE_C64 : FPE_R64);
  k_eval_point<PK, CK, OK><<<grid_for(n, 128), 128, 0, s>>>(pts, n, P, lr, vals, exps);
}

template <int PK, int CK>
static void launch_horner_t(const void* pts, long long n, const PolyDev& P, void* vals, long long* exps,
                            cudaStream_t s) {
  constexpr bool cplx = PtTraits<PK>::cplx || PtTraits<CK>::cplx;
  constexpr int OK = PtTraits<CK>::f32 ? (cplx ? FPE_C32 : FPE_R32) : (cplx ? FPE_C64 : FPE_R64);
  k_horner_full<PK, CK, OK><<<grid_for(n, 128), 128, 0, s>>>(pts, n, P, vals, exps);
}

#define FPE_DISPATCH_PC(FN, ...)                                                        \
  switch (pk * 4 + P.cdt) {                                                             \
    case FPE_R64 * 4 + FPE_R64: FN<FPE_R64, FPE_R64>(__VA_ARGS__); break;               \
    case FPE_R64 * 4 + FPE_C64: FN<FPE_R64, FPE_C64>(__VA_ARGS__); break;               \
    case FPE_C64 * 4 + FPE_R64: FN<FPE_C64, FPE_R64>(__VA_ARGS__); break;               \
    case FPE_C64 * 4 + FPE_C64: FN<FPE_C64, FPE_C64>(__VA_ARGS__); break;               \
    case FPE_R32 * 4 + FPE_R32: FN<FPE_R32, FPE_R32>(__VA_ARGS__); break;               \
    case FPE_R32 * 4 + FPE_C32: FN<FPE_R32, FPE_C32>(__VA_ARGS__); break;               \
    case FPE_C32 * 4 + FPE_R32: FN<FPE_C32, FPE_R32>(__VA_ARGS__); break;               \
    case FPE_C32 * 4 + FPE_C32: FN<FPE_C32, FPE_C32>(__VA_ARGS__); break;               \
    default: return false;                                                              \
  }

bool launch_eval_point(int pk, const void* pts, long long n, const PolyDev& P, const int2* lr, void* vals,
                       long long* exps, cudaStream_t s) {
  FPE_DISPATCH_PC(launch_eval_point_t, pts, n, P, lr, vals, exps, s)
  return true;
}

bool launch_horner(int pk, const void* pts, long long n, const PolyDev& P, void* vals, long long* exps,
                   cudaStream_t s) {
  FPE_DISPATCH_PC(launch_horner_t, pts, n, P, vals, exps, s)
  return true;
}

}  // namespace fpe
