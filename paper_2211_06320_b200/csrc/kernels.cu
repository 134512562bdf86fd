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
#include "device_common.cuh"
#include "kernels.cuh"

namespace fpe {

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
