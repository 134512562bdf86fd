// kernels.cu -- sm_100a kernels of the FPE hot path.
//
//   k_classify     lines 5-8 of Algorithm FPE_p: lambda = log2|z| (correctly
//                  rounded, fpe_math.cuh), k_lambda by binary search over the cover slopes staged in
//                  shared memory, [l, r] by binary searches with exact predicates.
//   k_eval_sparse  line 9 for sparse handles: the few kept terms a_k z^k of the compact
//                  good-index list, each z^k by the polar route, summed in extended range.
//   k_confidence   fpe_diag::cancel; k_newton: the Newton step of fpe_newton_step.
//   k_horner_full  Horner's scheme over the whole coefficient range with
//                  in-loop exponent rescaling -- the context baseline.
#include <cuda_runtime.h>
#include <cstdint>
#include <algorithm>
#include "fpe_internal.h"
#include "fpe_math.cuh"
#include "fpe_polar.cuh"
#include "device_common.cuh"
#include "kernels.cuh"

namespace fpe {

template <int PK>
__global__ void __launch_bounds__(256) k_classify(const void* __restrict__ pts, long long n, PolyDev P,
                                                  int2* __restrict__ lr, fpe_diag* __restrict__ diag,
                                                  unsigned long long* __restrict__ hard_ctr) {
  // the cover in shared memory, also as exact doubles when small (the fast path of k_classify_bucket:
  // searches on an fp64 enclosure of log2|z|, the correctly rounded lambda only for undecided points)
  extern __shared__ __align__(16) unsigned char s_cls[];
  const bool dbl = P.nv <= kSmemHullDbl;
  double2* hv = reinterpret_cast<double2*>(s_cls);
  int2* sh = reinterpret_cast<int2*>(s_cls + (dbl ? (size_t)P.nv * sizeof(double2) : 0));
  const int2* hull = P.hull;
  if (P.nv <= kSmemHullMax) {
    for (int i = threadIdx.x; i < P.nv; i += blockDim.x) {
      const int2 v = P.hull[i];
      sh[i] = v;
      if (dbl) hv[i] = make_double2((double)v.x, (double)v.y);
    }
    __syncthreads();
    hull = sh;
  }
  const long long stride = (long long)gridDim.x * blockDim.x;
  double xn = 0.0, yn = 0.0;   // the next iteration's point, loaded one iteration ahead
  if (blockIdx.x * (long long)blockDim.x + threadIdx.x < n) load_point<PK>(pts, blockIdx.x * (long long)blockDim.x + threadIdx.x, xn, yn);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    const double x = xn, y = yn;
    if (i + stride < n) load_point<PK>(pts, i + stride, xn, yn);
    int hard = 0;
    double lam = 0.0;
    int istar, l, r;
    bool done = false;
    if (dbl && P.dbl_ok && isfinite(x) && isfinite(y) && (x != 0.0 || (PtTraits<PK>::cplx && y != 0.0))) {
      double lo, hi;
      lambda_enclosure(x, y, PtTraits<PK>::cplx, lo, hi, lam);
      bool amb = false;
      classify_lambda_vp(hull, hv, P.nv, P.drop, LamIv{lo, hi, &amb}, istar, l, r);
      done = !amb;
      if (done && diag) lam = lambda_fast(x, y, PtTraits<PK>::cplx, &hard);
    }
    if (!done) {
      lam = lambda_fast(x, y, PtTraits<PK>::cplx, &hard);
      if (dbl && P.dbl_ok) classify_lambda_v<true>(hull, hv, P.nv, P.drop, lam, istar, l, r);
      else classify_lambda(hull, P.nv, P.drop, lam, istar, l, r);
    }
    lr[i] = make_int2(l, r);
    if (diag) {
      fpe_diag d;
      d.lambda = lam; d.region = istar; d.l = l; d.r = r;
      d.kept = kept_count(P, l, r); d.hard = hard; d.cancel = INT32_MIN; d.trusted = 0; d.err_exp = INT32_MIN; d.pad = 0;
      diag[i] = d;
    }
    if (hard) atomicAdd(hard_ctr, 1ull);
  }
}

// ------------------------------------------------------------------------------------------
// Sparse handles (compact good-index list): the kept terms of a window are few
// (cfg4: K ~ 1), so every term a_k z^k is formed directly with z^k by the polar route (one
// log2|z| / arg z per point, then ~one exp2 + sincospi per term; fpe_polar.cuh) and the terms are
// summed in extended range in increasing k.  The good indices are binary-searched in shared memory.
__device__ __forceinline__ void xadd(double& sr, double& si, long long& se, double tr, double ti, long long te) {
  if (tr == 0.0 && ti == 0.0) return;
  if (sr == 0.0 && si == 0.0) { sr = tr; si = ti; se = te; return; }
  if (te > se) { const long long d = te - se; const int s = (int)min(d, 2000ll); sr = ldexp_fast(sr, -s); si = ldexp_fast(si, -s); se = te; }
  else if (te < se) { const long long d = se - te; const int s = (int)min(d, 2000ll); tr = ldexp_fast(tr, -s); ti = ldexp_fast(ti, -s); }
  sr += tr; si += ti;
  const double m = fmax(fabs(sr), fabs(si));
  if (m != 0.0) { const int e = frexp_exp(m); sr = ldexp_fast(sr, -e); si = ldexp_fast(si, -e); se += e; }
}


// Points have very uneven kept counts (cfg4: mean 1.15, 96% with K = 1, up to all 4096 terms near |z| = 1),
// so a lane-per-point loop would run each warp for its longest point (round 1: 62% of the instructions at
// 1-7 active lanes).  Warps claim 32-point items from a work queue.  For points with K <= kSpLong the warp
// lays the kept terms out flat (exclusive scan of K over the lanes) and computes them round-robin over all
// 32 lanes (kSpRound at a time, into shared memory) -- each term a_k z^k by the polar route from its
// point's (lambda, tau), a pure function of (z, k) -- and every lane sums its own point's terms in
// increasing k in extended range.  A longer list is summed by the whole warp: lane t takes the terms
// t, t + 32, ... and a fixed tree combines the partials (one lane summing 4096 terms alone kept a chunk
// busy for 1.2 ms, twice the rest of the kernel).  Either way a point's result is the same whatever
// points share its warp.
constexpr int kSpWarps = 8;
constexpr int kSpRound = 64;    // terms per warp and round in shared memory
constexpr int kSpTab = kSparseTab;
#ifndef FPE_SP_GRAB
#define FPE_SP_GRAB 4
#endif
#ifndef FPE_SP_MINB
#define FPE_SP_MINB 4
#endif
constexpr int kSpGrab = FPE_SP_GRAB;
#ifndef FPE_SP_LONG
#define FPE_SP_LONG 32
#endif
constexpr int kSpLong = FPE_SP_LONG;   // kept lists longer than this are summed by the whole warp      // warp-items of 32 points claimed per atomic (dynamic work queue)
struct SpTerm { double r, i; long long e; };

template <int CK, bool CPLX>
__device__ __forceinline__ SpTerm sparse_term(const PolyDev& P, const polar_t& pz, int j, int k) {
  double cr, ci;
  if constexpr (PtTraits<CK>::f32) { float a, b; Coef<CK>::get(P.coef, j, a, b); cr = a; ci = b; }
  else Coef<CK>::get(P.coef, j, cr, ci);
  SpTerm t{cr, ci, 0};
  if (k == 0) return t;
  if constexpr (CPLX) {
    const xc_t p = pow_polar(pz.lam, pz.tau, k);
    t.r = __fma_rn(cr, p.hr, -ci * p.hi);
    t.i = __fma_rn(cr, p.hi, ci * p.hr);
    t.e = p.E;
  } else {
    const xr_t p = pow_polar_real(pz.lam, pz.neg, k);
    t.r = cr * p.h; t.i = 0.0; t.e = p.E;
  }
  return t;
}

// A bucket table over [k_min, k_max] (buckets of 2^tb indices): the first good index >= k lies in
// [tab[b], tab[b + 1]] for b = (k - k_min) >> tb, so each window bound costs a search over ~n_good / kSpTab
// entries instead of log2(n_good) steps.  Built once per call (one CTA).
__global__ void __launch_bounds__(1024) k_sparse_table(PolyDev P, int* __restrict__ tab) {
  int tb = 0;
  while (((P.k_max - P.k_min) >> tb) >= kSpTab) ++tb;
  const int nb = (int)((P.k_max - P.k_min) >> tb) + 1;
  const int ng = (int)P.n_good;
  if (threadIdx.x == 0) tab[kSpTab + 1] = 0;   // the evaluator's work-queue counter
  for (int b = threadIdx.x; b <= nb; b += blockDim.x) {
    const long long key = P.k_min + ((long long)b << tb);
    int lo = 0, hi = ng;
    while (lo < hi) { const int m = (lo + hi) >> 1; if ((long long)__ldg(P.sidx + m) < key) lo = m + 1; else hi = m; }
    tab[b] = lo;
  }
}

#ifdef FPE_ITEM_TRACE
// Debugging (build with -DFPE_ITEM_TRACE): per claimed chunk of k_eval_sparse_coop, {start ns, end ns,
// max K << 32 | sum K}.
__device__ unsigned long long fpe_sp_trace[1 << 20][3];
__device__ unsigned int fpe_sp_trace_n;
__device__ __forceinline__ unsigned long long sp_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

template <int PK, int CK, int OK>
__global__ void __launch_bounds__(kSpWarps * 32, FPE_SP_MINB) k_eval_sparse_coop(const void* __restrict__ pts, long long n, PolyDev P,
                                                                    const int2* __restrict__ lr,
                                                                    int* __restrict__ tab,
                                                                    void* __restrict__ vals,
                                                                    long long* __restrict__ exps) {
  constexpr bool CPLX = PtTraits<OK>::cplx;
  extern __shared__ __align__(16) unsigned char sp_smem[];
  SpTerm* terms = reinterpret_cast<SpTerm*>(sp_smem);                                              // [warps][kSpRound]
  polar_t* pol = reinterpret_cast<polar_t*>(sp_smem + sizeof(SpTerm) * kSpWarps * kSpRound);      // [warps][32]
  int* offs = reinterpret_cast<int*>(pol + kSpWarps * 32);                                         // [warps][33]
  int* firsts = offs + kSpWarps * 33;                                                              // [warps][32]
  const int32_t* __restrict__ sidx = P.sidx;       // read through L1 (16 KiB at cfg4)
  int tb = 0;                                      // the bucket table's shift (k_sparse_table)
  while (((P.k_max - P.k_min) >> tb) >= kSpTab) ++tb;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  SpTerm* T = terms + w * kSpRound;
  polar_t* PL = pol + w * 32;
  int* OF = offs + w * 33;
  int* FI = firsts + w * 32;
  // dynamic work queue: a warp claims kSpGrab warp-items at a time (kept counts are very uneven, and a
  // static split left the SMs idle for a third of the kernel waiting for the slowest ones)
  unsigned int* ctr = reinterpret_cast<unsigned int*>(tab + kSpTab + 1);
  const long long nchunks = ((n + 31) / 32 + kSpGrab - 1) / kSpGrab;
  for (;;) {
  unsigned int c = 0;
  if (lane == 0) c = atomicAdd(ctr, 1u);
  c = __shfl_sync(0xffffffffu, c, 0);
  if ((long long)c >= nchunks) break;
#ifdef FPE_ITEM_TRACE
  const unsigned long long tr_t0 = sp_gtimer();
  unsigned long long tr_info = 0;
#endif
  for (int sub = 0; sub < kSpGrab; ++sub) {
    const long long base = ((long long)c * kSpGrab + sub) * 32;
    if (base >= n) break;
    const long long i = base + lane;
    double x = 0.0, y = 0.0;
    int first = 0, K = 0, state = 0;   // state 0: sum of the kept terms; 1: non-finite z (NaN); 2: z = 0
    if (i < n) {
      load_point<PK>(pts, i, x, y);
      const int2 wv = lr[i];
      if (wv.y < wv.x) state = 1;
      else if (x == 0.0 && y == 0.0) state = 2;
      else {
        const int bl = (int)((wv.x - P.k_min) >> tb), br_ = (int)((wv.y - P.k_min) >> tb);
        int lo = __ldg(tab + bl), hi = __ldg(tab + bl + 1);           // first good index >= l
        while (lo < hi) { const int m = (lo + hi) >> 1; if (__ldg(sidx + m) < wv.x) lo = m + 1; else hi = m; }
        int lo2 = max(lo, __ldg(tab + br_)), hi2 = __ldg(tab + br_ + 1);   // first good index > r
        while (lo2 < hi2) { const int m = (lo2 + hi2) >> 1; if (__ldg(sidx + m) <= wv.y) lo2 = m + 1; else hi2 = m; }
        first = lo; K = lo2 - lo;
        if (K > 0) PL[lane] = polar_of<CPLX>(x, y);
      }
    }
    // points with long kept lists are summed by the whole warp (below); the rest lay their terms out flat
    const bool lng = K > kSpLong;
    const int Kf = lng ? 0 : K;
    int off = Kf;   // inclusive scan of the flat counts over the warp
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int v = __shfl_up_sync(0xffffffffu, off, o); if (lane >= o) off += v; }
    const int total = __shfl_sync(0xffffffffu, off, 31);
#ifdef FPE_ITEM_TRACE
    {
      const unsigned long long mk = __reduce_max_sync(0xffffffffu, (unsigned)K);
      tr_info = (max(tr_info >> 32, mk) << 32) | ((tr_info & 0xffffffffull) + (unsigned)__reduce_add_sync(0xffffffffu, (unsigned)K));
    }
#endif
    OF[lane + 1] = off;
    if (lane == 0) OF[0] = 0;
    FI[lane] = first;
    off -= Kf;   // exclusive
    __syncwarp();
    double sr = 0.0, si = 0.0;
    long long se = 0;
    for (int r0 = 0; r0 < total; r0 += kSpRound) {
      const int rn = min(kSpRound, total - r0);
      for (int f = lane; f < rn; f += 32) {   // flat term g = r0 + f: owner = the lane q with OF[q] <= g < OF[q+1]
        const int g = r0 + f;
        int a = 0, b = 31;
        while (a < b) { const int m = (a + b + 1) >> 1; if (OF[m] <= g) a = m; else b = m - 1; }
        const int j = FI[a] + (g - OF[a]);
        T[f] = sparse_term<CK, CPLX>(P, PL[a], j, __ldg(sidx + j));
      }
      __syncwarp();
      // this lane's terms inside the round, in increasing k (the flat order)
      const int t0 = max(off, r0), t1 = min(off + Kf, r0 + rn);
      for (int g = t0; g < t1; ++g) { const SpTerm t = T[g - r0]; xadd(sr, si, se, t.r, t.i, t.e); }
      __syncwarp();
    }
    // long lists (K > kSpLong, rare: points near the unit circle): lane t sums the terms t, t + 32, ... of the
    // point in increasing k, then a fixed xor tree combines the 32 partials (xadd is commutative, so every
    // lane ends with the same value) -- a fixed order per point, whatever points share the warp
    for (unsigned lm = __ballot_sync(0xffffffffu, lng); lm; lm &= lm - 1) {
      const int q = __ffs(lm) - 1;
      const int fq = __shfl_sync(0xffffffffu, first, q), Kq = __shfl_sync(0xffffffffu, K, q);
      const polar_t pz = PL[q];
      double pr = 0.0, pim = 0.0;
      long long pe = 0;
      for (int t = lane; t < Kq; t += 32) {
        const SpTerm u = sparse_term<CK, CPLX>(P, pz, fq + t, __ldg(sidx + fq + t));
        xadd(pr, pim, pe, u.r, u.i, u.e);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double qr = __shfl_xor_sync(0xffffffffu, pr, o), qi = __shfl_xor_sync(0xffffffffu, pim, o);
        const long long qe = __shfl_xor_sync(0xffffffffu, pe, o);
        xadd(pr, pim, pe, qr, qi, qe);
      }
      if (lane == q) { sr = pr; si = pim; se = (pr == 0.0 && pim == 0.0) ? 0 : pe; }
    }
    if (i < n) {
      if (state == 1) {
        const double nan = __longlong_as_double(0x7ff8000000000000LL);
        store_value<OK>(vals, exps, i, nan, CPLX ? nan : 0.0, 0);
      } else if (state == 2) {
        double cr, ci;
        a0_value<CK>(P, cr, ci);
        store_value<OK>(vals, exps, i, cr, ci, cr == 0 && ci == 0 ? 0 : P.shift);
      } else {
        store_value<OK>(vals, exps, i, sr, si, se + P.shift);
      }
    }
  }
#ifdef FPE_ITEM_TRACE
  if (lane == 0) {
    const unsigned int q = atomicAdd(&fpe_sp_trace_n, 1u);
    if (q < (1u << 20)) { fpe_sp_trace[q][0] = tr_t0; fpe_sp_trace[q][1] = sp_gtimer(); fpe_sp_trace[q][2] = tr_info; }
  }
#endif
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
// Per-point confidence (eq:def_prec_loss; the errors file of P:2114-2118): after the
// evaluation, c = max(0, ceil(N_lambda) - s(Q)) with N_lambda = hh_i* + lambda hk_i* (the sheared cover's
// top, log2 max_k |a_k z^k| in [N - 1, N)) and s(Q) the exact scale of the result (value = m 2^e with
// max(|m_re|, |m_im|) in [1/2, 1): s = e + [m_re^2 + m_im^2 >= 1]); c = 0 when |Q| >= M (the first case
// of eq:def_prec_loss; ceil(N) >= s(M), so the clamp only removes the overestimate).  The error bound
// err_exp and the trusted bits follow fpe.h (fpe_diag).  Written into the point's fpe_diag.
template <int OK>
__global__ void __launch_bounds__(256) k_confidence(long long n, PolyDev P, const void* __restrict__ vals,
                                                    const long long* __restrict__ exps, fpe_diag* __restrict__ diag) {
  constexpr int pw = (OK == FPE_R32 || OK == FPE_C32) ? 24 : 53;   // working precision (bits)
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    fpe_diag d = diag[i];
    int c = INT32_MIN, trusted = 0, eexp = INT32_MIN;
    if (d.region >= 0 && isfinite(d.lambda)) {
      double mr, mi;
      if constexpr (OK == FPE_R64) { mr = static_cast<const double*>(vals)[i]; mi = 0.0; }
      else if constexpr (OK == FPE_C64) { const double2 v = static_cast<const double2*>(vals)[i]; mr = v.x; mi = v.y; }
      else if constexpr (OK == FPE_R32) { mr = static_cast<const float*>(vals)[i]; mi = 0.0; }
      else { const float2 v = static_cast<const float2*>(vals)[i]; mr = v.x; mi = v.y; }
      long long e = exps ? exps[i] : 0;
      const int2 v = P.hull[d.region];
      const double N = __fma_rn(d.lambda, (double)v.x, (double)v.y);
      const double K = (double)max(d.kept, 1);
      const double E = ceil(N) + ceil(log2(2.0 * K + 256.0)) + ceil(log2(K)) + 1.0 - pw;
      eexp = (int)max(-2147483647.0, min(2147483647.0, E));
      const double m = fmax(fabs(mr), fabs(mi));
      if (m != 0.0 && isfinite(m)) {
        const int k = frexp_exp(m);       // renormalise (plain-float outputs)
        mr = ldexp(mr, -k); mi = ldexp(mi, -k); e += k;
        const long long sQ = e + ((__fma_rn(mr, mr, mi * mi) >= 1.0) ? 1 : 0);
        c = (int)max(0.0, min(2000000000.0, ceil(N) - (double)sQ));
        trusted = (int)max(0.0, min((double)pw, (double)sQ - E));
      }
    } else if (d.region >= 0) {   // z = 0: the value a_0 is exact
      c = 0; trusted = pw; eexp = INT32_MIN;
    }
    diag[i].cancel = c;
    diag[i].trusted = trusted;
    diag[i].err_exp = eexp;
  }
}

// ------------------------------------------------------------------------------------------
// Newton step (eq:newton): N_P(z) = z - Q1/Q2 with Q1 = m1 2^e1, Q2 = m2 2^e2 the
// extended-range FPE values of P and P'; the quotient is (m1/m2) 2^(e1 - e2), so huge or tiny P(z), P'(z)
// cancel their scales before any rounding to the working format (the valuation cancellation of P:1985).
template <int PK, int OK>
__global__ void __launch_bounds__(256) k_newton(long long n, const void* __restrict__ pts, const void* __restrict__ v1,
                                                const long long* __restrict__ e1, const void* __restrict__ v2,
                                                const long long* __restrict__ e2, void* __restrict__ out,
                                                void* __restrict__ incr) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double x, y;
    load_point<PK>(pts, i, x, y);
    double ar, ai, br, bi;
    if constexpr (OK == FPE_R64) { ar = static_cast<const double*>(v1)[i]; ai = 0; br = static_cast<const double*>(v2)[i]; bi = 0; }
    else if constexpr (OK == FPE_C64) {
      const double2 a = static_cast<const double2*>(v1)[i], b = static_cast<const double2*>(v2)[i];
      ar = a.x; ai = a.y; br = b.x; bi = b.y;
    } else if constexpr (OK == FPE_R32) { ar = static_cast<const float*>(v1)[i]; ai = 0; br = static_cast<const float*>(v2)[i]; bi = 0; }
    else {
      const float2 a = static_cast<const float2*>(v1)[i], b = static_cast<const float2*>(v2)[i];
      ar = a.x; ai = a.y; br = b.x; bi = b.y;
    }
    // (a / b) 2^(e1 - e2), mantissas in [1/2, 1): the complex quotient is formed in fp64
    const double den = __fma_rn(br, br, bi * bi);
    double qr = __fma_rn(ar, br, ai * bi) / den, qi = __fma_rn(ai, br, -ar * bi) / den;
    const long long de = e1[i] - e2[i];
    const int sc = (int)max(-4000ll, min(4000ll, de));
    qr = ldexp(qr, sc); qi = ldexp(qi, sc);
    const double zr = x - qr, zi = y - qi;
    if constexpr (OK == FPE_R64) {
      static_cast<double*>(out)[i] = zr;
      if (incr) static_cast<double*>(incr)[i] = qr;
    } else if constexpr (OK == FPE_C64) {
      static_cast<double2*>(out)[i] = make_double2(zr, zi);
      if (incr) static_cast<double2*>(incr)[i] = make_double2(qr, qi);
    } else if constexpr (OK == FPE_R32) {
      static_cast<float*>(out)[i] = (float)zr;
      if (incr) static_cast<float*>(incr)[i] = (float)qr;
    } else {
      static_cast<float2*>(out)[i] = make_float2((float)zr, (float)zi);
      if (incr) static_cast<float2*>(incr)[i] = make_float2((float)qr, (float)qi);
    }
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
  const size_t smem = (P.nv <= kSmemHullMax ? P.nv * sizeof(int2) : 0) + (P.nv <= kSmemHullDbl ? P.nv * sizeof(double2) : 0);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_classify<PK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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

template <int PK, int CK>
static void launch_eval_sparse_t(const void* pts, long long n, const PolyDev& P, const int2* lr, int* tab, void* vals,
                                 long long* exps, cudaStream_t s) {
  constexpr bool cplx = PtTraits<PK>::cplx || PtTraits<CK>::cplx;
  constexpr int OK = PtTraits<CK>::f32 ? (cplx ? FPE_C32 : FPE_R32) : (cplx ? FPE_C64 : FPE_R64);
  const size_t smem = sizeof(SpTerm) * kSpWarps * kSpRound + sizeof(polar_t) * kSpWarps * 32 +
                      sizeof(int) * (kSpWarps * 65);
  k_sparse_table<<<1, 1024, 0, s>>>(P, tab);
  // one wave of resident CTAs (grid-stride): a grid of several partial waves left the last one at
  // a fraction of the occupancy this latency-bound kernel needs
  static int resident[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !resident[dev]) {
    cudaFuncSetAttribute(k_eval_sparse_coop<PK, CK, OK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    int occ = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_eval_sparse_coop<PK, CK, OK>, kSpWarps * 32, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    resident[dev] = std::max(1, occ) * sms;
  }
  const long long warps = (n + 31) / 32;
  const long long blocks = std::min<long long>((warps + kSpWarps - 1) / kSpWarps, dev < 64 ? resident[dev] : 148ll * 4);
  k_eval_sparse_coop<PK, CK, OK><<<(int)std::max(1ll, blocks), kSpWarps * 32, smem, s>>>(pts, n, P, lr, tab, vals, exps);
}

bool launch_eval_sparse(int pk, const void* pts, long long n, const PolyDev& P, const int2* lr, int* tab, void* vals,
                        long long* exps, cudaStream_t s) {
  FPE_DISPATCH_PC(launch_eval_sparse_t, pts, n, P, lr, tab, vals, exps, s)
  return true;
}

template <int PK>
static void launch_newton_t(int ok, long long n, const void* pts, const void* v1, const long long* e1, const void* v2,
                            const long long* e2, void* out, void* incr, cudaStream_t s) {
  switch (ok) {
    case FPE_R64: k_newton<PK, FPE_R64><<<grid_for(n, 256), 256, 0, s>>>(n, pts, v1, e1, v2, e2, out, incr); break;
    case FPE_C64: k_newton<PK, FPE_C64><<<grid_for(n, 256), 256, 0, s>>>(n, pts, v1, e1, v2, e2, out, incr); break;
    case FPE_R32: k_newton<PK, FPE_R32><<<grid_for(n, 256), 256, 0, s>>>(n, pts, v1, e1, v2, e2, out, incr); break;
    default: k_newton<PK, FPE_C32><<<grid_for(n, 256), 256, 0, s>>>(n, pts, v1, e1, v2, e2, out, incr); break;
  }
}

void launch_newton(int pk, int ok, long long n, const void* pts, const void* v1, const long long* e1, const void* v2,
                   const long long* e2, void* out, void* incr, cudaStream_t s) {
  switch (pk) {
    case FPE_R64: launch_newton_t<FPE_R64>(ok, n, pts, v1, e1, v2, e2, out, incr, s); break;
    case FPE_C64: launch_newton_t<FPE_C64>(ok, n, pts, v1, e1, v2, e2, out, incr, s); break;
    case FPE_R32: launch_newton_t<FPE_R32>(ok, n, pts, v1, e1, v2, e2, out, incr, s); break;
    default: launch_newton_t<FPE_C32>(ok, n, pts, v1, e1, v2, e2, out, incr, s); break;
  }
}

void launch_confidence(int ok, long long n, const PolyDev& P, const void* vals, const long long* exps,
                       fpe_diag* diag, cudaStream_t s) {
  switch (ok) {
    case FPE_R64: k_confidence<FPE_R64><<<grid_for(n, 256), 256, 0, s>>>(n, P, vals, exps, diag); break;
    case FPE_C64: k_confidence<FPE_C64><<<grid_for(n, 256), 256, 0, s>>>(n, P, vals, exps, diag); break;
    case FPE_R32: k_confidence<FPE_R32><<<grid_for(n, 256), 256, 0, s>>>(n, P, vals, exps, diag); break;
    default: k_confidence<FPE_C32><<<grid_for(n, 256), 256, 0, s>>>(n, P, vals, exps, diag); break;
  }
}

bool launch_horner(int pk, const void* pts, long long n, const PolyDev& P, void* vals, long long* exps,
                   cudaStream_t s) {
  FPE_DISPATCH_PC(launch_horner_t, pts, n, P, vals, exps, s)
  return true;
}

}  // namespace fpe

#ifdef FPE_ITEM_TRACE
extern "C" int fpe_debug_sp_trace(unsigned long long* host, int cap, int reset) {
  unsigned int n = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&n, fpe::fpe_sp_trace_n, sizeof(n));
  n = n < (1u << 20) ? n : (1u << 20);
  const int m = (int)(n < (unsigned)cap ? n : (unsigned)cap);
  if (host && m) cudaMemcpyFromSymbol(host, fpe::fpe_sp_trace, (size_t)m * 24);
  if (reset) { unsigned int z = 0; cudaMemcpyToSymbol(fpe::fpe_sp_trace_n, &z, sizeof(z)); }
  return m;
}
#endif
