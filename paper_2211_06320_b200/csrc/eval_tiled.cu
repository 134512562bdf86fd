// eval_tiled.cu -- the bucketed, shared-memory-tiled window evaluator (north star subsystems 2-4).
//
// Pipeline (all on the caller's stream, no host round trip):
//   k_bucket_hist    per-CTA histogram of a 23-bit key monotone in an fp64 estimate of lambda, slice claims;
//                    k_bucket_scan: bucket starts (sort.cu).
//   k_classify_bucket lines 5-8 of FPE_p per point (lambda = RN(log2|z|) via lambda_fast, k_lambda,
//                    [l, r]; device_common.cuh) and the point's record written to its bucket position.
//                    l and r are both non-decreasing in lambda (d/dlambda of cover(k) + lambda k - N is
//                    k - k_lambda), so points with close keys have nested, nearly equal windows.
//   k_plan (sort.cu) the bucket order cut into groups of 32*NP consecutive points; per group the union
//                    window and the work items (one whole group, or one item per kPiece-aligned piece of a
//                    long window).
//   k_eval_tiled     persistent warps: first the parallel pieces, then every other group in order.  A warp streams the coefficients of its item's range through a
//                    private 3-stage shared-memory ring filled by 1-D TMA bulk copies (cp.async.bulk +
//                    mbarrier complete_tx), reads them as warp-uniform broadcasts (one LDS per
//                    coefficient for NP points per lane) and runs NP independent Horner chains per lane
//                    (fp64 / fp32 FMA), masked only at the ragged ends of the windows (exact Q_lambda,
//                    eq:reducedQlambda).  Windows are cut at absolute multiples of kPiece and the piece
//                    partials are folded top-down with z^kPiece (compensated powering) and z^gap /
//                    z^l (polar route, fpe_polar.cuh) -- every point's arithmetic depends only on its
//                    own window, so results are bitwise independent of the batch and of whether its
//                    pieces were evaluated by one warp or in parallel (scratch + last-arriver fold).
#include <cuda_runtime.h>
#include <cstdint>
#include <algorithm>
#include "fpe_internal.h"
#include "fpe_math.cuh"
#include "fpe_polar.cuh"
#include "device_common.cuh"
#include "sort.cuh"
#include "eval_tiled.cuh"
#include "kernels.cuh"
#include "tma.cuh"
#include "mma_piece.cuh"

namespace fpe {

constexpr int kWarps = 4;      // warps per CTA of k_eval_tiled
constexpr int kStages = 3;     // TMA ring depth per warp

// ------------------------------------------------------------------------------------------------
// Work bucketing (the sort key: bucket_key, bucket_estimates in fpe_math.cuh, host-tested) and classification,
// which writes every point's record straight to its bucket position.

// Window bounds of every bucket's points for k_plan: a point's lambda = RN(log2|z|) lies within 2^-50 +
// 2^-53 |lambda| (+ half an ulp) of its estimate, so within [lo - eps, hi + eps] of its bucket's estimates
// (eps = 2^-44 (1 + |lambda|), generous); l and r are non-decreasing in lambda, so the windows at the two ends
// (exact classification, device_common.cuh) bound every point's.  Bucket 0 holds only z = 0 (window {k_min})
// and non-finite z (empty windows): no finite z has an estimate below -1100.  Also flags buckets whose points
// are all below / all above mma_covers' |z| range (|z| in [max(|x|,|y|), sqrt2 max(|x|,|y|)), so lambda
// < -3 or >= 3.5 rules a point out).
__global__ void __launch_bounds__(256) k_bucket_windows(PolyDev P, int cb, int4* __restrict__ bwin) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= (1 << cb)) return;
  int4 w = make_int4(0, 0, 1, 0);
  if (b > 0) {
    double lo, hi;
    bucket_estimates((uint32_t)b, cb, lo, hi);
    const double la = lo - 0x1p-44 * (1.0 + fabs(lo)), lb = hi + 0x1p-44 * (1.0 + fabs(hi));
    int istar, l, r, l2, r2;
    classify_lambda(P.hull, P.nv, P.drop, la, istar, l, r);
    classify_lambda(P.hull, P.nv, P.drop, lb, istar, l2, r2);
    w = make_int4((int)(l - P.k_min), (int)(r2 - P.k_min), lb < -3.0 ? 1 : 0, la >= 3.5 ? 1 : 0);
  }
  bwin[b] = w;
}

// Pass 1 of the counting sort: per classify CTA (the same contiguous range of points k_classify_bucket
// gives it), a shared-memory histogram of the top coarse_bits(n) key bits, then one global atomicAdd per
// nonzero bucket claims the CTA's slice of that bucket.  A streaming pass over the points (16 B each for
// complex fp64), no classification.
template <int PK>
__global__ void __launch_bounds__(kScatterThreads) k_bucket_hist(const void* __restrict__ pts, long long n,
                                                                 long long ppc, uint32_t* __restrict__ gcount,
                                                                 uint2* __restrict__ cta_slice) {
  extern __shared__ __align__(16) unsigned char s_dyn[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(s_dyn);
  const int cb = coarse_bits(n), nbk = 1 << cb;
  for (int b = threadIdx.x; b < nbk; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const long long beg = (long long)blockIdx.x * ppc, end = min(n, beg + ppc);
#ifndef FPE_HIST_U
#define FPE_HIST_U 8   // 4: 0.319 ms, 8: 0.309, 16: 0.61 (cfg3 hist + scan)
#endif
  constexpr int U = FPE_HIST_U;   // independent point loads in flight per thread
  for (long long i0 = beg + threadIdx.x; i0 < end; i0 += U * blockDim.x) {
    double x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + (long long)u * blockDim.x;
      x[u] = 0.0; y[u] = 0.0;
      if (i < end) load_point<PK>(pts, i, x[u], y[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + (long long)u * blockDim.x < end)
        atomicAdd(&hist[bucket_key(x[u], y[u], PtTraits<PK>::cplx) >> (kKeyBits - cb)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbk; b += blockDim.x) {
    const uint32_t c = hist[b];
    cta_slice[((size_t)blockIdx.x << cb) + b] = make_uint2(c ? atomicAdd(gcount + b, c) : 0u, c);
  }
}

// Pass 2: lines 5-8 of FPE_p per point (lambda, k_lambda, [l, r]; device_common.cuh) and the point's record
// {index, key, l, r, z} written to its bucket position: bucket start + this CTA's slice (k_bucket_hist,
// k_bucket_scan) + a shared-memory counter.  The order inside a (CTA, bucket) slice is unspecified.  At the
// end every counter must stand at its slice's end (both passes computed the same keys): checked, counted in
// kStatSliceMismatch.
template <int PK>
__global__ void __launch_bounds__(kScatterThreads) k_classify_bucket(const void* __restrict__ pts, long long n,
                                                                     long long ppc, PolyDev P,
                                                                     const uint32_t* __restrict__ bstart,
                                                                     const uint2* __restrict__ cta_slice,
                                                                     PtRec* __restrict__ rec,
                                                                     fpe_diag* __restrict__ diag,
                                                                     unsigned long long* __restrict__ stats) {
  extern __shared__ __align__(16) unsigned char s_dyn[];
  uint32_t* slot = reinterpret_cast<uint32_t*>(s_dyn);   // next position of every bucket's slice, then the cover
  const int2* hull = P.hull;
  double2* hv = reinterpret_cast<double2*>(s_dyn + kBuckets * sizeof(uint32_t));
  const bool staged = P.nv <= kSmemHullDbl;
  if (staged) {
    int2* sh = reinterpret_cast<int2*>(s_dyn + kBuckets * sizeof(uint32_t) + (size_t)P.nv * sizeof(double2));
    for (int i = threadIdx.x; i < P.nv; i += blockDim.x) {
      const int2 v = P.hull[i];
      sh[i] = v;
      hv[i] = make_double2((double)v.x, (double)v.y);
    }
    hull = sh;
  }
  const int cb = coarse_bits(n), nbk = 1 << cb;
  const uint2* my = cta_slice + ((size_t)blockIdx.x << cb);
  for (int b = threadIdx.x; b < nbk; b += blockDim.x) slot[b] = __ldg(bstart + b) + __ldg(my + b).x;
  __syncthreads();
  const long long beg = (long long)blockIdx.x * ppc, end = min(n, beg + ppc);
  double xn = 0.0, yn = 0.0;   // the next iteration's point, loaded one iteration ahead
  if (beg + threadIdx.x < end) load_point<PK>(pts, beg + threadIdx.x, xn, yn);
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    const double x = xn, y = yn;
    if (i + blockDim.x < end) load_point<PK>(pts, i + blockDim.x, xn, yn);
    int hard = 0;
    double lam = 0.0;
    int istar, l, r;
    bool done = false;
    // the enclosure of log2|z| (its midpoint gives the bucket key, exactly as in k_bucket_hist)
    const bool kp = key_point(x, y, PtTraits<PK>::cplx);
    double lo = 0.0, hi = 0.0, mid = 0.0;
    if (kp) lambda_enclosure(x, y, PtTraits<PK>::cplx, lo, hi, mid);
    const uint32_t key = kp ? key_of_estimate(mid) : 0u;
    if (staged && P.dbl_ok && kp) {
      // fast path: searches on the enclosure; only undecided points compute the rounded lambda
      // (the diagnostics still report the rounded lambda, so the tests check this path's indexing)
      bool amb = false;
      classify_lambda_vp(hull, hv, P.nv, P.drop, LamIv{lo, hi, &amb}, istar, l, r);
      done = !amb;
      if (done && diag) lam = lambda_fast(x, y, PtTraits<PK>::cplx, &hard);
    }
    if (!done) {
      lam = lambda_fast(x, y, PtTraits<PK>::cplx, &hard);
      if (staged && P.dbl_ok) classify_lambda_v<true>(hull, hv, P.nv, P.drop, lam, istar, l, r);
      else if (staged) classify_lambda_v<false>(hull, hv, P.nv, P.drop, lam, istar, l, r);
      else classify_lambda(hull, P.nv, P.drop, lam, istar, l, r);
    }
    if (diag) {
      fpe_diag dg;
      dg.lambda = lam; dg.region = istar; dg.l = l; dg.r = r;
      dg.kept = kept_count(P, l, r); dg.hard = hard; dg.cancel = INT32_MIN; dg.trusted = 0;
      dg.err_exp = INT32_MIN; dg.pad = 0;
      diag[i] = dg;
    }
    if (hard) atomicAdd(stats + kStatHard, 1ull);
    // one shared-memory atomic per point (buckets rarely repeat within a warp)
    const uint32_t pos = atomicAdd(&slot[key >> (kKeyBits - cb)], 1u);
    // one 256-bit store (STG.E.ENL2.256): the record's whole 32-byte sector in one request
    const unsigned long long zx = __double_as_longlong(x), zy = __double_as_longlong(y);
    asm volatile("st.global.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(rec + pos), "r"((uint32_t)i),
                 "r"(key), "r"((uint32_t)l), "r"((uint32_t)r), "r"((uint32_t)zx), "r"((uint32_t)(zx >> 32)),
                 "r"((uint32_t)zy), "r"((uint32_t)(zy >> 32))
                 : "memory");
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbk; b += blockDim.x) {
    const uint2 sl = __ldg(my + b);
    if (slot[b] != __ldg(bstart + b) + sl.x + sl.y) atomicAdd(stats + kStatSliceMismatch, 1ull);
  }
}

// ------------------------------------------------------------------------------------------------
// Horner step on one coefficient (W = working real type)
template <int CK> struct Step;
template <> struct Step<FPE_C64> {
  using CT = double2; using W = double;
  __device__ static void apply(W& br, W& bi, W zr, W zi, CT a) {
    W t = fma(br, zr, fma(-bi, zi, a.x));
    bi = fma(br, zi, fma(bi, zr, a.y));
    br = t;
  }
};
template <> struct Step<FPE_C32> {
  using CT = float2; using W = float;
  __device__ static void apply(W& br, W& bi, W zr, W zi, CT a) {
    W t = fmaf(br, zr, fmaf(-bi, zi, a.x));
    bi = fmaf(br, zi, fmaf(bi, zr, a.y));
    br = t;
  }
};
// real coefficients: complex point (CPLX) or real point
template <> struct Step<FPE_R64> {
  using CT = double; using W = double;
  template <bool CPLX>
  __device__ static void apply_t(W& br, W& bi, W zr, W zi, CT a) {
    if constexpr (CPLX) { W t = fma(br, zr, fma(-bi, zi, a)); bi = fma(br, zi, bi * zr); br = t; }
    else br = fma(br, zr, a);
  }
};
template <> struct Step<FPE_R32> {
  using CT = float; using W = float;
  template <bool CPLX>
  __device__ static void apply_t(W& br, W& bi, W zr, W zi, CT a) {
    if constexpr (CPLX) { W t = fmaf(br, zr, fmaf(-bi, zi, a)); bi = fmaf(br, zi, bi * zr); br = t; }
    else br = fmaf(br, zr, a);
  }
};
template <int CK, bool CPLX>
__device__ __forceinline__ void horner_step(typename Step<CK>::W& br, typename Step<CK>::W& bi,
                                            typename Step<CK>::W zr, typename Step<CK>::W zi,
                                            typename Step<CK>::CT a) {
  if constexpr (CK == FPE_C64 || CK == FPE_C32) Step<CK>::apply(br, bi, zr, zi, a);
  else Step<CK>::template apply_t<CPLX>(br, bi, zr, zi, a);
}

// Two complex fp64 Horner steps (two points, one shared coefficient) in the source order that lets
// ptxas reuse operands between consecutive DFMAs (coefficient, then b, then z): a DFMA that reads three
// fresh register pairs issues at 2/3 of the fp64 rate on B200, one with a reused operand at full rate
// (tools/dfma_bench2.cu: 13.4 vs 12.5 T FMA/s for this loop).
__device__ __forceinline__ void horner_step2_c64(double& br0, double& bi0, double& br1, double& bi1, double zr0,
                                                 double zi0, double zr1, double zi1, double2 a) {
  const double u0 = fma(-bi0, zi0, a.x);
  const double u1 = fma(-bi1, zi1, a.x);
  const double v1 = fma(bi1, zr1, a.y);
  const double v0 = fma(bi0, zr0, a.y);
  const double nr0 = fma(br0, zr0, u0);
  const double ni0 = fma(br0, zi0, v0);
  const double nr1 = fma(br1, zr1, u1);
  const double ni1 = fma(br1, zi1, v1);
  br0 = nr0; bi0 = ni0; br1 = nr1; bi1 = ni1;
}

// Packed single precision (sm_100a FFMA2: two fp32 FMAs per instruction, the scalar coefficient broadcast
// to both halves): the fp32 Horner of two points per instruction, with the same roundings as the scalar
// steps (Step<FPE_C32> / Step<FPE_R32>), so results are bitwise unchanged.
__device__ __forceinline__ unsigned long long f2pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2unpack(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ unsigned long long fmul2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

template <int CK> struct Ring {
  using CT = typename Step<CK>::CT;
  CT* buf;            // kStages * kChunk coefficients of this warp
  uint64_t* bar;      // kStages mbarriers
  const CT* coef;     // padded dense coefficient array (relative to k_min)
  uint32_t g;         // chunks consumed (warp-uniform)
  uint32_t gi;        // chunks issued (warp-uniform)
  int q_next, q_end;  // next chunk to issue and the last chunk of the current range
  int dir;            // -1: chunks in decreasing order (Horner), +1: increasing (mma_piece.cuh)
};

template <int CK>
__device__ __forceinline__ void ring_issue_n(Ring<CK>& R, int n) {
  using CT = typename Step<CK>::CT;
  if ((threadIdx.x & 31) == 0) {
    for (int i = 0; i < n; ++i) {
      const int s = (int)((R.gi + i) % kStages);
      fence_proxy_async();
      mbar_expect_tx(R.bar + s, kChunk * sizeof(CT));
      tma_load_1d(R.buf + s * kChunk, R.coef + (size_t)(R.q_next + R.dir * i) * kChunk, kChunk * sizeof(CT), R.bar + s);
    }
  }
  R.gi += n;
  R.q_next += R.dir * n;
}
// Start streaming the chunks that cover [lo, hi] (relative indices, lo <= hi), highest chunk first.
template <int CK>
__device__ __forceinline__ void ring_begin(Ring<CK>& R, int lo, int hi) {
#ifdef FPE_EXP_NO_STREAM
  return;
#endif
  R.q_next = hi / kChunk;
  R.q_end = lo / kChunk;
  R.dir = -1;
  ring_issue_n(R, min(kStages - (int)(R.gi - R.g), R.q_next - R.q_end + 1));
}
// The same in increasing chunk order (the tensor-core pieces).
template <int CK>
__device__ __forceinline__ void ring_begin_up(Ring<CK>& R, int lo, int hi) {
  R.q_next = lo / kChunk;
  R.q_end = hi / kChunk;
  R.dir = 1;
  ring_issue_n(R, min(kStages - (int)(R.gi - R.g), R.q_end - R.q_next + 1));
}
template <int CK>
__device__ __forceinline__ const typename Step<CK>::CT* ring_wait(Ring<CK>& R) {
  const int s = (int)(R.g % kStages);
  mbar_wait(R.bar + s, (R.g / kStages) & 1u);
  return R.buf + s * kChunk;
}
template <int CK>
__device__ __forceinline__ void ring_release(Ring<CK>& R) {
  __syncwarp();
  ++R.g;
  if (R.dir < 0 ? R.q_next >= R.q_end : R.q_next <= R.q_end) ring_issue_n(R, 1);
}

// The in-warp tensor-core pass of piece p for 16 points (x, y, act: the point of lane & 15, as in
// k_eval_mma's warp layout): the piece's 64 chunks through this warp's ring, the same mma_piece.cuh
// arithmetic as k_eval_mma, so the partial is bitwise k_eval_mma's.  Used only by groups whose items did
// not fit the DMMA scratch (GroupDesc::mma_slot == kMmaInWarp); kept out of line (rare path).
struct MmaPassOut {
  Ring<FPE_C64> R;
  double r, i;   // the partial of point lane (lanes 0..15)
};
__device__ __noinline__ MmaPassOut mma_pass_inwarp(Ring<FPE_C64> R, double x, double y, int act, int p) {
  MmaFrag F;
  mma_setup(F, x, y, act);
  ring_begin_up(R, p * kPiece, p * kPiece + kPiece - 1);
  for (int k = 0; k < kMmaPieceChunks; ++k) {
    mma_chunk(F, ring_wait(R));
    ring_release(R);
  }
  MmaPassOut o;
  mma_finish(F, x, y, o.r, o.i);
  o.R = R;
  return o;
}

// Horner over the coefficient range [lo, hi] (relative, descending) for the NP points of every lane:
// point j updates b_j = b_j z_j + a_k only for k in its own window [wl_j, wr_j] (b_j must be 0 on
// entry).  Inside [F_lo, F_hi], common to all points whose window meets [lo, hi], the steps are
// unmasked (8 coefficients loaded ahead, then NP independent Horner chains per coefficient); outside
// it a masked step freezes b outside the window (above it b stays exactly 0, as the unmasked step would keep it).
// Points whose window misses [lo, hi] compute garbage that the caller discards.
template <int CK, int NP, bool CPLX>
__device__ __forceinline__ void stream_range(Ring<CK>& R, int lo, int hi, const int (&wl)[NP], const int (&wr)[NP],
                                             const typename Step<CK>::W (&zr)[NP],
                                             const typename Step<CK>::W (&zi)[NP],
                                             typename Step<CK>::W (&br)[NP], typename Step<CK>::W (&bi)[NP]) {
  using CT = typename Step<CK>::CT;
  using W = typename Step<CK>::W;
#ifdef FPE_EXP_NO_STREAM
  return;
#endif
  int mx = lo, mn = hi;
  bool any = false;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    if (wl[j] <= wr[j] && wl[j] <= hi && wr[j] >= lo) {
      mx = max(mx, wl[j]);
      mn = min(mn, wr[j]);
      any = true;
    }
  }
  int F_lo = __reduce_max_sync(0xffffffffu, mx);
  int F_hi = __reduce_min_sync(0xffffffffu, mn);
  if (!__any_sync(0xffffffffu, any) || F_lo > F_hi) { F_lo = lo; F_hi = lo - 1; }
  for (int q = hi / kChunk; q >= lo / kChunk; --q) {
    const CT* cb = ring_wait(R) - q * kChunk;
    const int k1 = min(hi, q * kChunk + kChunk - 1), k0 = max(lo, q * kChunk);
    int k = k1;
#ifdef FPE_EXP_NO_MASK
    k = min(k, F_hi);
#endif
    // masked steps (ragged window ends): 8 coefficients loaded ahead as in the unmasked loop, so that a
    // warp running alone (the tail of a batch) is not bound by one shared-memory latency per coefficient
    auto masked_step = [&](const CT a, int kk) {
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        W nr = br[j], ni = bi[j];
        horner_step<CK, CPLX>(nr, ni, zr[j], zi[j], a);
        if (kk >= wl[j] && kk <= wr[j]) { br[j] = nr; bi[j] = ni; }
      }
    };
    {
      const int m1 = max(k0, F_hi + 1);
      for (; k - 7 >= m1; k -= 8) {
        CT a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = cb[k - u];
#pragma unroll
        for (int u = 0; u < 8; ++u) masked_step(a[u], k - u);
      }
      for (; k >= m1; --k) masked_step(cb[k], k);
    }
    const int f0 = max(k0, F_lo);
#ifdef FPE_EXP_NO_HOT
    k = min(k, f0 - 1);
#endif
    if constexpr ((CK == FPE_C32 || CK == FPE_R32) && NP % 2 == 0) {
      if (k - 7 >= f0) {   // points (j, j + 1) packed into one register pair each
        unsigned long long pr[NP / 2], pi[NP / 2], qr[NP / 2], qi[NP / 2], qn[NP / 2];
#pragma unroll
        for (int q = 0; q < NP / 2; ++q) {
          pr[q] = f2pack(br[2 * q], br[2 * q + 1]); pi[q] = f2pack(bi[2 * q], bi[2 * q + 1]);
          qr[q] = f2pack(zr[2 * q], zr[2 * q + 1]); qi[q] = f2pack(zi[2 * q], zi[2 * q + 1]);
          qn[q] = f2pack(-zi[2 * q], -zi[2 * q + 1]);
        }
        for (; k - 7 >= f0; k -= 8) {
          CT a[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) a[u] = cb[k - u];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int q = 0; q < NP / 2; ++q) {
              if constexpr (CK == FPE_C32) {   // Step<FPE_C32>: t = fma(-bi, zi, ar), bi = fma(br, zi, fma(bi, zr, ai))
                const unsigned long long t = ffma2(pi[q], qn[q], f2pack(a[u].x, a[u].x));
                const unsigned long long v = ffma2(pi[q], qr[q], f2pack(a[u].y, a[u].y));
                pi[q] = ffma2(pr[q], qi[q], v);
                pr[q] = ffma2(pr[q], qr[q], t);
              } else if constexpr (CPLX) {     // Step<FPE_R32> at complex points
                const unsigned long long t = ffma2(pi[q], qn[q], f2pack(a[u], a[u]));
                pi[q] = ffma2(pr[q], qi[q], fmul2(pi[q], qr[q]));
                pr[q] = ffma2(pr[q], qr[q], t);
              } else {                         // Step<FPE_R32> at real points
                pr[q] = ffma2(pr[q], qr[q], f2pack(a[u], a[u]));
              }
            }
          }
        }
#pragma unroll
        for (int q = 0; q < NP / 2; ++q) {
          f2unpack(pr[q], br[2 * q], br[2 * q + 1]);
          f2unpack(pi[q], bi[2 * q], bi[2 * q + 1]);
        }
      }
    } else {
    for (; k - 7 >= f0; k -= 8) {
      CT a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = cb[k - u];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if constexpr (NP % 2 == 0 && CK == FPE_C64) {
#pragma unroll
          for (int j = 0; j < NP; j += 2)
            horner_step2_c64(br[j], bi[j], br[j + 1], bi[j + 1], zr[j], zi[j], zr[j + 1], zi[j + 1], a[u]);
        } else {
#pragma unroll
          for (int j = 0; j < NP; ++j) horner_step<CK, CPLX>(br[j], bi[j], zr[j], zi[j], a[u]);
        }
      }
    }
    }
    for (; k >= f0; --k) {
      const CT a = cb[k];
#pragma unroll
      for (int j = 0; j < NP; ++j) horner_step<CK, CPLX>(br[j], bi[j], zr[j], zi[j], a);
    }
#ifdef FPE_EXP_NO_MASK
    k = k0 - 1;
#endif
    for (; k - 7 >= k0; k -= 8) {
      CT a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = cb[k - u];
#pragma unroll
      for (int u = 0; u < 8; ++u) masked_step(a[u], k - u);
    }
    for (; k >= k0; --k) masked_step(cb[k], k);
    ring_release(R);
  }
}

// ------------------------------------------------------------------------------------------------
// combining piece partials (top-down Horner over the pieces, PAPER.md:1621-1622 generalised) and the
// epilogue Q = acc z^l.  Shared by the serial and the parallel path, so that a point's
// result does not depend on which one evaluated it.
struct Acc {
  double r, i;
  int base;        // relative index of the lowest coefficient folded in so far
  bool started;
  bool have_zk;    // zk = z^kPiece computed (once per point: a long window folds up to ~256 pieces)
  xc_t zk;
};

// (re, im) * (h + e) 2^E, scaled into range (the product is bounded by the cover argument).
__device__ __forceinline__ void mul_ext(double& re, double& im, const xc_t& p) {
  double r = __fma_rn(re, p.hr, __fma_rn(-im, p.hi, __fma_rn(re, p.er, -im * p.ei)));
  double i = __fma_rn(re, p.hi, __fma_rn(im, p.hr, __fma_rn(re, p.ei, im * p.er)));
  int sc = (int)max(-3000ll, min(3000ll, p.E));
  re = ldexp_fast(r, sc); im = ldexp_fast(i, sc);
}

template <bool CPLX>
__device__ __forceinline__ xc_t power_piece(double x, double y) {   // z^kPiece, compensated powering
  if constexpr (CPLX) return xc_pow(x, y, kPiece);
  else { xr_t v = xr_pow(x, kPiece); return xc_t{v.h, 0.0, v.e, 0.0, v.E}; }
}
template <bool CPLX>
__device__ __forceinline__ xc_t power_polar(double x, double y, long long n) {   // z^n by the polar route
  polar_t p = polar_of<CPLX>(x, y);
  if constexpr (CPLX) return pow_polar(p.lam, p.tau, n);
  else { xr_t v = pow_polar_real(p.lam, p.neg, n); return xc_t{v.h, 0.0, 0.0, 0.0, v.E}; }
}

template <bool CPLX>
__device__ __noinline__ void acc_fold(Acc& A, double hr, double hi, int pbase, double x, double y) {
  if (!A.started) { A.r = hr; A.i = hi; A.base = pbase; A.started = true; return; }
  const int gap = A.base - pbase;
  if (gap == kPiece) {
    if (!A.have_zk) { A.zk = power_piece<CPLX>(x, y); A.have_zk = true; }
    mul_ext(A.r, A.i, A.zk);
  } else {
    mul_ext(A.r, A.i, power_polar<CPLX>(x, y, gap));
  }
  A.r += hr; A.i += hi;
  A.base = pbase;
}

// The evaluators stage a point's accumulator -- acc (re, im) 2^E, relative to z^n with n = base + k_min (n = -1:
// nothing accumulated) -- and k_unsort applies the epilogue Q = acc z^n (finalize) on the way to the caller's
// order: the polar-route power is fp64 work that would compete with the Horner DFMAs for the fp64 pipe here,
// while k_unsort is bound by its random gathers and has the issue slots to spare.
// The staged accumulators are written at random (the point's input index) and read once, by k_unsort: an L2
// evict-first policy keeps them from displacing the coefficients the evaluator warps re-read from L2.
__device__ __forceinline__ void stage_acc(PtOut* out, long long pos, const Acc& A, long long extraE, int kmin) {
  const unsigned long long a = __double_as_longlong(A.started ? A.r : 0.0), b = __double_as_longlong(A.started ? A.i : 0.0);
  const unsigned long long e = (unsigned long long)extraE;
  const unsigned long long nn = (unsigned long long)(A.started ? (long long)A.base + kmin : -1ll);
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;" ::"l"(out + pos),
               "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)),
               "r"((uint32_t)e), "r"((uint32_t)(e >> 32)), "r"((uint32_t)nn), "r"((uint32_t)(nn >> 32)), "l"(pol)
               : "memory");
}


// Q = acc z^l as (re + i im) 2^E (finalize: k_unsort, and the full Horner's direct stores).
struct Fin {
  double re, im;
  long long E;
};

// z^n for single-precision outputs (tolerance 2^-16 S): plain fp64 log2 / atan2 / exp2 / sincospi.  The
// product n log2|z| is split exactly (TwoProduct), so the error is n times that of log2|z| and arg z,
// ~2^-53 absolute each: below 2^-26 relative for n < 2^26 (d_eff < 2^26 for every dense handle).
template <bool CPLX>
__device__ __forceinline__ xc_t power_polar_lite(double x, double y, long long n) {
  const double dn = (double)n;
  const double lam = CPLX ? log2(hypot(x, y)) : log2(fabs(x));
  const double mh = dn * lam, ml = fma(dn, lam, -mh);
  const double E = rint(mh);
  const double mod = exp2((mh - E) + ml);
  xc_t v;
  v.er = 0.0; v.ei = 0.0; v.E = (long long)E;
  if constexpr (CPLX) {
    const double tau = atan2(y, x) * 0.15915494309189535;   // arg z / 2 pi
    const double ah = dn * tau, al = fma(dn, tau, -ah);
    const double f = (ah - rint(ah)) + al;
    double sn, cs;
    sincospi(2.0 * f, &sn, &cs);
    v.hr = cs * mod; v.hi = sn * mod;
  } else {
    v.hr = (x < 0.0 && (n & 1)) ? -mod : mod; v.hi = 0.0;
  }
  return v;
}

template <bool CPLX, bool LITE = false>
__device__ __noinline__ Fin finalize(double x, double y, Acc A, const PolyDev& P) {
#ifdef FPE_EXP_NO_FINALIZE
  return Fin{A.r, A.i, 0};
#endif
  if (!isfinite(x) || !isfinite(y)) {
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    return Fin{nan, CPLX ? nan : 0.0, 0};
  }
  double qr = A.started ? A.r : 0.0, qi = A.started ? A.i : 0.0;
  if (x == 0.0 && y == 0.0) {   // z = 0: P(0) = a_0 (window {k_min})
    if (P.k_min != 0) { qr = 0.0; qi = 0.0; }
    return Fin{qr, qi, (qr == 0.0 && qi == 0.0) ? 0 : (long long)P.shift};
  }
  long long E = 0;
  const long long n = A.started ? (long long)A.base + P.k_min : 0;
#ifdef FPE_EXP_NO_ZPOW
  if (false) {
#else
  if (n > 0) {
#endif
    const xc_t p = LITE ? power_polar_lite<CPLX>(x, y, n) : power_polar<CPLX>(x, y, n);
    const double r = __fma_rn(qr, p.hr, -qi * p.hi);
    const double i = __fma_rn(qr, p.hi, qi * p.hr);
    qr = r; qi = i; E = p.E;
  }
  return Fin{qr, qi, E + P.shift};
}

// The NP points of each lane of a group: sorted position j*32 + lane.
template <int NP>
struct Pts {
  long long idx[NP];   // input index (the caller's order): where the accumulator is staged
  double x[NP], y[NP];
  int wl[NP], wr[NP];   // relative window; empty (wl > wr) for padding and non-finite points
  bool valid[NP];
};

// Group g holds the positions [g*32*NP, min(n, (g+1)*32*NP)) of the bucket order (k_plan); its records
// (index, window, z) are read coalesced and without waiting for the descriptor.
template <int PK, int NP>
__device__ __forceinline__ void load_group(Pts<NP>& S, uint32_t g, long long n, const PtRec* __restrict__ rec,
                                           int kmin) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const long long pos = (long long)g * (32 * NP) + j * 32 + lane;
    S.valid[j] = pos < n;
    S.idx[j] = 0; S.x[j] = 0.0; S.y[j] = 0.0; S.wl[j] = 0x3fffffff; S.wr[j] = -1;
    if (S.valid[j]) {
      const int4 h = __ldcg(reinterpret_cast<const int4*>(rec + pos));
      const double2 z = __ldcg(reinterpret_cast<const double2*>(rec + pos) + 1);
      S.idx[j] = (uint32_t)h.x; S.x[j] = z.x; S.y[j] = z.y;
      if (h.w >= h.z) { S.wl[j] = h.z - kmin; S.wr[j] = h.w - kmin; }
    }
  }
}

// Self-check of the plan's union window (k_plan bounds it by per-bucket window bounds): every point's
// window must lie inside it, else its terms outside would be skipped.  Counted in kStatWindowEscape.
template <int NP>
__device__ __forceinline__ void check_union(const Pts<NP>& S, const GroupDesc& d, const Plan& plan) {
  int bad = 0;
#pragma unroll
  for (int j = 0; j < NP; ++j) bad += (S.wl[j] <= S.wr[j] && (S.wl[j] < d.lo || S.wr[j] > d.hi)) ? 1 : 0;
  if (bad) atomicAdd(plan.stats + kStatWindowEscape, (unsigned long long)bad);
}

// The Horner sums of piece p = [rlo, rhi] for the NP points of every lane (b = 0 on entry).  Points that
// cover the whole piece on the tensor cores (mma_covers; complex fp64 coefficients) take k_eval_mma's
// partial from its scratch instead; the others stream the part of the piece their windows need.
// INWARP (k_eval_overflow only): the group's tensor-core pieces did not fit the DMMA scratch and are run
// here with k_eval_mma's arithmetic; k_eval_tiled never sees such groups, so its code has no DMMA path.
template <int CK, int NP, bool CPLX, bool INWARP = false>
__device__ __forceinline__ void eval_piece(Ring<CK>& R, const Pts<NP>& S, int rlo, int rhi, int p, const GroupDesc& d,
                                           const Plan& plan, typename Step<CK>::W (&br)[NP],
                                           typename Step<CK>::W (&bi)[NP]) {
  using W = typename Step<CK>::W;
  W zr[NP], zi[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) { zr[j] = (W)S.x[j]; zi[j] = (W)S.y[j]; br[j] = 0; bi[j] = 0; }
  if constexpr (CK == FPE_C64) {
    if (d.mma_np > 0 && p >= d.mma_p0 && p < d.mma_p0 + d.mma_np) {
      int wl[NP], wr[NP];
      bool cov[NP];
      int v_lo = rhi + 1, v_hi = rlo - 1;
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        cov[j] = mma_covers(S.wl[j], S.wr[j], S.x[j], S.y[j], p);
        wl[j] = cov[j] ? 0x3fffffff : S.wl[j];
        wr[j] = cov[j] ? -1 : S.wr[j];
        if (wl[j] <= wr[j] && wl[j] <= rhi && wr[j] >= rlo) { v_lo = min(v_lo, wl[j]); v_hi = max(v_hi, wr[j]); }
      }
      v_lo = max(rlo, __reduce_min_sync(0xffffffffu, v_lo));
      v_hi = min(rhi, __reduce_max_sync(0xffffffffu, v_hi));
      if (v_lo <= v_hi) {
        ring_begin(R, v_lo, v_hi);
        stream_range<CK, NP, CPLX>(R, v_lo, v_hi, wl, wr, zr, zi, br, bi);
      }
      const int lane = threadIdx.x & 31;
      if constexpr (!INWARP) {   // k_eval_mma's partials
        const double2* scr = plan.mma_scratch + (size_t)(d.mma_slot + (p - d.mma_p0)) * plan.gsize;
#pragma unroll
        for (int j = 0; j < NP; ++j)
          if (cov[j]) { const double2 v = __ldcg(scr + j * 32 + lane); br[j] = v.x; bi[j] = v.y; }
      } else {
      // DMMA scratch was full: the same passes in this warp, 16 points (positions 16 w .. 16 w + 15 of the
      // group, w = 2 j + h) at a time, exactly k_eval_mma's layout
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        if (!__any_sync(0xffffffffu, cov[j])) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int src = 16 * h + (lane & 15);
          const int act = __shfl_sync(0xffffffffu, cov[j] ? 1 : 0, src);
          if (!__any_sync(0xffffffffu, act)) continue;
          const double x = __shfl_sync(0xffffffffu, S.x[j], src), y = __shfl_sync(0xffffffffu, S.y[j], src);
          const MmaPassOut o = mma_pass_inwarp(R, x, y, act, p);
          R = o.R;
          const double vr = __shfl_sync(0xffffffffu, o.r, lane & 15), vi = __shfl_sync(0xffffffffu, o.i, lane & 15);
          if ((lane >> 4) == h && cov[j]) { br[j] = vr; bi[j] = vi; }
        }
      }
      }
      return;
    }
  }
  ring_begin(R, rlo, rhi);
  stream_range<CK, NP, CPLX>(R, rlo, rhi, S.wl, S.wr, zr, zi, br, bi);
}

// One warp evaluates a whole group: the pieces of its union window top-down, folding as it goes.
// The group's records and descriptor were loaded by the caller (one group ahead, so that their latency
// hides behind the previous group's epilogue); `prefetch` is called once the coefficient stream is done
// and before the epilogue, to issue the loads of the next group.
template <int NP>
struct GroupCtx {   // raw loads of a group, consumed only when the group is evaluated
  uint32_t g;
  bool second;      // fetched in the bucket-order pass (after the long-group list)
  GroupDesc d;
  int4 h[NP];
  double2 z[NP];
};

template <int PK, int NP>
__device__ __forceinline__ void group_load(GroupCtx<NP>& c, uint32_t g, long long n, const Plan& plan,
                                           const PtRec* rec, int kmin) {
  const int lane = threadIdx.x & 31;
  c.g = g;
  if (g < plan.ngroups) {
    c.d = plan.desc[g];
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const long long pos = (long long)g * (32 * NP) + j * 32 + lane;
      if (pos < n) {
        c.h[j] = __ldcg(reinterpret_cast<const int4*>(rec + pos));
        c.z[j] = __ldcg(reinterpret_cast<const double2*>(rec + pos) + 1);
      }
    }
  }
}

template <int NP>
__device__ __forceinline__ void group_unpack(Pts<NP>& S, const GroupCtx<NP>& c, long long n, int kmin) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const long long pos = (long long)c.g * (32 * NP) + j * 32 + lane;
    S.valid[j] = pos < n;
    S.idx[j] = 0; S.x[j] = 0.0; S.y[j] = 0.0; S.wl[j] = 0x3fffffff; S.wr[j] = -1;
    if (S.valid[j]) {
      S.idx[j] = (uint32_t)c.h[j].x;
      S.x[j] = c.z[j].x; S.y[j] = c.z[j].y;
      if (c.h[j].w >= c.h[j].z) { S.wl[j] = c.h[j].z - kmin; S.wr[j] = c.h[j].w - kmin; }
    }
  }
}

template <int PK, int CK, int OK, int NP, typename Prefetch, bool INWARP = false>
__device__ __forceinline__ void single_group(Ring<CK>& R, const GroupCtx<NP>& c, long long n, const PolyDev& P,
                                             const Plan& plan, PtOut* out, Prefetch prefetch) {
  constexpr bool CPLX = PtTraits<OK>::cplx;
  using W = typename Step<CK>::W;
  const GroupDesc d = c.d;
  Pts<NP> S;
  group_unpack<NP>(S, c, n, (int)P.k_min);
  check_union<NP>(S, d, plan);
  const bool nonempty = d.hi >= d.lo;
  const int p_hi = nonempty ? d.hi / kPiece : 0, p_lo = nonempty ? d.lo / kPiece : 0;
  Acc A[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) A[j] = Acc{0.0, 0.0, 0, false};
  if (nonempty) {
    for (int p = p_hi; p >= p_lo; --p) {
      const int rlo = max(d.lo, p * kPiece), rhi = min(d.hi, p * kPiece + kPiece - 1);
      W br[NP], bi[NP];
      eval_piece<CK, NP, CPLX, INWARP>(R, S, rlo, rhi, p, d, plan, br, bi);
#pragma unroll
      for (int j = 0; j < NP; ++j)
        if (S.wl[j] <= S.wr[j] && S.wl[j] <= p * kPiece + kPiece - 1 && S.wr[j] >= p * kPiece)
          acc_fold<CPLX>(A[j], (double)br[j], (double)bi[j], max(S.wl[j], p * kPiece), S.x[j], S.y[j]);
    }
  }
  prefetch();
#pragma unroll
  for (int j = 0; j < NP; ++j)
    if (S.valid[j]) stage_acc(out, S.idx[j], A[j], 0, (int)P.k_min);
}

// One warp evaluates piece p of a multi-piece group into its scratch slot; the warp that completes
// the group's last piece folds all partials in order and finalises.
template <int PK, int CK, int OK, int NP>
__device__ __forceinline__ bool multi_piece(Ring<CK>& R, uint32_t g, int p, long long n, const Plan& plan,
                                            const PtRec* rec, const PolyDev& P, PtOut* out) {
  constexpr bool CPLX = PtTraits<OK>::cplx;
  using W = typename Step<CK>::W;
  using W2 = typename std::conditional<std::is_same<W, float>::value, float2, double2>::type;
  constexpr int G = 32 * NP;
  const int lane = threadIdx.x & 31;
  const GroupDesc d = plan.desc[g];
  const int kmin = (int)P.k_min;
  const int rlo = max(d.lo, p * kPiece), rhi = min(d.hi, p * kPiece + kPiece - 1);
  Pts<NP> S;
  load_group<PK, NP>(S, g, n, rec, kmin);
  if (p == d.lo / kPiece) check_union<NP>(S, d, plan);   // once per group
  W br[NP], bi[NP];
  eval_piece<CK, NP, CPLX>(R, S, rlo, rhi, p, d, plan, br, bi);
  const int p0 = d.lo / kPiece;
  W2* scr = static_cast<W2*>(plan.scratch);
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    W2 v; v.x = br[j]; v.y = bi[j];
    scr[(size_t)(d.slot + (p - p0)) * G + j * 32 + lane] = v;
  }
  __threadfence();
  __syncwarp();
  uint32_t done = 0;
  if (lane == 0) done = atomicAdd(plan.gcnt + g, 1u);
  done = __shfl_sync(0xffffffffu, done, 0);
  if (done != (uint32_t)d.npieces - 1) return false;
  __threadfence();
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    if (!S.valid[j]) continue;
    Acc A{0.0, 0.0, 0, false};
    if (S.wl[j] <= S.wr[j]) {
      for (int pp = d.hi / kPiece; pp >= p0; --pp) {
        if (S.wl[j] <= pp * kPiece + kPiece - 1 && S.wr[j] >= pp * kPiece) {
          const W2 v = __ldcg(scr + (size_t)(d.slot + (pp - p0)) * G + j * 32 + lane);
          acc_fold<CPLX>(A, (double)v.x, (double)v.y, max(S.wl[j], pp * kPiece), S.x[j], S.y[j]);
        }
      }
    }
    stage_acc(out, S.idx[j], A, 0, (int)P.k_min);
  }
  return true;
}

template <int CK>
constexpr size_t ring_bytes() {
  return (size_t)kWarps * kStages * kChunk * sizeof(typename Step<CK>::CT);
}

// Persistent evaluator: every warp first takes parallel pieces of long windows, then whole groups,
// both from global atomic counters (largest work first; the tail is at most one group).
#ifdef FPE_ITEM_TRACE
// Debugging (build with -DFPE_ITEM_TRACE): per work item of k_eval_tiled, {start ns, end ns, info} with
// info = kind (1 multi piece, 2 group) << 60 | group << 20 | union length / 16 (or the piece index).
__device__ unsigned long long fpe_item_trace[1 << 20][3];
__device__ unsigned int fpe_item_trace_n;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_item(unsigned long long t0, unsigned long long info) {
  if ((threadIdx.x & 31) == 0) {
    const unsigned int i = atomicAdd(&fpe_item_trace_n, 1u);
    if (i < (1u << 20)) { fpe_item_trace[i][0] = t0; fpe_item_trace[i][1] = gtimer(); fpe_item_trace[i][2] = info; }
  }
}
#define FPE_TRACE_T0 const unsigned long long trace_t0 = gtimer()
#define FPE_TRACE(info) trace_item(trace_t0, (info))
#else
#define FPE_TRACE_T0
#define FPE_TRACE(info)
#endif

template <int PK, int CK, int OK, int NP>
#ifndef FPE_EVAL_MIN_CTAS
#define FPE_EVAL_MIN_CTAS 3   // CTAs per SM the register budget is sized for (12 warps)
#endif
__global__ void __launch_bounds__(kWarps * 32, FPE_EVAL_MIN_CTAS) k_eval_tiled(long long n, PolyDev P,
                                                               const PtRec* rec, Plan plan, PtOut* out) {
  using CT = typename Step<CK>::CT;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  CT* ring_buf = reinterpret_cast<CT*>(smem) + (size_t)wib * kStages * kChunk;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ring_bytes<CK>()) + wib * kStages;
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  Ring<CK> R{ring_buf, bars, static_cast<const CT*>(P.coef), 0u, 0u, 0, 0, -1};
  const uint32_t n_multi = min(plan.ctrs[2], plan.cap);
  // the next item index is fetched one item ahead, so the atomic's latency hides behind the work
  uint32_t nxt = 0;
  if (lane == 0) nxt = atomicAdd(plan.ctrs + 0, 1u);
  for (;;) {
    const uint32_t it = __shfl_sync(0xffffffffu, nxt, 0);
    if (it >= n_multi) break;
    if (lane == 0) nxt = atomicAdd(plan.ctrs + 0, 1u);
    const uint2 item = plan.items[it];
    if (item.x == ~0u) continue;
    FPE_TRACE_T0;
    const bool folded = multi_piece<PK, CK, OK, NP>(R, item.x, (int)item.y, n, plan, rec, P, out);
    FPE_TRACE((1ull << 60) | ((unsigned long long)folded << 59) | ((unsigned long long)item.x << 20) | item.y);
    (void)folded;
  }
  // groups: software-pipelined one group ahead (the next group's records load during this epilogue)
  const int kmin = (int)P.k_min;
  if (lane == 0) nxt = atomicAdd(plan.ctrs + 1, 1u);
  GroupCtx<NP> cur;
  // the listed long-window groups (the largest single items) first, then the others in reverse bucket
  // order, so that the tail of the persistent loop is short
  const uint32_t n_long1 = plan.ctrs[3], n_long = n_long1 + plan.ctrs[8];
  auto gid = [&](uint32_t it) {
    return it < n_long1 ? __ldg(plan.long_groups + it)
         : it < n_long ? __ldg(plan.long_groups + plan.ngroups - 1 - (it - n_long1))
                       : (it - n_long < plan.ngroups ? plan.ngroups - 1 - (it - n_long) : plan.ngroups);
  };
  auto load = [&](GroupCtx<NP>& c) {
    const uint32_t it = __shfl_sync(0xffffffffu, nxt, 0);
    group_load<PK, NP>(c, gid(it), n, plan, rec, kmin);
    c.second = it >= n_long;
    if (lane == 0) nxt = atomicAdd(plan.ctrs + 1, 1u);
  };
  load(cur);
  while (cur.g < plan.ngroups) {
    GroupCtx<NP> nx;
    auto fetch_next = [&]() { load(nx); };
    if (cur.d.npieces > 1 || (cur.d.mma_np > 0 && cur.d.mma_slot == kMmaInWarp) || (cur.second && cur.d.listed))
      fetch_next();   // evaluated as parallel pieces (multi_piece), by k_eval_overflow, or from the list
    else {
      FPE_TRACE_T0;
      single_group<PK, CK, OK, NP>(R, cur, n, P, plan, out, fetch_next);
      FPE_TRACE((2ull << 60) | ((unsigned long long)cur.g << 20) |
                (unsigned long long)(cur.d.hi >= cur.d.lo ? (cur.d.hi - cur.d.lo + 1) / 16 : 0));
    }
    cur = nx;
  }
}

// Groups whose tensor-core items did not fit the DMMA scratch (k_plan's overflow list): one warp per group,
// every piece top-down as single_group does, the covered whole pieces by in-warp DMMA passes with
// k_eval_mma's arithmetic (eval_piece<INWARP>) -- so these points get the bits they would get in any batch.
// Launched after k_eval_tiled whenever tensor-core items are planned; exits at once when the list is empty.
template <int PK, int CK, int OK, int NP>
__global__ void __launch_bounds__(kWarps * 32) k_eval_overflow(long long n, PolyDev P, const PtRec* rec, Plan plan,
                                                               PtOut* out) {
  using CT = typename Step<CK>::CT;
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t n_ovf = plan.mma_ctrs[2];
  if (n_ovf == 0) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  CT* ring_buf = reinterpret_cast<CT*>(smem) + (size_t)wib * kStages * kChunk;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ring_bytes<CK>()) + wib * kStages;
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  Ring<CK> R{ring_buf, bars, static_cast<const CT*>(P.coef), 0u, 0u, 0, 0, -1};
  const int kmin = (int)P.k_min;
  for (;;) {
    uint32_t it = 0;
    if (lane == 0) it = atomicAdd(plan.mma_ctrs + 3, 1u);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= n_ovf) break;
    GroupCtx<NP> c;
    group_load<PK, NP>(c, plan.ovf_groups[it], n, plan, rec, kmin);
    auto none = []() {};
    single_group<PK, CK, OK, NP, decltype(none), true>(R, c, n, P, plan, out, none);
  }
}

// ------------------------------------------------------------------------------------------------
// Wide handles (PolyDev::wide: the good scales span more than one common power-of-two shift can hold in
// the working format; the coefficients are stored as given): the window sum by an exponent-rescaled Horner
// (north_star "exponent-rescaled Horner ... frexp/ldexp rescaling to avoid overflow").
// One thread per point of the bucket order; the same absolute kPiece pieces, folded top-down with the same
// acc_fold powers, so the decomposition (and its error bound) is the fast path's.  Inside a piece
// b = m 2^E with max(|m_re|, |m_im|) in [1/2, 1) after every step; z = w 2^ez with max(|w_re|, |w_im|) in
// [1/2, 1), so m w never overflows; a coefficient larger than b by more than 2^60 moves b to the
// coefficient's scale first (b may then underflow: it is below the coefficient's rounding).  All in fp64
// (fp32 handles too: more accurate than their 2^-16 tolerance needs).
struct XAcc { double r, i; long long E; int base; bool started; bool have_zk; xc_t zk; };

__device__ __forceinline__ void xnorm(double& r, double& i, long long& E) {
  const double m = fmax(fabs(r), fabs(i));
  if (m != 0.0 && isfinite(m)) { const int e = frexp_exp(m); r = ldexp_fast(r, -e); i = ldexp_fast(i, -e); E += e; }
  else if (m == 0.0) E = 0;
}

template <int CK, bool CPLX>
__device__ __forceinline__ void wide_piece(const PolyDev& P, int lo, int hi, double wr, double wi, int ez,
                                           double& br, double& bi, long long& E) {
  br = 0.0; bi = 0.0; E = 0;
  bool nz = false;
  for (int k = hi; k >= lo; --k) {
    long long E1 = nz ? E + ez : E;   // the exponent of b w
    double cr, ci;
    if constexpr (PtTraits<CK>::f32) { float a, b; Coef<CK>::get(P.coef, k, a, b); cr = a; ci = b; }
    else Coef<CK>::get(P.coef, k, cr, ci);
    double sr = 0.0, si = 0.0;
    if (cr != 0.0 || ci != 0.0) {
      const int ec = frexp_exp(fmax(fabs(cr), fabs(ci)));
      if (!nz || (long long)ec > E1 + 60) {   // b negligible next to a_k: continue at a_k's scale
        if (nz) {
          const int s = (int)max(-2200ll, min(2200ll, E1 - ec));
          br = ldexp_fast(br, s); bi = ldexp_fast(bi, s);
        }
        E1 = ec;
      }
      const int s = (int)max(-2200ll, -E1);
      sr = ldexp_fast(cr, s); si = ldexp_fast(ci, s);
    }
    if (nz) {   // b <- b w + a_k 2^-E1: the fast path's fused steps (Step<>::apply)
      if constexpr (CPLX) { const double t = __fma_rn(br, wr, __fma_rn(-bi, wi, sr)); bi = __fma_rn(br, wi, __fma_rn(bi, wr, si)); br = t; }
      else br = __fma_rn(br, wr, sr);
    } else {
      br = sr; bi = si;
    }
    E = E1;
    xnorm(br, bi, E);
    nz = (br != 0.0 || bi != 0.0);
  }
}

// A <- A z^(A.base - pbase) + (hr + i hi) 2^hE, all in extended range (acc_fold with exponents).
template <bool CPLX>
__device__ __noinline__ void xacc_fold(XAcc& A, double hr, double hi, long long hE, int pbase, double x, double y) {
  if (!A.started) { A.r = hr; A.i = hi; A.E = hE; A.base = pbase; A.started = true; return; }
  const int gap = A.base - pbase;
  if (gap == kPiece && !A.have_zk) { A.zk = power_piece<CPLX>(x, y); A.have_zk = true; }
  const xc_t m = (gap == kPiece) ? A.zk : power_polar<CPLX>(x, y, gap);
  double r = __fma_rn(A.r, m.hr, __fma_rn(-A.i, m.hi, __fma_rn(A.r, m.er, -A.i * m.ei)));
  double i = __fma_rn(A.r, m.hi, __fma_rn(A.i, m.hr, __fma_rn(A.r, m.ei, A.i * m.er)));
  long long E = A.E + m.E;
  xnorm(r, i, E);
  if (hr != 0.0 || hi != 0.0) {   // align and add
    if (r == 0.0 && i == 0.0) { r = hr; i = hi; E = hE; }
    else if (hE > E) { const int s = (int)max(-2200ll, E - hE); r = ldexp_fast(r, s) + hr; i = ldexp_fast(i, s) + hi; E = hE; }
    else { const int s = (int)max(-2200ll, hE - E); r += ldexp_fast(hr, s); i += ldexp_fast(hi, s); }
    xnorm(r, i, E);
  }
  A.r = r; A.i = i; A.E = E; A.base = pbase;
}

template <int PK, int CK, int OK>
__global__ void __launch_bounds__(256) k_eval_wide(long long n, PolyDev P, const PtRec* rec, PtOut* out) {
  constexpr bool CPLX = PtTraits<OK>::cplx;
  const int kmin = (int)P.k_min;
  for (long long pos = blockIdx.x * (long long)blockDim.x + threadIdx.x; pos < n; pos += (long long)gridDim.x * blockDim.x) {
    const int4 h = __ldcg(reinterpret_cast<const int4*>(rec + pos));
    const double2 z = __ldcg(reinterpret_cast<const double2*>(rec + pos) + 1);
    const double x = z.x, y = z.y;
    XAcc A{0.0, 0.0, 0, 0, false};
    if (h.w >= h.z && isfinite(x) && isfinite(y) && (x != 0.0 || y != 0.0)) {
      const int wl = h.z - kmin, wr_ = h.w - kmin;
      const int ez = frexp_exp(fmax(fabs(x), fabs(y)));
      const double ux = ldexp(x, -ez), uy = ldexp(y, -ez);
      for (int p = wr_ / kPiece; p >= wl / kPiece; --p) {
        const int lo = max(wl, p * kPiece), hi = min(wr_, p * kPiece + kPiece - 1);
        double br, bi;
        long long E;
        wide_piece<CK, CPLX>(P, lo, hi, ux, uy, ez, br, bi, E);
        xacc_fold<CPLX>(A, br, bi, E, lo, x, y);
      }
    }
    if (!A.started && x == 0.0 && y == 0.0 && h.w >= h.z) {   // z = 0: the window {k_min}, value a_0 (finalize)
      double cr = 0.0, ci = 0.0;
      a0_value<CK>(P, cr, ci);
      A = XAcc{cr, ci, 0, 0, true};
    }
    const Acc a{A.r, A.i, A.base, A.started};
    stage_acc(out, (uint32_t)h.x, a, A.started ? A.E : 0, kmin);
  }
}

// ------------------------------------------------------------------------------------------------
// Full Horner over all coefficients (the context baseline), with the evaluator's
// streaming: warps take 64 consecutive input points (2 per lane) and stream every coefficient chunk
// through the TMA ring.  Without the band there is no magnitude bound, so after every chunk each point
// whose partial sum exceeds 2^(emax/2) is rescaled by a power of two (exponent E_j), and later
// coefficients enter multiplied by 2^-E_j (0 once that is below the working range: they are then
// below the partial sum's rounding).
template <int CK, int NP, bool CPLX>
__device__ __forceinline__ void stream_full(Ring<CK>& R, int lo, int hi, const typename Step<CK>::W (&zr)[NP],
                                            const typename Step<CK>::W (&zi)[NP], typename Step<CK>::W (&br)[NP],
                                            typename Step<CK>::W (&bi)[NP], int (&E)[NP]) {
  using CT = typename Step<CK>::CT;
  using W = typename Step<CK>::W;
  constexpr bool F32 = std::is_same<W, float>::value;
  constexpr int kHalf = F32 ? 60 : 500;      // rescale above 2^kHalf
  constexpr int kDrop = F32 ? 150 : 1100;    // 2^-E underflows the working type
  constexpr int kBlk = F32 ? 1 : 8;          // steps between checks: |z|^kBlk 2^kHalf stays finite for
                                             // |z| < 2^65 (fp64); fp32 checks every step
  W s[NP];                                   // 2^-E: the scale of the coefficients still to come
#pragma unroll
  for (int j = 0; j < NP; ++j) s[j] = (W)1;
  auto rescale = [&]() {
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const double m = fmax(fabs((double)br[j]), fabs((double)bi[j]));
      if (m > ldexp(1.0, kHalf) && isfinite(m)) {
        const int e = frexp_exp(m);
        br[j] = (W)ldexp_fast((double)br[j], -e);
        bi[j] = (W)ldexp_fast((double)bi[j], -e);
        E[j] += e;
        s[j] = E[j] > kDrop ? (W)0 : (W)ldexp(1.0, -E[j]);
      }
    }
  };
  for (int q = hi / kChunk; q >= lo / kChunk; --q) {
    const CT* cb = ring_wait(R) - q * kChunk;
    const int k1 = min(hi, q * kChunk + kChunk - 1), k0 = max(lo, q * kChunk);
    for (int kb = k1; kb >= k0; kb -= kBlk) {
      const int ke = max(k0, kb - kBlk + 1);
      bool any_scaled = false;
#pragma unroll
      for (int j = 0; j < NP; ++j) any_scaled |= E[j] != 0;
      if (!__any_sync(0xffffffffu, any_scaled)) {
        if (kb - ke == 7) {
          CT a[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) a[u] = cb[kb - u];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if constexpr (NP % 2 == 0 && CK == FPE_C64) {
#pragma unroll
              for (int j = 0; j < NP; j += 2)
                horner_step2_c64(br[j], bi[j], br[j + 1], bi[j + 1], zr[j], zi[j], zr[j + 1], zi[j + 1], a[u]);
            } else {
#pragma unroll
              for (int j = 0; j < NP; ++j) horner_step<CK, CPLX>(br[j], bi[j], zr[j], zi[j], a[u]);
            }
          }
        } else {
          for (int k = kb; k >= ke; --k) {
            const CT a = cb[k];
#pragma unroll
            for (int j = 0; j < NP; ++j) horner_step<CK, CPLX>(br[j], bi[j], zr[j], zi[j], a);
          }
        }
      } else {
        auto scaled_step = [&](const CT& a) {
#pragma unroll
          for (int j = 0; j < NP; ++j) {
            CT as = a;
            if constexpr (CK == FPE_C64 || CK == FPE_C32) { as.x *= s[j]; as.y *= s[j]; }
            else as *= s[j];
            horner_step<CK, CPLX>(br[j], bi[j], zr[j], zi[j], as);
          }
        };
        if (kb - ke == 7) {
          CT a[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) a[u] = cb[kb - u];
#pragma unroll
          for (int u = 0; u < 8; ++u) scaled_step(a[u]);
        } else {
          for (int k = kb; k >= ke; --k) scaled_step(cb[k]);
        }
      }
      rescale();
    }
    ring_release(R);
  }
}

template <int PK, int CK, int OK, int NP>
__global__ void __launch_bounds__(kWarps * 32, 3) k_horner_tiled(const void* __restrict__ pts, long long n, PolyDev P,
                                                                 uint32_t* __restrict__ ctr, void* __restrict__ vals,
                                                                 long long* __restrict__ exps,
                                                                 const uint32_t* __restrict__ list,
                                                                 const uint32_t* __restrict__ list_n) {
  using CT = typename Step<CK>::CT;
  using W = typename Step<CK>::W;
  constexpr bool CPLX = PtTraits<OK>::cplx;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  CT* ring_buf = reinterpret_cast<CT*>(smem) + (size_t)wib * kStages * kChunk;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ring_bytes<CK>()) + wib * kStages;
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  Ring<CK> R{ring_buf, bars, static_cast<const CT*>(P.coef), 0u, 0u, 0, 0, -1};
  const int hi = (int)(P.k_max - P.k_min);
  // list mode (the points k_horner_mma leaves to this kernel): positions index list[0 .. *list_n)
  const long long nn = list ? (long long)*list_n : n;
  const long long ngroups = (nn + 32 * NP - 1) / (32 * NP);
  for (;;) {
    uint32_t g = 0;
    if (lane == 0) g = atomicAdd(ctr, 1u);
    g = __shfl_sync(0xffffffffu, g, 0);
    if ((long long)g >= ngroups) break;
    ring_begin(R, 0, hi);
    double x[NP], y[NP];
    long long idx[NP];   // the point's index in the caller's order (-1: none)
    W zr[NP], zi[NP], br[NP], bi[NP];
    int E[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const long long q = (long long)g * (32 * NP) + j * 32 + lane;
      idx[j] = q < nn ? (list ? (long long)__ldg(list + q) : q) : -1;
      x[j] = 0.0; y[j] = 0.0;
      if (idx[j] >= 0) load_point<PK>(pts, idx[j], x[j], y[j]);
      zr[j] = (W)x[j]; zi[j] = (W)y[j]; br[j] = 0; bi[j] = 0; E[j] = 0;
    }
    stream_full<CK, NP, CPLX>(R, 0, hi, zr, zi, br, bi, E);
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      if (idx[j] < 0) continue;
      Acc A{(double)br[j], (double)bi[j], 0, true};
      if (!isfinite(x[j]) || !isfinite(y[j]) || (x[j] == 0.0 && y[j] == 0.0)) {
        const Fin f = finalize<CPLX>(x[j], y[j], A, P);   // NaN / a_0 (the E = 0 paths)
        store_value<OK>(vals, exps, idx[j], f.re, f.im, f.E);
        continue;
      }
      double qr = A.r, qi = A.i;
      long long Ez = 0;
      if (P.k_min > 0) {
        const xc_t p = power_polar<CPLX>(x[j], y[j], P.k_min);
        const double r = __fma_rn(qr, p.hr, -qi * p.hi);
        const double i = __fma_rn(qr, p.hi, qi * p.hr);
        qr = r; qi = i; Ez = p.E;
      }
      store_value<OK>(vals, exps, idx[j], qr, qi, Ez + E[j] + P.shift);
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Full Horner on the FP64 tensor cores (the context baseline, fpe_horner, complex fp64 coefficients): the
// same phase-split contraction as the tensor-core pieces (mma_piece.cuh), over EVERY piece of the
// coefficient range for every point.  A CTA of 8 warps takes 128 consecutive points and walks the pieces
// top-down, each piece's chunks in increasing order through a CTA-shared TMA ring; a piece's partial is
// folded into the point's extended-range accumulator with z^16384 (as the evaluator's long windows).
// Without the band there is no magnitude bound inside a piece: for |z| > 1 the accumulators and the B
// fragment are rescaled by 2^-delta per chunk, delta = floor(256 log2|z|) (exact powers of two, so only
// underflowing -- negligible -- early terms are lost); for |z| <= 1 the terms only shrink.  Points outside
// 2^-4 <= |z| < 2^3.99 (the range of w = z^256 and of the chunk powers u^i <= z^(256 - P)), zero and
// non-finite points (0.8% of sphere points) are appended to a list that k_horner_tiled evaluates afterwards
// with one point per lane (its tail is one warp streaming every coefficient: the shortest chain per
// coefficient wins).
constexpr int kHmWarps = 8;
constexpr int kHmStages = 6;

template <int PK>
__global__ void __launch_bounds__(kHmWarps * 32, 2) k_horner_mma(const void* __restrict__ pts, long long n, PolyDev P,
                                                                uint32_t* __restrict__ ctrs, uint32_t* __restrict__ rejects,
                                                                void* __restrict__ vals, long long* __restrict__ exps) {
  constexpr bool CPLX = true;
  __shared__ __align__(128) double2 ring[kHmStages][kChunk];
  __shared__ uint64_t full[kHmStages], empty[kHmStages];
  __shared__ uint32_t grp_sh;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    for (int st = 0; st < kHmStages; ++st) { mbar_init(full + st, 1); mbar_init(empty + st, kHmWarps); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const double2* coef = static_cast<const double2*>(P.coef);
  const long long nchunks = (P.k_max - P.k_min) / kChunk + 1;      // chunks holding [0, d_eff]
  const int ptop = (int)((nchunks - 1) / kMmaPieceChunks);
  const int nq_top = (int)(nchunks - (long long)ptop * kMmaPieceChunks);
  auto chunk_of = [&](long long t) -> long long {   // the t-th chunk of a group: pieces top-down, chunks up
    if (t < nq_top) return (long long)ptop * kMmaPieceChunks + t;
    const long long u = t - nq_top;
    return (long long)(ptop - 1 - u / kMmaPieceChunks) * kMmaPieceChunks + (u % kMmaPieceChunks);
  };
  uint32_t t_seq = 0, t_issued = 0;
  auto issue = [&](long long chunk) {   // thread 0
    const int st = (int)(t_issued % kHmStages);
    if (t_issued >= (uint32_t)kHmStages) mbar_wait(empty + st, ((t_issued / kHmStages) - 1) & 1u);
    fence_proxy_async();
    mbar_expect_tx(full + st, kChunk * sizeof(double2));
    tma_load_1d(ring[st], coef + (size_t)chunk * kChunk, kChunk * sizeof(double2), full + st);
    ++t_issued;
  };
  const long long ngroups = (n + 127) / 128;
  for (;;) {
    if (tid == 0) grp_sh = atomicAdd(ctrs, 1u);
    __syncthreads();
    const uint32_t grp = grp_sh;
    __syncthreads();
    if ((long long)grp >= ngroups) break;
    if (tid == 0)
      for (long long i = 0; i < kHmStages && i < nchunks; ++i) issue(chunk_of(i));
    long long issued_local = min((long long)kHmStages, nchunks);
    const long long pos = (long long)grp * 128 + 16 * w + (lane & 15);
    double x = 0.0, y = 0.0;
    if (pos < n) load_point<PK>(pts, pos, x, y);
    // 2^-4 <= |z| < 2^3.99: z^256 (w) stays below 2^1022, the chunk powers u^i <= z^(256 - P) too
    const double r2 = __fma_rn(x, x, y * y);
    const int act = (pos < n && isfinite(x) && isfinite(y) && r2 >= 0x1p-8 && r2 < 252.0) ? 1 : 0;
    if (lane < 16 && pos < n && !act) rejects[atomicAdd(ctrs + 1, 1u)] = (uint32_t)pos;
    // rescaling for |z| > 1: the chunk powers u^i start at 2^-delta0, delta0 = floor(kMmaMaxBPow log2|z|) (so
    // that the largest, z^(256 - P), is ~1), and every chunk scales by 2^-delta, delta = floor(256 log2|z|)
    const double l2z = act ? log2(hypot(x, y)) : 0.0;
    const int delta = act ? max(0, (int)floor(256.0 * l2z)) : 0;
    const int delta0 = act ? max(0, (int)floor((double)kMmaMaxBPow * l2z)) : 0;
    const int g = lane >> 2, c = lane & 3;
    double sb[2], sb0[2], sc[2][2];   // 2^-delta (2^-delta0) of the B columns g, 8 + g; 2^-delta of C columns 2c, 2c + 1
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      sb[t] = pow2i(-__shfl_sync(0xffffffffu, delta, 8 * t + g));
      sb0[t] = pow2i(-__shfl_sync(0xffffffffu, delta0, 8 * t + g));
#pragma unroll
      for (int e = 0; e < 2; ++e) sc[t][e] = pow2i(-__shfl_sync(0xffffffffu, delta, 8 * t + 2 * c + e));
    }
    XAcc A{0.0, 0.0, 0, 0, false, false, {}};
    for (int p = ptop; p >= 0; --p) {
      const int nq = (p == ptop) ? nq_top : kMmaPieceChunks;
      MmaFrag F;
      mma_setup(F, x, y, act);
#pragma unroll
      for (int t = 0; t < 2; ++t) { F.cwr[t] *= sb[t]; F.cwi[t] *= sb[t]; }   // V advances by w 2^-delta
      mma_scale_b(F, sb0);                                                  // V_0 = u^i 2^-delta0
      const bool busy = __any_sync(0xffffffffu, act);
      for (int k = 0; k < nq; ++k) {
        const int st = (int)(t_seq % kHmStages);
        mbar_wait(full + st, (t_seq / kHmStages) & 1u);
        if (busy) {
          mma_chunk(F, ring[st]);
          if (k + 1 < nq) mma_scale_c(F, sc);   // C 2^-delta before the next chunk's terms
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + st);
        ++t_seq;
        if (tid == 0 && issued_local < nchunks) issue(chunk_of(issued_local));
        ++issued_local;
        __syncwarp();
      }
      double pr, pi;
      mma_finish(F, x, y, pr, pi);
      if (act) {
        long long pe = (long long)delta0 + (long long)delta * (nq - 1);
        double r = pr, i = pi;
        xnorm(r, i, pe);
        xacc_fold<CPLX>(A, r, i, pe, p * kPiece, x, y);
      }
    }
    if (lane < 16 && act) {
      const Acc a{A.r, A.i, A.base, A.started};
      Fin f = finalize<CPLX>(x, y, a, P);
      store_value<FPE_C64>(vals, exps, pos, f.re, f.im, f.E + A.E);
    }
  }
}

// ------------------------------------------------------------------------------------------------
// The epilogue in the caller's order: the evaluators staged every point's accumulator at its input index
// (one whole 32-byte sector per point, written at random from the bucket order -- whole sectors need no
// read-modify-write, unlike the 16-byte values and 8-byte exponents themselves), so this is a coalesced
// pass over the staged accumulators and the points.
#ifndef FPE_UNSORT_U
#define FPE_UNSORT_U 2      // independent loads in flight per thread
#endif
#ifndef FPE_UNSORT_MINB
#define FPE_UNSORT_MINB 3   // CTAs per SM the register budget is sized for (2 x 3: 2.27 -> 2.02 ms at cfg3)
#endif
// Half of the points need no power (window starting at k_min), and they are spread at random over the
// lanes, so a warp used to run the polar route for its few lanes that need it while the rest idled
// (fpe_polar / dd arithmetic were 85% of k_unsort's instructions).  The points that need z^l are queued per
// warp in shared memory and the polar route runs on 32 queued points at a time (the rest at the end).
struct UTask { double re, im, x, y; long long E, nn, i; };
constexpr int kUnsortWarps = 8;
constexpr int kUnsortQ = 32 + 32 * FPE_UNSORT_U;   // queue entries per warp: < 32 left over + one iteration

template <int PK, int OK>
__global__ void __launch_bounds__(32 * kUnsortWarps, FPE_UNSORT_MINB) k_unsort(const PtOut* __restrict__ staged,
                                                long long n, const void* __restrict__ pts, PolyDev P,
                                                void* __restrict__ vals, long long* __restrict__ exps) {
  constexpr bool CPLX = PtTraits<OK>::cplx;
  constexpr int U = FPE_UNSORT_U;
  const long long stride = (long long)gridDim.x * blockDim.x;
#ifndef FPE_UNSORT_NOQ
  __shared__ UTask q_s[kUnsortWarps][kUnsortQ];
  UTask* Q = q_s[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int qn = 0;   // queued points (warp-uniform)
  auto run = [&](const UTask& t) {
    const Acc A{t.re, t.im, (int)(t.nn - P.k_min), true};
    const Fin f = finalize<CPLX, PtTraits<OK>::f32>(t.x, t.y, A, P);
    store_value<OK>(vals, exps, t.i, f.re, f.im, f.E + t.E);
  };
#endif
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 - (threadIdx.x & 31) < n; i0 += U * stride) {
    double re[U], im[U], x[U], y[U];
    long long E[U], nn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + u * stride;
      if (i < n) {
        uint32_t w[8];
        asm volatile("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                     : "l"(staged + i));
        re[u] = __hiloint2double((int)w[1], (int)w[0]);
        im[u] = __hiloint2double((int)w[3], (int)w[2]);
        E[u] = (long long)(((unsigned long long)w[5] << 32) | w[4]);
        nn[u] = (long long)(((unsigned long long)w[7] << 32) | w[6]);
        load_point<PK>(pts, i, x[u], y[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + u * stride;
#ifndef FPE_UNSORT_NOQ
      // z^l is needed (finalize's power branch) for a finite nonzero z with a window above k_min
      const bool need = i < n && nn[u] > 0 && isfinite(x[u]) && isfinite(y[u]) && (x[u] != 0.0 || y[u] != 0.0);
      const unsigned m = __ballot_sync(0xffffffffu, need);
      if (need) Q[qn + __popc(m & lt)] = UTask{re[u], im[u], x[u], y[u], E[u], nn[u], i};
      else if (i < n) {
#else
      if (i < n) {
#endif
        const Acc A{re[u], im[u], (int)(nn[u] >= 0 ? nn[u] - P.k_min : 0), nn[u] >= 0};
        const Fin f = finalize<CPLX, PtTraits<OK>::f32>(x[u], y[u], A, P);
        store_value<OK>(vals, exps, i, f.re, f.im, f.E + E[u]);
      }
#ifndef FPE_UNSORT_NOQ
      qn += __popc(m);
#endif
    }
#ifndef FPE_UNSORT_NOQ
    __syncwarp();
    while (qn >= 32) {
      qn -= 32;
      const UTask t = Q[qn + lane];
      __syncwarp();
      run(t);
    }
#endif
  }
#ifndef FPE_UNSORT_NOQ
  __syncwarp();
  if (lane < qn) run(Q[lane]);
#endif
}

// ------------------------------------------------------------------------------------------------
// host side
static inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t n_ctas(long long n) { const long long p = pts_per_cta(n); return (size_t)((n + p - 1) / p); }
// scratch for parallel pieces: 4 bytes per point (at least 1 MiB), counted in 1 KiB units
static size_t scratch_slots(long long n) {
  size_t bytes = max((size_t)n * 4, (size_t)1 << 20);
  return bytes / 1024;
}

// DMMA items: scratch of 2 KiB per (group, piece), 4 bytes per point (at least 64 items)
static size_t mma_cap(long long n) { return max((size_t)64, (size_t)n * 4 / (128 * sizeof(double2))); }

size_t tiled_ws_bytes(long long n) {
  return al256(n * sizeof(PtOut)) + al256(n * sizeof(PtRec)) +
         al256(mma_cap(n) * sizeof(uint2)) + al256(mma_cap(n) * 128 * sizeof(double2)) +
         al256(n_ctas(n) * kBuckets * sizeof(uint2)) + 2 * al256((kBuckets + 1) * sizeof(uint32_t)) +
         al256(kBuckets * sizeof(int4)) +
         al256(max_groups(n) * sizeof(GroupDesc)) + 3 * al256(max_groups(n) * sizeof(uint32_t)) +
         al256(scratch_slots(n) * sizeof(uint2)) + al256(scratch_slots(n) * 1024) + 256;
}

template <int CK>
static size_t eval_smem() {
  return ring_bytes<CK>() + kWarps * kStages * sizeof(uint64_t);
}

template <int PK, int CK, int OK, int NP>
static int launch_eval_tiled_t(long long n, const PolyDev& P, const PtRec* rec, const Plan& plan, PtOut* out,
                               cudaStream_t s) {
  const size_t smem = eval_smem<CK>();
  const int grid = persistent_grid(reinterpret_cast<const void*>(k_eval_tiled<PK, CK, OK, NP>), kWarps * 32, smem);
  k_eval_tiled<PK, CK, OK, NP><<<grid, kWarps * 32, smem, s>>>(n, P, rec, plan, out);
  return 1;
}

template <int PK, int CK, int OK>
static int launch_eval_wide_t(long long n, const PolyDev& P, const PtRec* rec, PtOut* out, cudaStream_t s) {
  const long long blocks = std::min<long long>((n + 255) / 256, 148ll * 16);
  k_eval_wide<PK, CK, OK><<<(int)std::max(1ll, blocks), 256, 0, s>>>(n, P, rec, out);
  return 1;
}

template <int PK, int CK, int OK, int NP>
static int launch_eval_overflow_t(long long n, const PolyDev& P, const PtRec* rec, const Plan& plan, PtOut* out,
                                  cudaStream_t s) {
  const size_t smem = eval_smem<CK>();
  const int grid = persistent_grid(reinterpret_cast<const void*>(k_eval_overflow<PK, CK, OK, NP>), kWarps * 32, smem);
  k_eval_overflow<PK, CK, OK, NP><<<grid, kWarps * 32, smem, s>>>(n, P, rec, plan, out);
  return 1;
}

// points per lane (groups of 32 NP points): 4 -- each coefficient load feeds 16 fp64 FMAs (complex) or 4
// (real) per lane; the single-precision evaluator as a build knob (packed FFMA2 pairs)
#ifndef FPE_NP_F32
#define FPE_NP_F32 2   // 2 vs 4: 22.07 vs 22.33 ms at cfg5-fp32
#endif
#ifndef FPE_NP_REAL
#define FPE_NP_REAL 2   // real coefficients at real points (fp64): 64-point groups, 0.72 vs 1.22 ms at cfg2
#endif
template <int PK, int CK>
struct NPFor {
  static constexpr bool cplx = PtTraits<PK>::cplx || PtTraits<CK>::cplx;
  static constexpr int value = PtTraits<CK>::f32 ? FPE_NP_F32 : (cplx ? 4 : FPE_NP_REAL);
  static constexpr int OK = PtTraits<CK>::f32 ? (cplx ? FPE_C32 : FPE_R32) : (cplx ? FPE_C64 : FPE_R64);
};

// Points per lane of the launch: 2 (groups of 64: tighter window unions) except for complex fp64
// coefficients whose windows can cover a whole tensor-core piece (d_eff + 1 >= kPiece), where the DMMA items
// need groups of 128 (k_eval_mma: 8 warps x 16 points).
static int np_for(int pk, int cdt, long long d_eff) {
  if (cdt == FPE_R32 || cdt == FPE_C32) return FPE_NP_F32;
#ifndef FPE_NP_C64_LONG
#define FPE_NP_C64_LONG 4   // experiments: 2 gives 64-point groups (and no tensor-core items)
#endif
  if (cdt == FPE_C64) return d_eff + 1 >= kPiece ? FPE_NP_C64_LONG : 2;
  return (pk == FPE_R64) ? FPE_NP_REAL : 2;
}

// histogram + slice claims (k_bucket_hist), bucket starts (k_bucket_scan), classification + records at their
// bucket positions (k_classify_bucket)
template <int PK>
static void launch_classify_bucket_t(const void* pts, long long n, const PolyDev& P, uint32_t* gcount,
                                     uint2* cta_slice, uint32_t* bstart, PtRec* rec, fpe_diag* diag,
                                     unsigned long long* stats, Stage& st, cudaStream_t s) {
  const size_t hsmem = kBuckets * sizeof(uint32_t);
  cudaFuncSetAttribute(k_bucket_hist<PK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsmem);
  k_bucket_hist<PK><<<(int)n_ctas(n), kScatterThreads, hsmem, s>>>(pts, n, pts_per_cta(n), gcount, cta_slice);
  bucket_scan(gcount, bstart, n, s);
  st.mark("bucket");
  const size_t smem = kBuckets * sizeof(uint32_t) + (P.nv <= kSmemHullDbl ? P.nv * (sizeof(int2) + sizeof(double2)) : 0);
  cudaFuncSetAttribute(k_classify_bucket<PK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_classify_bucket<PK><<<(int)n_ctas(n), kScatterThreads, smem, s>>>(pts, n, pts_per_cta(n), P, bstart, cta_slice,
                                                                     rec, diag, stats);
}

template <int PK, int CK>
static void launch_horner_tiled_t(const void* pts, long long n, const PolyDev& P, uint32_t* ctr, void* vals,
                                  long long* exps, cudaStream_t s) {
  constexpr int NP = NPFor<PK, CK>::value, OK = NPFor<PK, CK>::OK;
  const size_t smem = eval_smem<CK>();
  const int grid = persistent_grid(reinterpret_cast<const void*>(k_horner_tiled<PK, CK, OK, NP>), kWarps * 32, smem);
  cudaMemsetAsync(ctr, 0, sizeof(uint32_t), s);
  k_horner_tiled<PK, CK, OK, NP><<<grid, kWarps * 32, smem, s>>>(pts, n, P, ctr, vals, exps, nullptr, nullptr);
}

template <int PK>
static void launch_horner_mma_t(const void* pts, long long n, const PolyDev& P, uint32_t* ctrs, uint32_t* rejects,
                                void* vals, long long* exps, cudaStream_t s) {
  const int grid = persistent_grid(reinterpret_cast<const void*>(k_horner_mma<PK>), kHmWarps * 32, 0);
  k_horner_mma<PK><<<grid, kHmWarps * 32, 0, s>>>(pts, n, P, ctrs, rejects, vals, exps);
  // the rejected points: the vector full Horner over the list, one point per lane
  constexpr int NP = 1;
  const size_t smem = eval_smem<FPE_C64>();
  const int g2 = persistent_grid(reinterpret_cast<const void*>(k_horner_tiled<PK, FPE_C64, FPE_C64, NP>), kWarps * 32, smem);
  k_horner_tiled<PK, FPE_C64, FPE_C64, NP><<<g2, kWarps * 32, smem, s>>>(pts, n, P, ctrs + 2, vals, exps, rejects, ctrs + 1);
}

bool run_horner_tiled(int pk, const void* pts, long long n, const PolyDev& P, uint32_t* ctr, void* vals,
                      long long* exps, cudaStream_t s, size_t ws_bytes) {
  // complex fp64 coefficients: the tensor-core full Horner (ctr: 3 counters + the reject list of n points)
  if (P.cdt == FPE_C64 && !P.wide && (pk == FPE_C64 || pk == FPE_R64) && ws_bytes >= 256 + (size_t)n * 4) {
    cudaMemsetAsync(ctr, 0, 4 * sizeof(uint32_t), s);
    uint32_t* rejects = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(ctr) + 256);
    if (pk == FPE_C64) launch_horner_mma_t<FPE_C64>(pts, n, P, ctr, rejects, vals, exps, s);
    else launch_horner_mma_t<FPE_R64>(pts, n, P, ctr, rejects, vals, exps, s);
    return true;
  }
  switch (pk * 4 + P.cdt) {
    case FPE_R64 * 4 + FPE_R64: launch_horner_tiled_t<FPE_R64, FPE_R64>(pts, n, P, ctr, vals, exps, s); break;
    case FPE_R64 * 4 + FPE_C64: launch_horner_tiled_t<FPE_R64, FPE_C64>(pts, n, P, ctr, vals, exps, s); break;
    case FPE_C64 * 4 + FPE_R64: launch_horner_tiled_t<FPE_C64, FPE_R64>(pts, n, P, ctr, vals, exps, s); break;
    case FPE_C64 * 4 + FPE_C64: launch_horner_tiled_t<FPE_C64, FPE_C64>(pts, n, P, ctr, vals, exps, s); break;
    case FPE_R32 * 4 + FPE_R32: launch_horner_tiled_t<FPE_R32, FPE_R32>(pts, n, P, ctr, vals, exps, s); break;
    case FPE_R32 * 4 + FPE_C32: launch_horner_tiled_t<FPE_R32, FPE_C32>(pts, n, P, ctr, vals, exps, s); break;
    case FPE_C32 * 4 + FPE_R32: launch_horner_tiled_t<FPE_C32, FPE_R32>(pts, n, P, ctr, vals, exps, s); break;
    case FPE_C32 * 4 + FPE_C32: launch_horner_tiled_t<FPE_C32, FPE_C32>(pts, n, P, ctr, vals, exps, s); break;
    default: return false;
  }
  return true;
}

int run_tiled(int pk, const void* pts, long long n, const PolyDev& P, void* vals, long long* exps,
              fpe_diag* diag, void* ws, unsigned long long* stats, Stage& st, cudaStream_t s) {
  char* p = static_cast<char*>(ws);
  // the evaluators' accumulators staged at the point's input index (random whole-sector writes from the
  // bucket order, so that k_unsort streams them back in order)
  PtOut* staged = reinterpret_cast<PtOut*>(p); p += al256(n * sizeof(PtOut));
  PtRec* rec = reinterpret_cast<PtRec*>(p); p += al256(n * sizeof(PtRec));   // bucket order
  uint2* cta_slice = reinterpret_cast<uint2*>(p); p += al256(n_ctas(n) * kBuckets * sizeof(uint2));   // {start, count}
  uint32_t* gcount = reinterpret_cast<uint32_t*>(p); p += al256((kBuckets + 1) * 4);
  uint32_t* bstart = reinterpret_cast<uint32_t*>(p); p += al256((kBuckets + 1) * 4);
  int4* bwin = reinterpret_cast<int4*>(p); p += al256(kBuckets * sizeof(int4));
  Plan plan;
  plan.desc = reinterpret_cast<GroupDesc*>(p); p += al256(max_groups(n) * sizeof(GroupDesc));
  plan.gcnt = reinterpret_cast<uint32_t*>(p); p += al256(max_groups(n) * sizeof(uint32_t));
  plan.ovf_groups = reinterpret_cast<uint32_t*>(p); p += al256(max_groups(n) * sizeof(uint32_t));
  plan.long_groups = reinterpret_cast<uint32_t*>(p); p += al256(max_groups(n) * sizeof(uint32_t));
  plan.items = reinterpret_cast<uint2*>(p); p += al256(scratch_slots(n) * sizeof(uint2));
  plan.scratch = p; p += al256(scratch_slots(n) * 1024);
  plan.mma_items = reinterpret_cast<uint2*>(p); p += al256(mma_cap(n) * sizeof(uint2));
  plan.mma_scratch = reinterpret_cast<double2*>(p); p += al256(mma_cap(n) * 128 * sizeof(double2));
  plan.mma_cap = (uint32_t)mma_cap(n);
  plan.stats = stats;
  plan.ctrs = reinterpret_cast<uint32_t*>(p);
  plan.mma_ctrs = plan.ctrs + 4;
  const int np = np_for(pk, P.cdt, P.k_max - P.k_min);
  plan.gsize = 32 * np;
  plan.mma_on = (P.cdt == FPE_C64 && plan.gsize == 128 && !FPE_NO_MMA_ITEMS && !P.wide) ? 1 : 0;
  plan.ngroups = (uint32_t)((n + plan.gsize - 1) / plan.gsize);
  const bool f32 = (P.cdt == FPE_R32 || P.cdt == FPE_C32);
  const size_t slot_bytes = (size_t)plan.gsize * (f32 ? sizeof(float2) : sizeof(double2));
  plan.cap = (uint32_t)(scratch_slots(n) * 1024 / slot_bytes);
  cudaMemsetAsync(gcount, 0, (kBuckets + 1) * 4, s);
  cudaMemsetAsync(plan.ctrs, 0, 48, s);   // [0..3] vector items / groups / slots / long groups, [4..7] DMMA items,
                                          // [8] long groups of the second class
  switch (pk) {
    case FPE_R64: launch_classify_bucket_t<FPE_R64>(pts, n, P, gcount, cta_slice, bstart, rec, diag, stats, st, s); break;
    case FPE_C64: launch_classify_bucket_t<FPE_C64>(pts, n, P, gcount, cta_slice, bstart, rec, diag, stats, st, s); break;
    case FPE_R32: launch_classify_bucket_t<FPE_R32>(pts, n, P, gcount, cta_slice, bstart, rec, diag, stats, st, s); break;
    default: launch_classify_bucket_t<FPE_C32>(pts, n, P, gcount, cta_slice, bstart, rec, diag, stats, st, s); break;
  }
  st.mark("classify");
  {
    const int nbk = 1 << coarse_bits(n);
    k_bucket_windows<<<(nbk + 255) / 256, 256, 0, s>>>(P, coarse_bits(n), bwin);
  }
  plan_groups(n, bstart, bwin, plan, s);
  st.mark("plan");
  int lm = 0;
  if (plan.mma_on) {
    launch_eval_mma(n, P, rec, plan, s);
    st.mark("eval_mma");
    lm = 1;
  }
  int le = 0;
#define FPE_EV(PKV, CKV, NPV)                                                                             \
  le = P.wide ? launch_eval_wide_t<PKV, CKV, NPFor<PKV, CKV>::OK>(n, P, rec, staged, s)                      \
              : launch_eval_tiled_t<PKV, CKV, NPFor<PKV, CKV>::OK, NPV>(n, P, rec, plan, staged, s)
  switch (pk * 4 + P.cdt) {
    case FPE_R64 * 4 + FPE_R64: FPE_EV(FPE_R64, FPE_R64, FPE_NP_REAL); break;
    case FPE_R64 * 4 + FPE_C64: if (np == 4) FPE_EV(FPE_R64, FPE_C64, 4); else FPE_EV(FPE_R64, FPE_C64, 2); break;
    case FPE_C64 * 4 + FPE_R64: FPE_EV(FPE_C64, FPE_R64, 2); break;
    case FPE_C64 * 4 + FPE_C64: if (np == 4) FPE_EV(FPE_C64, FPE_C64, 4); else FPE_EV(FPE_C64, FPE_C64, 2); break;
    case FPE_R32 * 4 + FPE_R32: FPE_EV(FPE_R32, FPE_R32, FPE_NP_F32); break;
    case FPE_R32 * 4 + FPE_C32: FPE_EV(FPE_R32, FPE_C32, FPE_NP_F32); break;
    case FPE_C32 * 4 + FPE_R32: FPE_EV(FPE_C32, FPE_R32, FPE_NP_F32); break;
    case FPE_C32 * 4 + FPE_C32: FPE_EV(FPE_C32, FPE_C32, FPE_NP_F32); break;
    default: return -1;
  }
#undef FPE_EV
  st.mark(P.wide ? "eval_wide" : "eval_tiled");
  if (plan.mma_on) {   // groups whose tensor-core items overflowed the DMMA scratch (usually none)
    if (pk == FPE_C64) le += launch_eval_overflow_t<FPE_C64, FPE_C64, NPFor<FPE_C64, FPE_C64>::OK, 4>(n, P, rec, plan, staged, s);
    else le += launch_eval_overflow_t<FPE_R64, FPE_C64, NPFor<FPE_R64, FPE_C64>::OK, 4>(n, P, rec, plan, staged, s);
    st.mark("eval_overflow");
  }
  const long long blocks = std::min<long long>((n + 4 * 256 - 1) / (4 * 256), 148ll * 16);
#define FPE_UN(PKV, OKV) k_unsort<PKV, OKV><<<(int)blocks, 256, 0, s>>>(staged, n, pts, P, vals, exps)
  switch (pk * 4 + P.cdt) {   // the output kind follows NPFor<PK, CK>::OK
    case FPE_R64 * 4 + FPE_R64: FPE_UN(FPE_R64, FPE_R64); break;
    case FPE_R64 * 4 + FPE_C64: FPE_UN(FPE_R64, FPE_C64); break;
    case FPE_C64 * 4 + FPE_R64: FPE_UN(FPE_C64, FPE_C64); break;
    case FPE_C64 * 4 + FPE_C64: FPE_UN(FPE_C64, FPE_C64); break;
    case FPE_R32 * 4 + FPE_R32: FPE_UN(FPE_R32, FPE_R32); break;
    case FPE_R32 * 4 + FPE_C32: FPE_UN(FPE_R32, FPE_C32); break;
    case FPE_C32 * 4 + FPE_R32: FPE_UN(FPE_C32, FPE_C32); break;
    default: FPE_UN(FPE_C32, FPE_C32); break;
  }
#undef FPE_UN
  st.mark("unsort");
  return 6 + le + lm;   // hist, scan, classify, bucket windows, plan, unsort
}

}  // namespace fpe

#ifdef FPE_ITEM_TRACE
extern "C" int fpe_debug_item_trace(unsigned long long* host, int cap, int reset) {
  unsigned int n = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&n, fpe::fpe_item_trace_n, sizeof(n));
  n = n < (1u << 20) ? n : (1u << 20);
  const int m = (int)(n < (unsigned)cap ? n : (unsigned)cap);
  if (host && m) cudaMemcpyFromSymbol(host, fpe::fpe_item_trace, (size_t)m * 24);
  if (reset) { unsigned int z = 0; cudaMemcpyToSymbol(fpe::fpe_item_trace_n, &z, sizeof(z)); }
  return m;
}
#endif
