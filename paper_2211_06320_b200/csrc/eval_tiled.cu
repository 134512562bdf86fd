// eval_tiled.cu -- the bucketed, shared-memory-tiled window evaluator (north star subsystems 2-4).
//
// Pipeline (all on the caller's stream, no host round trip):
//   k_classify_bucket lines 5-8 of FPE_p per point (lambda, k_lambda, [l, r]; device_common.cuh) and
//                    a 24-bit key: bit 23 = "long window" (r - l + 1 > kSegLen), bits 0..22 monotone
//                    in lambda; per-CTA coarse-bucket histogram and slice claims (sort.cu).  l and r
//                    are both non-decreasing in lambda (d/dlambda of cover(k) + lambda k - N is
//                    k - k_lambda), so points with close keys have nested, nearly equal windows.
//   bucket scan/scatter (sort.cu) -> permutation grouped by coarse bucket, item table.
//   k_eval_tiled     persistent; items = chunks of one bucket, sorted in shared memory, then:
//     long group  = 32 consecutive long-window points, one CTA (8 warps): the union window is cut at
//                   ABSOLUTE multiples of kSegLen (a point's arithmetic depends only on its own window,
//                   so results stay bitwise independent of the batch); warp w evaluates segment t and
//                   the CTA combines the per-segment Horner partials top-down with dd-accurate powers
//                   z^gap (PAPER.md:1621-1622, 2171-2177 generalised to segment gaps).
//     short group = 32 consecutive short-window points, one warp, the whole union window.
//   Coefficients are streamed per warp through a 4-stage shared-memory ring filled by 1-D TMA bulk
//   copies (cp.async.bulk + mbarrier complete_tx) and read as warp-uniform broadcasts; lanes run a
//   predicated Horner step (fp64 / fp32 FMA) only inside their own window (exact Q_lambda, eq:reducedQlambda).
#include <cuda_runtime.h>
#include <cstdint>
#include "fpe_internal.h"
#include "fpe_math.cuh"
#include "device_common.cuh"
#include "sort.cuh"
#include "eval_tiled.cuh"
#include "kernels.cuh"

namespace fpe {

constexpr int kWarps = 8;      // warps per CTA of k_eval_tiled
constexpr int kStages = 4;     // TMA ring depth per warp
constexpr int kMergeGap = 256; // short-group windows closer than this share one streamed interval

// ------------------------------------------------------------------------------------------------
// classification + sort key + first radix upsweep
__device__ __forceinline__ uint32_t lambda_key(double lam, int l, int r) {
  uint32_t longw = (r - l + 1 > kSegLen) ? 1u : 0u;
  uint32_t u;
  if (!(lam == lam) || lam == -INFINITY) {
    u = 0;
  } else {
    double a = fabs(lam);
    uint32_t mag = 0;
    if (a >= 0x1p-52) {
      int e = frexp_exp(a);                       // a = f 2^e, f in [1/2, 1), e in [-51, 11]
      uint32_t ec = (uint32_t)(e + 52);           // 6 bits
      double f = ldexp(a, -e);
      uint32_t m16 = (uint32_t)((f - 0.5) * 131072.0);   // 16 bits
      mag = (ec << 16) | min(m16, 65535u);
    }
    u = (lam >= 0.0) ? (1u << 22) + mag : (1u << 22) - 1u - mag;
  }
  return (longw << 23) | u;
}

template <int PK>
__global__ void __launch_bounds__(256) k_classify_bucket(const void* __restrict__ pts, long long n, PolyDev P,
                                                         int2* __restrict__ lr, uint32_t* __restrict__ keys,
                                                         uint32_t* __restrict__ gcount,
                                                         uint32_t* __restrict__ cta_base,
                                                         fpe_diag* __restrict__ diag,
                                                         unsigned long long* __restrict__ hard_ctr) {
  extern __shared__ int2 s_hull[];
  __shared__ uint32_t hist[kBuckets];
  const int2* hull = P.hull;
  if (P.nv <= kSmemHullMax) {
    for (int i = threadIdx.x; i < P.nv; i += blockDim.x) s_hull[i] = P.hull[i];
    hull = s_hull;
  }
  for (int b = threadIdx.x; b < kBuckets; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const long long beg = (long long)blockIdx.x * kPtsPerCta, end = min(n, beg + kPtsPerCta);
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    double x, y;
    load_point<PK>(pts, i, x, y);
    int hard;
    double lam = lambda_cr(x, y, PtTraits<PK>::cplx, &hard);
    int istar, l, r;
    classify_lambda(hull, P.nv, P.drop, lam, istar, l, r);
    lr[i] = make_int2(l, r);
    uint32_t key = lambda_key(lam, l, r);
    keys[i] = key;
    atomicAdd(&hist[key >> (24 - kCoarseBits)], 1u);
    if (diag) {
      fpe_diag dg;
      dg.lambda = lam; dg.region = istar; dg.l = l; dg.r = r;
      dg.kept = kept_count(P, l, r); dg.hard = hard; dg.pad = 0;
      diag[i] = dg;
    }
    if (hard) atomicAdd(hard_ctr, 1ull);
  }
  __syncthreads();
  // claim this CTA's slice of every bucket
  for (int b = threadIdx.x; b < kBuckets; b += blockDim.x) {
    const uint32_t c = hist[b];
    cta_base[(size_t)blockIdx.x * kBuckets + b] = c ? atomicAdd(gcount + b, c) : 0u;
  }
}

// ------------------------------------------------------------------------------------------------
// TMA ring helpers (PTX)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t a = smem_u32(bar);
  while (!mbar_try_wait(a, parity)) {}
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

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

template <int CK>
struct WarpRing {
  using CT = typename Step<CK>::CT;
  CT* buf;            // kStages * kChunk
  uint64_t* bar;      // kStages
  const CT* coef;     // padded dense coefficient array (relative to k_min)
  uint32_t g;         // chunks consumed so far by this warp (uniform)
};

template <int CK>
__device__ __forceinline__ void ring_issue(WarpRing<CK>& R, uint32_t g, int q) {
  using CT = typename Step<CK>::CT;
  const int s = g % kStages;
  fence_proxy_async();
  mbar_expect_tx(R.bar + s, kChunk * sizeof(CT));
  tma_load_1d(R.buf + s * kChunk, R.coef + (size_t)q * kChunk, kChunk * sizeof(CT), R.bar + s);
}

// Horner over the coefficient range [lo, hi] (relative indices, descending) for the warp; each lane
// updates (br, bi) only for k in its own window [wl, wr] (empty if wl > wr).
template <int CK, bool CPLX>
__device__ __forceinline__ void stream_window(WarpRing<CK>& R, int lo, int hi, int wl, int wr,
                                              typename Step<CK>::W zr, typename Step<CK>::W zi,
                                              typename Step<CK>::W& br, typename Step<CK>::W& bi) {
  using CT = typename Step<CK>::CT;
  const int lane = threadIdx.x & 31;
  if (lo > hi) return;
  // warp-uniform range where every lane is active (empty if some lane is idle)
  const bool nonempty = wl <= wr;
  const bool all = __all_sync(0xffffffffu, nonempty);
  int F_lo = __reduce_max_sync(0xffffffffu, (unsigned)(nonempty ? wl : 0));
  int F_hi = (int)__reduce_min_sync(0xffffffffu, (unsigned)(nonempty ? wr : 0x7fffffff));
  if (!all) { F_lo = 1; F_hi = 0; }
  const int q_hi = hi / kChunk, q_lo = lo / kChunk;
  const int nq = q_hi - q_lo + 1;
  if (lane == 0)
    for (int j = 0; j < nq && j < kStages; ++j) ring_issue<CK>(R, R.g + j, q_hi - j);
  for (int j = 0; j < nq; ++j) {
    const uint32_t g = R.g + j;
    const int s = g % kStages;
    mbar_wait(R.bar + s, (g / kStages) & 1u);
    const int q = q_hi - j;
    const CT* cb = R.buf + s * kChunk - q * kChunk;   // cb[k] for k in chunk q
    const int klo = max(lo, q * kChunk), khi = min(hi, q * kChunk + kChunk - 1);
    const int a = max(klo, F_lo), b = min(khi, F_hi);
    int k = khi;
    if (a <= b) {
      for (; k > b; --k) if (k >= wl && k <= wr) horner_step<CK, CPLX>(br, bi, zr, zi, cb[k]);
#pragma unroll 8
      for (; k >= a; --k) horner_step<CK, CPLX>(br, bi, zr, zi, cb[k]);
    }
    for (; k >= klo; --k) if (k >= wl && k <= wr) horner_step<CK, CPLX>(br, bi, zr, zi, cb[k]);
    __syncwarp();
    if (lane == 0 && j + kStages < nq) ring_issue<CK>(R, g + kStages, q - kStages);
  }
  R.g += nq;
}

// (re, im) * (h + e) 2^E, scaled into range (the product is bounded by the cover argument).
__device__ __forceinline__ void mul_ext(double& re, double& im, const xc_t& p) {
  double r = __fma_rn(re, p.hr, __fma_rn(-im, p.hi, __fma_rn(re, p.er, -im * p.ei)));
  double i = __fma_rn(re, p.hi, __fma_rn(im, p.hr, __fma_rn(re, p.ei, im * p.er)));
  int sc = (int)max(-3000ll, min(3000ll, p.E));
  re = ldexp(r, sc); im = ldexp(i, sc);
}

template <int OK, bool CPLX>
__device__ __forceinline__ void finalize_point(void* vals, long long* exps, long long idx, double x, double y,
                                               double br, double bi, long long l_abs, const PolyDev& P) {
  if (x == 0.0 && y == 0.0) {   // z = 0: P(0) = a_0 (window {k_min})
    if (P.k_min != 0) { br = 0.0; bi = 0.0; }
    store_value<OK>(vals, exps, idx, br, bi, (br == 0.0 && bi == 0.0) ? 0 : P.shift);
    return;
  }
  double qr, qi;
  long long E;
  times_zpow<CPLX>(br, bi, x, y, l_abs, qr, qi, E);
  store_value<OK>(vals, exps, idx, qr, qi, E + P.shift);
}

struct LongShared {
  double hr[kWarps][32], hi[kWarps][32];
  int base[kWarps][32];
};

struct ItemShared {
  const uint32_t* gidx;
  int count, done;
};

// Long group (32 long-window points, all 8 warps): absolute segments, combined top-down by warp 0.
template <int PK, int CK, int OK>
__device__ __forceinline__ void long_group(WarpRing<CK>& R, LongShared* LS, const uint32_t* gidx, int gcount,
                                           const void* __restrict__ pts, const int2* __restrict__ lr,
                                           const PolyDev& P, void* vals, long long* exps) {
  constexpr bool CPLX = PtTraits<OK>::cplx;
  using W = typename Step<CK>::W;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int kmin = (int)P.k_min;
  const bool valid = lane < gcount;
  long long idx = 0;
  double x = 0.0, y = 0.0;
  int wl = 1, wr = 0;
  if (valid) {
    idx = __ldg(gidx + lane);
    load_point<PK>(pts, idx, x, y);
    int2 w2 = __ldg(lr + idx);
    wl = w2.x - kmin; wr = w2.y - kmin;
  }
  const int lo = (int)__reduce_min_sync(0xffffffffu, (unsigned)(valid ? wl : 0x7fffffff));
  const int hi = (int)__reduce_max_sync(0xffffffffu, (unsigned)(valid ? wr : 0));
  const int T_lo = lo / kSegLen, T_hi = hi / kSegLen;
  double acc_r = 0.0, acc_i = 0.0;
  int last_base = 0;
  bool started = false;
  xc_t zL;
  if (wib == 0 && valid) zL = xc_pow(x, y, kSegLen);
  for (int tb = T_hi; tb >= T_lo; tb -= kWarps) {
    const int t = tb - wib;
    if (t >= T_lo) {
      const int s_lo = t * kSegLen, s_hi = s_lo + kSegLen - 1;
      const int swl = max(wl, s_lo), swr = min(wr, s_hi);
      W br = 0, bi = 0;
      stream_window<CK, CPLX>(R, max(lo, s_lo), min(hi, s_hi), swl, swr, (W)x, (W)y, br, bi);
      LS->hr[wib][lane] = (double)br;
      LS->hi[wib][lane] = (double)bi;
      LS->base[wib][lane] = (swl <= swr) ? swl : -1;
    }
    __syncthreads();
    if (wib == 0 && valid) {
      for (int ww = 0; ww < kWarps && tb - ww >= T_lo; ++ww) {
        const int base = LS->base[ww][lane];
        if (base < 0) continue;
        const double hr = LS->hr[ww][lane], hi_ = LS->hi[ww][lane];
        if (!started) {
          acc_r = hr; acc_i = hi_; started = true;
        } else {
          const int gap = last_base - base;
          if (gap == kSegLen) mul_ext(acc_r, acc_i, zL);
          else { xc_t zg = xc_pow(x, y, gap); mul_ext(acc_r, acc_i, zg); }
          acc_r += hr; acc_i += hi_;
        }
        last_base = base;
      }
    }
    __syncthreads();
  }
  if (wib == 0 && valid)
    finalize_point<OK, CPLX>(vals, exps, idx, x, y, acc_r, acc_i, (long long)last_base + kmin, P);
}

// Short group (32 short-window points, one warp): the union processed as merged intervals (windows
// closer than kMergeGap share one streamed interval; several intervals only where the key order
// jumps, e.g. across the lambda range of the long windows).
template <int PK, int CK, int OK>
__device__ __forceinline__ void short_group(WarpRing<CK>& R, const uint32_t* gidx, int gcount,
                                            const void* __restrict__ pts, const int2* __restrict__ lr,
                                            const PolyDev& P, void* vals, long long* exps) {
  constexpr bool CPLX = PtTraits<OK>::cplx;
  using W = typename Step<CK>::W;
  const int lane = threadIdx.x & 31;
  const int kmin = (int)P.k_min;
  const bool valid = lane < gcount;
  long long idx = 0;
  double x = 0.0, y = 0.0;
  int wl = 1, wr = 0, l_abs = 0;
  if (valid) {
    idx = __ldg(gidx + lane);
    load_point<PK>(pts, idx, x, y);
    int2 w2 = __ldg(lr + idx);
    l_abs = w2.x;
    wl = w2.x - kmin; wr = w2.y - kmin;
  }
  W br = 0, bi = 0;
  const bool act = valid && wl <= wr;
  unsigned pending = __ballot_sync(0xffffffffu, act);
  while (pending) {
    const bool pend = (pending >> lane) & 1u;
    const int top = (int)__reduce_max_sync(0xffffffffu, pend ? (unsigned)wr : 0u);
    int lo = (int)__reduce_min_sync(0xffffffffu, (pend && wr == top) ? (unsigned)wl : 0x7fffffffu);
    for (;;) {
      const bool in = pend && wr >= lo - kMergeGap;
      const int lo2 = (int)__reduce_min_sync(0xffffffffu, in ? (unsigned)wl : 0x7fffffffu);
      if (lo2 >= lo) break;
      lo = lo2;
    }
    const bool mine = pend && wr >= lo - kMergeGap;
    stream_window<CK, CPLX>(R, lo, top, mine ? wl : 1, mine ? wr : 0, (W)x, (W)y, br, bi);
    pending &= ~__ballot_sync(0xffffffffu, mine);
  }
  if (valid) {
    if (wl > wr) {   // non-finite point
      double nan = __longlong_as_double(0x7ff8000000000000LL);
      store_value<OK>(vals, exps, idx, nan, CPLX ? nan : 0.0, 0);
    } else {
      finalize_point<OK, CPLX>(vals, exps, idx, x, y, (double)br, (double)bi, l_abs, P);
    }
  }
}

template <int CK>
constexpr size_t ring_bytes() {
  return (size_t)kWarps * kStages * kChunk * sizeof(typename Step<CK>::CT);
}

// Persistent evaluator.  Work items are the 32-point group slots of the sorted chunks (64 per
// chunk): long-bucket slots first, each taken by a whole CTA (long_group), then short-bucket slots,
// each taken by one warp (short_group); both fetched with global atomic counters.
template <int PK, int CK, int OK>
__global__ void __launch_bounds__(kWarps * 32, 3) k_eval_tiled(const void* __restrict__ pts, long long n, PolyDev P,
                                                               const int2* __restrict__ lr,
                                                               const uint32_t* __restrict__ perm,
                                                               const uint32_t* __restrict__ gcount,
                                                               const uint32_t* __restrict__ bstart,
                                                               const uint32_t* __restrict__ istart,
                                                               uint32_t* __restrict__ ctrs, void* __restrict__ vals,
                                                               long long* __restrict__ exps) {
  using CT = typename Step<CK>::CT;
  constexpr int kSlots = kChunkPts / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  CT* ring_buf = reinterpret_cast<CT*>(smem) + (size_t)wib * kStages * kChunk;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ring_bytes<CK>()) + wib * kStages;
  LongShared* LS = reinterpret_cast<LongShared*>(smem + ring_bytes<CK>() + kWarps * kStages * sizeof(uint64_t));
  ItemShared* IS = reinterpret_cast<ItemShared*>(reinterpret_cast<unsigned char*>(LS) + sizeof(LongShared));
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  WarpRing<CK> R{ring_buf, bars, static_cast<const CT*>(P.coef), 0u};
  const int n_long_chunks = (int)istart[kBuckets / 2];
  const int n_chunks = (int)istart[kBuckets];
  const long long n_long_items = (long long)n_long_chunks * kSlots;
  const long long n_short_items = (long long)(n_chunks - n_long_chunks) * kSlots;

  for (;;) {   // long-window groups: whole CTA
    if (threadIdx.x == 0) {
      const long long it = atomicAdd(ctrs + 0, 1u);
      IS->done = it >= n_long_items;
      IS->count = 0;
      if (!IS->done) {
        int bucket, npts;
        uint32_t p0;
        chunk_of(istart, gcount, bstart, (int)(it / kSlots), bucket, p0, npts);
        const int slot = (int)(it % kSlots);
        IS->count = max(0, min(32, npts - 32 * slot));
        IS->gidx = perm + p0 + 32 * slot;
      }
    }
    __syncthreads();
    const int done = IS->done, count = IS->count;
    const uint32_t* gidx = IS->gidx;
    __syncthreads();
    if (done) break;
    if (count > 0) long_group<PK, CK, OK>(R, LS, gidx, count, pts, lr, P, vals, exps);
  }
  for (;;) {   // short-window groups: one warp each
    long long it = 0;
    if (lane == 0) it = atomicAdd(ctrs + 1, 1u);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= n_short_items) break;
    int bucket, npts;
    uint32_t p0;
    chunk_of(istart, gcount, bstart, n_long_chunks + (int)(it / kSlots), bucket, p0, npts);
    const int slot = (int)(it % kSlots);
    const int count = min(32, npts - 32 * slot);
    if (count > 0) short_group<PK, CK, OK>(R, perm + p0 + 32 * slot, count, pts, lr, P, vals, exps);
  }
}

// ------------------------------------------------------------------------------------------------
// host side
static inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t n_ctas(long long n) { return (size_t)((n + kPtsPerCta - 1) / kPtsPerCta); }

size_t tiled_ws_bytes(long long n) {
  return al256(n * sizeof(int2)) + 2 * al256(n * sizeof(uint32_t)) +
         al256(n_ctas(n) * kBuckets * sizeof(uint32_t)) + 3 * al256((kBuckets + 1) * sizeof(uint32_t)) + 256;
}

template <int CK>
static size_t eval_smem() {
  return ring_bytes<CK>() + kWarps * kStages * sizeof(uint64_t) + sizeof(LongShared) + sizeof(ItemShared);
}

template <int PK, int CK, int OK>
static int launch_eval_tiled_t(const void* pts, long long n, const PolyDev& P, const int2* lr,
                               const uint32_t* perm, const uint32_t* gcount, const uint32_t* bstart,
                               const uint32_t* istart, uint32_t* ctrs, void* vals, long long* exps, cudaStream_t s) {
  static int grid = 0;
  const size_t smem = eval_smem<CK>();
  if (grid == 0) {
    cudaFuncSetAttribute(k_eval_tiled<PK, CK, OK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_eval_tiled<PK, CK, OK>, kWarps * 32, smem);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = max(1, per_sm) * sms;
  }
  k_eval_tiled<PK, CK, OK><<<grid, kWarps * 32, smem, s>>>(pts, n, P, lr, perm, gcount, bstart, istart,
                                                             ctrs, vals, exps);
  return 1;
}

template <int PK, int CK>
static int dispatch_eval(const void* pts, long long n, const PolyDev& P, const int2* lr,
                         const uint32_t* perm, const uint32_t* gcount, const uint32_t* bstart, const uint32_t* istart,
                         uint32_t* ctrs, void* vals, long long* exps, cudaStream_t s) {
  constexpr bool cplx = PtTraits<PK>::cplx || PtTraits<CK>::cplx;
  constexpr int OK = PtTraits<CK>::f32 ? (cplx ? FPE_C32 : FPE_R32) : (cplx ? FPE_C64 : FPE_R64);
  return launch_eval_tiled_t<PK, CK, OK>(pts, n, P, lr, perm, gcount, bstart, istart, ctrs, vals, exps, s);
}

template <int PK>
static void launch_classify_bucket_t(const void* pts, long long n, const PolyDev& P, int2* lr, uint32_t* keys,
                                     uint32_t* gcount, uint32_t* cta_base, fpe_diag* diag, unsigned long long* hard,
                                     cudaStream_t s) {
  size_t smem = P.nv <= kSmemHullMax ? P.nv * sizeof(int2) : 0;
  k_classify_bucket<PK><<<(int)n_ctas(n), 256, smem, s>>>(pts, n, P, lr, keys, gcount, cta_base, diag, hard);
}

int run_tiled(int pk, const void* pts, long long n, const PolyDev& P, void* vals, long long* exps,
              fpe_diag* diag, void* ws, unsigned long long* hard, Stage& st, cudaStream_t s) {
  char* p = static_cast<char*>(ws);
  int2* lr = reinterpret_cast<int2*>(p); p += al256(n * sizeof(int2));
  uint32_t* keys = reinterpret_cast<uint32_t*>(p); p += al256(n * 4);
  uint32_t* perm = reinterpret_cast<uint32_t*>(p); p += al256(n * 4);
  uint32_t* cta_base = reinterpret_cast<uint32_t*>(p); p += al256(n_ctas(n) * kBuckets * 4);
  uint32_t* gcount = reinterpret_cast<uint32_t*>(p); p += al256((kBuckets + 1) * 4);
  uint32_t* bstart = reinterpret_cast<uint32_t*>(p); p += al256((kBuckets + 1) * 4);
  uint32_t* istart = reinterpret_cast<uint32_t*>(p); p += al256((kBuckets + 1) * 4);
  uint32_t* ctrs = reinterpret_cast<uint32_t*>(p);
  cudaMemsetAsync(gcount, 0, (kBuckets + 1) * 4, s);
  cudaMemsetAsync(ctrs, 0, 16, s);
  switch (pk) {
    case FPE_R64: launch_classify_bucket_t<FPE_R64>(pts, n, P, lr, keys, gcount, cta_base, diag, hard, s); break;
    case FPE_C64: launch_classify_bucket_t<FPE_C64>(pts, n, P, lr, keys, gcount, cta_base, diag, hard, s); break;
    case FPE_R32: launch_classify_bucket_t<FPE_R32>(pts, n, P, lr, keys, gcount, cta_base, diag, hard, s); break;
    default: launch_classify_bucket_t<FPE_C32>(pts, n, P, lr, keys, gcount, cta_base, diag, hard, s); break;
  }
  st.mark("classify");
  bucket_finish(keys, n, gcount, cta_base, bstart, istart, perm, s);
  st.mark("bucket");
  int le = 0;
#define FPE_EV(PKV, CKV) \
  le = dispatch_eval<PKV, CKV>(pts, n, P, lr, perm, gcount, bstart, istart, ctrs, vals, exps, s)
  switch (pk * 4 + P.cdt) {
    case FPE_R64 * 4 + FPE_R64: FPE_EV(FPE_R64, FPE_R64); break;
    case FPE_R64 * 4 + FPE_C64: FPE_EV(FPE_R64, FPE_C64); break;
    case FPE_C64 * 4 + FPE_R64: FPE_EV(FPE_C64, FPE_R64); break;
    case FPE_C64 * 4 + FPE_C64: FPE_EV(FPE_C64, FPE_C64); break;
    case FPE_R32 * 4 + FPE_R32: FPE_EV(FPE_R32, FPE_R32); break;
    case FPE_R32 * 4 + FPE_C32: FPE_EV(FPE_R32, FPE_C32); break;
    case FPE_C32 * 4 + FPE_R32: FPE_EV(FPE_C32, FPE_R32); break;
    case FPE_C32 * 4 + FPE_C32: FPE_EV(FPE_C32, FPE_C32); break;
    default: return -1;
  }
#undef FPE_EV
  st.mark("eval_tiled");
  return 4 + le;
}

}  // namespace fpe
