// sort.cu -- work bucketing (north star subsystem 3).
//
// Points carry a 23-bit key that is monotone in an fp64 estimate of lambda (eval_tiled.cu bucket_key); l and
// r are both non-decreasing in lambda, so points with close keys have nested, nearly equal windows.  One
// counting sort by the top coarse_bits(n) key bits (32768 buckets from 2^20 points up): k_bucket_hist
// (eval_tiled.cu) builds a per-CTA histogram in shared memory and claims each CTA's slice of every bucket
// with one global atomicAdd per nonzero bin; k_bucket_scan turns bucket totals into starts;
// k_classify_bucket (eval_tiled.cu) classifies the same points and writes every record {index, key, l, r, z}
// to bucket start + its CTA's slice + a shared-memory counter; k_bucket_windows bounds the windows of every
// bucket's points; k_plan cuts the bucket order into groups of 32*NP points and plans their work items.
// Order inside a (CTA, bucket) slice is unspecified; every point's arithmetic depends only on its own
// window, so results do not depend on it (bitwise).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include "sort.cuh"
#include "fpe_internal.h"
#include "mma_piece.cuh"

namespace fpe {

// Exclusive scan of the kBuckets bucket totals into bucket starts (one CTA; buckets are laid out in
// key order, so the record array ends up sorted by the top kCoarseBits of the key).
__global__ void __launch_bounds__(1024) k_bucket_scan(const uint32_t* __restrict__ gcount,
                                                      uint32_t* __restrict__ bstart, int cb) {
  constexpr int kPer = kBuckets / 1024;
  const int per = (1 << cb) / 1024;   // buckets per thread (cb >= 10)
  __shared__ uint32_t ws[32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  uint32_t c[kPer];
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) { c[j] = j < per ? gcount[t * per + j] : 0u; s += c[j]; }
  uint32_t x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
  if (lane == 31) ws[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t z = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, z, o); if (lane >= o) z += y; }
    ws[lane] = z;
  }
  __syncthreads();
  uint32_t run = (wid ? ws[wid - 1] : 0) + x - s;
#pragma unroll
  for (int j = 0; j < kPer; ++j) if (j < per) { bstart[t * per + j] = run; run += c[j]; }
}

// The evaluator's work plan: groups of gsize consecutive points in bucket order (across bucket
// boundaries: neighbouring buckets hold neighbouring lambdas), one warp per group, one thread here per group.
// A group's union window is bounded by its buckets' window bounds (k_bucket_windows: l and r are
// non-decreasing in lambda, so [l of its first bucket, r of its last] contains every point's window) -- no
// pass over the records.  Within a bucket the points are in no particular order, so a group inside one bucket
// spans nearly the bucket's whole lambda range anyway: the bound is essentially the exact union.  Then either
// one single item (one warp, pieces in order) or npieces parallel items with scratch slots for their
// partials (windows longer than kPiece), plus a tensor-core item for every whole piece of the union when some
// point of the group could be in mma_covers' |z| range (the evaluators test each point exactly).
__device__ __forceinline__ int bucket_of(const uint32_t* __restrict__ bstart, int nbk, uint32_t pos) {
  int lo = 0, hi = nbk;   // the last bucket whose start is <= pos (empty buckets before it share its start)
  while (hi - lo > 1) { const int m = (lo + hi) >> 1; if (__ldg(bstart + m) <= pos) lo = m; else hi = m; }
  return lo;
}

__global__ void __launch_bounds__(256) k_plan(long long n, const uint32_t* __restrict__ bstart, int nbk,
                                              const int4* __restrict__ bwin, Plan plan) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int gs = plan.gsize;
  const long long first = g * gs;
  if (first >= n) return;
  const int count = (int)min((long long)gs, n - first);
  const int4 wf = __ldg(bwin + bucket_of(bstart, nbk, (uint32_t)first));
  const int4 wl = __ldg(bwin + bucket_of(bstart, nbk, (uint32_t)(first + count - 1)));
  const int lo = wf.x, hi = wl.y;
  int clo = 0x7fffffff, chi = -1;
  if (plan.mma_on && hi >= lo && !wf.w && !wl.z) {   // some point may have 2^-3 <= max(|x|, |y|) < 2^3
    clo = (lo + kPiece - 1) / kPiece;
    chi = (hi + 1) / kPiece - 1;
  }
  GroupDesc d;
  d.p0 = (uint32_t)first;
  d.count = count;
  d.lo = lo; d.hi = hi; d.slot = 0; d.npieces = 1;
  d.mma_p0 = 0; d.mma_np = 0; d.mma_slot = 0; d.listed = 0;
  if (clo <= chi) {
    const int np = chi - clo + 1;
    d.mma_p0 = clo; d.mma_np = np;
    atomicAdd(plan.stats + kStatMmaItems, (unsigned long long)np);
    const uint32_t base = atomicAdd(plan.mma_ctrs, (uint32_t)np);
    if ((unsigned long long)base + np <= plan.mma_cap) {
      d.mma_slot = base;
      for (int i = 0; i < np; ++i) plan.mma_items[base + i] = make_uint2((uint32_t)g, (uint32_t)(clo + i));
    } else {   // DMMA scratch exhausted: k_eval_overflow runs the same DMMA passes in-warp (bitwise equal)
      d.mma_slot = kMmaInWarp;
      atomicAdd(plan.stats + kStatMmaInWarp, (unsigned long long)np);
      plan.ovf_groups[atomicAdd(plan.mma_ctrs + 2, 1u)] = (uint32_t)g;
      for (uint32_t i = base; i < plan.mma_cap && i < base + (uint32_t)np; ++i) plan.mma_items[i] = make_uint2(~0u, 0u);
    }
  }
  if (hi >= lo && hi - lo + 1 > kPiece && d.mma_slot != kMmaInWarp) {   // (overflow groups: one warp each)
    const int np = hi / kPiece - lo / kPiece + 1;
    const uint32_t base = atomicAdd(plan.ctrs + 2, (uint32_t)np);
    if ((unsigned long long)base + np <= plan.cap) {
      d.slot = base; d.npieces = np;
      plan.gcnt[g] = 0;
      atomicAdd(plan.stats + kStatPieceItems, (unsigned long long)np);
      for (int i = 0; i < np; ++i) plan.items[base + i] = make_uint2((uint32_t)g, (uint32_t)(lo / kPiece + i));
    } else {   // scratch exhausted: evaluated serially by one warp (bitwise the same result)
      atomicAdd(plan.stats + kStatPieceSerial, 1ull);
      for (uint32_t i = base; i < plan.cap && i < base + (uint32_t)np; ++i) plan.items[i] = make_uint2(~0u, 0u);
    }
  }
  if (FPE_LONG_FIRST && d.npieces == 1 && d.mma_slot != kMmaInWarp && hi >= lo && hi - lo + 1 > kLongWin) {
    d.listed = 1;   // the largest single items first, so that the persistent evaluator's tail is short
    if (FPE_LONG_WIN2 == 0 || hi - lo + 1 > FPE_LONG_WIN2) plan.long_groups[atomicAdd(plan.ctrs + 3, 1u)] = (uint32_t)g;
    else plan.long_groups[plan.ngroups - 1 - atomicAdd(plan.ctrs + 8, 1u)] = (uint32_t)g;
  }
  plan.desc[g] = d;
}

void bucket_scan(const uint32_t* gcount, uint32_t* bstart, long long n, cudaStream_t s) {
  k_bucket_scan<<<1, 1024, 0, s>>>(gcount, bstart, coarse_bits(n));
}

void plan_groups(long long n, const uint32_t* bstart, const int4* bwin, const Plan& plan, cudaStream_t s) {
  const long long groups = (n + plan.gsize - 1) / plan.gsize;
  k_plan<<<(int)((groups + 255) / 256), 256, 0, s>>>(n, bstart, 1 << coarse_bits(n), bwin, plan);
}

}  // namespace fpe
