// sort.cu -- work bucketing (north star subsystem 3).
//
// Points carry a 24-bit key that is monotone in lambda (bits 0..22) with bit 23 = "long window";
// l and r are both non-decreasing in lambda, so points with close keys have nested, nearly equal
// windows.  Two levels:
//   global  : one counting-sort scatter by the top kCoarseBits of the key (4096 coarse buckets).
//             k_classify_bucket (eval_tiled.cu) builds a per-CTA histogram in shared memory and
//             claims each CTA's slice of every bucket with one global atomicAdd per nonzero bin;
//             k_bucket_scan turns bucket totals into starts and enumerates work items (chunks of at
//             most kChunkPts points of one bucket, long buckets first); k_bucket_scatter writes the
//             records {index, key, l, r} in bucket order (contiguous runs per (CTA, bucket), so L2
//             merges the partial sectors).
//   local   : k_chunk_sort sorts each chunk by the remaining low bits in shared memory (counting
//             sort); k_plan cuts the sorted permutation into groups of 32*NP points and plans their
//             work items.
// Order inside a (CTA, bucket) run and inside equal keys is unspecified; every point's arithmetic
// depends only on its own window, so results do not depend on it (bitwise).
#include <cuda_runtime.h>
#include <cstdint>
#include "sort.cuh"

namespace fpe {

__global__ void __launch_bounds__(1024) k_bucket_scan(const uint32_t* __restrict__ gcount,
                                                      uint32_t* __restrict__ bstart,
                                                      uint32_t* __restrict__ istart) {
  // kBuckets = 4096 = 1024 threads x 4
  __shared__ uint32_t ws[32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  uint32_t c[4], ch[4];
  uint32_t s = 0, sc = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    c[j] = gcount[t * 4 + j];
    s += c[j];
  }
  // item order: long buckets (top half) first -> position b' holds bucket (b' + half) % kBuckets
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t b = (uint32_t)((t * 4 + j + kBuckets / 2) % kBuckets);
    ch[j] = (gcount[b] + kChunkPts - 1) / kChunkPts;
    sc += ch[j];
  }
  // two block scans (bucket starts, item starts)
  uint32_t v[2] = {s, sc}, ex[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    uint32_t x = v[q];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t z = ws[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += y;
      }
      ws[lane] = z;
    }
    __syncthreads();
    ex[q] = (wid ? ws[wid - 1] : 0) + x - v[q];
    if (q == 1 && t == 1023) istart[kBuckets] = ws[31];
    __syncthreads();
  }
  uint32_t run = ex[0], runi = ex[1];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    bstart[t * 4 + j] = run;
    run += c[j];
    istart[t * 4 + j] = runi;
    runi += ch[j];
  }
}

__global__ void __launch_bounds__(256) k_bucket_scatter(const uint32_t* __restrict__ keys,
                                                        const int2* __restrict__ lr, long long n,
                                                        const uint32_t* __restrict__ bstart,
                                                        const uint32_t* __restrict__ cta_base,
                                                        int4* __restrict__ rec) {
  __shared__ uint32_t cnt[kBuckets];
  __shared__ uint32_t base[kBuckets];
  for (int b = threadIdx.x; b < kBuckets; b += blockDim.x) {
    cnt[b] = 0;
    base[b] = bstart[b] + cta_base[(size_t)blockIdx.x * kBuckets + b];
  }
  __syncthreads();
  const long long beg = (long long)blockIdx.x * kPtsPerCta;
  const long long end = min(n, beg + kPtsPerCta);
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    const uint32_t key = __ldg(keys + i);
    const int2 w = __ldg(lr + i);
    const uint32_t c = key >> (24 - kCoarseBits);
    const uint32_t r = atomicAdd(&cnt[c], 1u);
    rec[base[c] + r] = make_int4((int)i, (int)key, w.x, w.y);
  }
}

// Counting sort of every chunk of the records by key bits [1, 1 + kLocalBits): afterwards the point
// indices (perm) and their windows (slr) are ordered by key bits 1..23 (buckets are laid out in key
// order), and every later pass reads them coalesced.
__global__ void __launch_bounds__(256) k_chunk_sort(const int4* __restrict__ rec, uint32_t* __restrict__ perm,
                                                    int2* __restrict__ slr,
                                                    const uint32_t* __restrict__ gcount,
                                                    const uint32_t* __restrict__ bstart,
                                                    const uint32_t* __restrict__ istart) {
  __shared__ uint32_t hist[1 << kLocalBits];
  __shared__ uint32_t s_idx[kChunkPts];
  __shared__ int2 s_lr[kChunkPts];
  const int c = blockIdx.x;
  if (c >= (int)istart[kBuckets]) return;
  int bucket, npts;
  uint32_t p0;
  chunk_of(istart, gcount, bstart, c, bucket, p0, npts);
  for (int b = threadIdx.x; b < (1 << kLocalBits); b += blockDim.x) hist[b] = 0;
  __syncthreads();
  constexpr int kPer = kChunkPts / 256;
  int4 my[kPer];
  uint32_t my_bin[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int j = threadIdx.x + q * 256;
    my_bin[q] = 0;
    if (j < npts) {
      my[q] = __ldg(rec + p0 + j);
      my_bin[q] = ((uint32_t)my[q].y >> 1) & ((1u << kLocalBits) - 1);
      atomicAdd(&hist[my_bin[q]], 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {   // exclusive scan of the bins (2048 = 32 lanes x 64)
    const int lane = threadIdx.x;
    constexpr int kB = (1 << kLocalBits) / 32;
    uint32_t run = 0;
    for (int j = 0; j < kB; ++j) run += hist[lane * kB + j];
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { uint32_t y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
    uint32_t off = x - run;
    for (int j = 0; j < kB; ++j) { uint32_t v = hist[lane * kB + j]; hist[lane * kB + j] = off; off += v; }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int j = threadIdx.x + q * 256;
    if (j < npts) {
      const uint32_t d = atomicAdd(&hist[my_bin[q]], 1u);
      s_idx[d] = (uint32_t)my[q].x;
      s_lr[d] = make_int2(my[q].z, my[q].w);
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < npts; j += 256) {
    perm[p0 + j] = s_idx[j];
    slr[p0 + j] = s_lr[j];
  }
}

// The evaluator's work plan: groups of gsize consecutive points of the sorted permutation (across
// bucket boundaries: neighbouring buckets hold neighbouring lambdas), one warp per group: the union
// of the windows and either one single item (one warp, pieces in order) or npieces parallel items
// with scratch slots for their partials (windows longer than kPiece).
__global__ void __launch_bounds__(256) k_plan(long long n, const int2* __restrict__ slr, long long k_min,
                                              Plan plan) {
  const int lane = threadIdx.x & 31;
  const long long g = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int gs = plan.gsize;
  const long long first = g * gs;
  if (first >= n) return;
  const int count = (int)min((long long)gs, n - first);
  int lo = 0x7fffffff, hi = -1;
  for (int j = lane; j < count; j += 32) {
    const int2 w2 = __ldg(slr + first + j);
    if (w2.y >= w2.x) {
      lo = min(lo, (int)(w2.x - k_min));
      hi = max(hi, (int)(w2.y - k_min));
    }
  }
  lo = (int)__reduce_min_sync(0xffffffffu, (unsigned)lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if (lane != 0) return;
  GroupDesc d;
  d.p0 = (uint32_t)first;
  d.count = count;
  d.lo = lo; d.hi = hi; d.slot = 0; d.npieces = 1;
  bool single = true;
  if (hi >= lo && hi - lo + 1 > kPiece) {
    const int np = hi / kPiece - lo / kPiece + 1;
    const uint32_t base = atomicAdd(plan.ctrs + 2, (uint32_t)np);
    if ((unsigned long long)base + np <= plan.cap) {
      d.slot = base; d.npieces = np;
      plan.gcnt[g] = 0;
      for (int i = 0; i < np; ++i) plan.items[base + i] = make_uint2((uint32_t)g, (uint32_t)(lo / kPiece + i));
      single = false;
    } else {   // scratch exhausted: evaluated serially by one warp (bitwise the same result)
      for (uint32_t i = base; i < plan.cap && i < base + (uint32_t)np; ++i) plan.items[i] = make_uint2(~0u, 0u);
    }
  }
  plan.desc[g] = d;
  (void)single;
}

void bucket_finish(const uint32_t* keys, int2* lr, long long n, const uint32_t* gcount, const uint32_t* cta_base,
                   uint32_t* bstart, uint32_t* istart, int4* rec, uint32_t* perm, long long k_min,
                   const Plan& plan, cudaStream_t s) {
  k_bucket_scan<<<1, 1024, 0, s>>>(gcount, bstart, istart);
  const int ctas = (int)((n + kPtsPerCta - 1) / kPtsPerCta);
  k_bucket_scatter<<<ctas, 256, 0, s>>>(keys, lr, n, bstart, cta_base, rec);
  // perm and slr may alias keys and lr: k_chunk_sort reads only the records
  k_chunk_sort<<<(int)max_chunks(n), 256, 0, s>>>(rec, perm, lr, gcount, bstart, istart);
  const long long groups = (n + plan.gsize - 1) / plan.gsize;
  k_plan<<<(int)((groups + 7) / 8), 256, 0, s>>>(n, lr, k_min, plan);
}

}  // namespace fpe
