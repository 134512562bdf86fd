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
#include <algorithm>
#include <cstdint>
#include "sort.cuh"
#include "fpe_internal.h"

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

__device__ __forceinline__ double2 load_point_any(int pk, const void* __restrict__ p, long long i) {
  switch (pk) {
    case FPE_R64: return make_double2(__ldg(static_cast<const double*>(p) + i), 0.0);
    case FPE_C64: return __ldg(static_cast<const double2*>(p) + i);
    case FPE_R32: return make_double2((double)__ldg(static_cast<const float*>(p) + i), 0.0);
    default: { const float2 v = __ldg(static_cast<const float2*>(p) + i); return make_double2(v.x, v.y); }
  }
}

// Records to bucket positions: bucket start + the classifying CTA's slice of the bucket + the point's rank
// in that slice (both from the classifier) -- a pure streaming pass over all points, no atomics.
__global__ void __launch_bounds__(256) k_bucket_scatter(const uint2* __restrict__ keys, const int2* __restrict__ lr,
                                                        long long n, long long ppc,
                                                        const uint32_t* __restrict__ bstart,
                                                        const uint32_t* __restrict__ cta_base,
                                                        PtRec* __restrict__ rec) {
  constexpr int U = 4;   // independent loads in flight per thread
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    uint2 kr[U];
    int2 w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + u * stride;
      if (i < n) { kr[u] = __ldg(keys + i); w[u] = __ldg(lr + i); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + u * stride;
      if (i < n) {
        const uint32_t c = kr[u].x >> (24 - kCoarseBits);
        const uint32_t pos = __ldg(bstart + c) + __ldg(cta_base + (size_t)(i / ppc) * kBuckets + c) + kr[u].y;
        rec[pos] = PtRec{(int32_t)i, kr[u].x, w[u].x, w[u].y};
      }
    }
  }
}

// Counting sort of every chunk of the records by key bits [1, 1 + kLocalBits), in place: afterwards the
// records (and the windows slr, for the planner) are ordered by key bits 1..23 (buckets are laid out in
// key order), so that every later pass reads them coalesced.
constexpr size_t kChunkSortSmem = (size_t)kChunkPts * (sizeof(PtRec) + sizeof(uint16_t)) +
                                  (1u << kLocalBits) * sizeof(uint32_t);
__global__ void __launch_bounds__(256) k_chunk_sort(PtRec* __restrict__ rec, int2* __restrict__ slr, int pk,
                                                    const void* __restrict__ pts, double2* __restrict__ zs,
                                                    const uint32_t* __restrict__ gcount,
                                                    const uint32_t* __restrict__ bstart,
                                                    const uint32_t* __restrict__ istart) {
  extern __shared__ __align__(16) unsigned char sm[];
  PtRec* s_rec = reinterpret_cast<PtRec*>(sm);
  uint16_t* s_dst = reinterpret_cast<uint16_t*>(sm + (size_t)kChunkPts * sizeof(PtRec));
  uint32_t* hist = reinterpret_cast<uint32_t*>(sm + (size_t)kChunkPts * (sizeof(PtRec) + sizeof(uint16_t)));
  const int c = blockIdx.x;
  if (c >= (int)istart[kBuckets]) return;
  int bucket, npts;
  uint32_t p0;
  chunk_of(istart, gcount, bstart, c, bucket, p0, npts);
  for (int b = threadIdx.x; b < (1 << kLocalBits); b += blockDim.x) hist[b] = 0;
  // records in (coalesced), staged in shared memory
  for (int j = threadIdx.x; j < npts; j += 256)
    reinterpret_cast<int4*>(s_rec)[j] = __ldg(reinterpret_cast<const int4*>(rec + p0 + j));
  __syncthreads();
  constexpr int kPer = kChunkPts / 256;
  uint32_t my_bin[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int j = threadIdx.x + q * 256;
    my_bin[q] = 0;
    if (j < npts) {
      my_bin[q] = (s_rec[j].key >> 1) & ((1u << kLocalBits) - 1);
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
    if (j < npts) s_dst[j] = (uint16_t)atomicAdd(&hist[my_bin[q]], 1u);
  }
  __syncthreads();
  // records out to their sorted positions inside the chunk (the chunk's lines complete in L2), with the
  // points gathered into the same order (independent random loads issued together)
  double2 z[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int j = threadIdx.x + q * 256;
    if (j < npts) z[q] = load_point_any(pk, pts, s_rec[j].idx);
  }
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int j = threadIdx.x + q * 256;
    if (j < npts) {
      const int d = s_dst[j];
      rec[p0 + d] = s_rec[j];
      slr[p0 + d] = make_int2(s_rec[j].l, s_rec[j].r);
      zs[p0 + d] = z[q];
    }
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

void bucket_finish(const uint2* keys, int2* lr, long long n, long long ppc, const uint32_t* gcount,
                   const uint32_t* cta_base, uint32_t* bstart, uint32_t* istart, PtRec* rec, int pk,
                   const void* pts, double2* zs, long long k_min, const Plan& plan, cudaStream_t s) {
  k_bucket_scan<<<1, 1024, 0, s>>>(gcount, bstart, istart);
  const long long blocks = std::min<long long>((n + 4 * 256 - 1) / (4 * 256), 148ll * 32);
  k_bucket_scatter<<<(int)blocks, 256, 0, s>>>(keys, lr, n, ppc, bstart, cta_base, rec);
  // the sorted windows are written over lr: k_chunk_sort reads only the records
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_chunk_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kChunkSortSmem);
    attr = true;
  }
  k_chunk_sort<<<(int)max_chunks(n), 256, kChunkSortSmem, s>>>(rec, lr, pk, pts, zs, gcount, bstart, istart);
  const long long groups = (n + plan.gsize - 1) / plan.gsize;
  k_plan<<<(int)((groups + 7) / 8), 256, 0, s>>>(n, lr, k_min, plan);
}

}  // namespace fpe
