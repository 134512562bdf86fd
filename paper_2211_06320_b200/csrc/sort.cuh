// sort.cuh -- work bucketing by a lambda-monotone key (sort.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fpe {
constexpr int kCoarseBits = 12;                 // global buckets: top 12 of the 24 key bits
constexpr int kBuckets = 1 << kCoarseBits;
constexpr int kPtsPerCta = 32768;               // points per CTA of classify / scatter
constexpr int kChunkPts = 2048;                 // points per evaluator work item (one bucket's slice)
constexpr int kLocalBits = 11;                  // in-chunk counting sort on key bits [1, 12)

// Locate work-item chunk c (item order, long buckets first): its bucket, first position in the
// permutation and its number of points.
__device__ __forceinline__ void chunk_of(const uint32_t* istart, const uint32_t* gcount, const uint32_t* bstart,
                                         int c, int& bucket, uint32_t& p0, int& npts) {
  int a = 0, b = kBuckets - 1;   // position b' with istart[b'] <= c < istart[b'+1]
  while (a < b) { int m = (a + b + 1) >> 1; if (istart[m] <= (uint32_t)c) a = m; else b = m - 1; }
  bucket = (a + kBuckets / 2) % kBuckets;
  const uint32_t off = (uint32_t)(c - (int)istart[a]) * kChunkPts;
  p0 = bstart[bucket] + off;
  npts = (int)min((uint32_t)kChunkPts, gcount[bucket] - off);
}
// bucket starts + item table (k_bucket_scan), the permutation (k_bucket_scatter) and the in-chunk
// order (k_chunk_sort)
void bucket_finish(const uint32_t* keys, long long n, const uint32_t* gcount, const uint32_t* cta_base,
                   uint32_t* bstart, uint32_t* istart, uint32_t* perm, cudaStream_t s);
}  // namespace fpe
