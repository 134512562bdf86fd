// sort.cuh -- work bucketing by a lambda-monotone key (sort.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fpe {
constexpr int kCoarseBits = 12;                 // global buckets: top 12 of the 24 key bits
constexpr int kBuckets = 1 << kCoarseBits;
constexpr int kScatterThreads = 1024;           // classify / scatter CTA size: one CTA per SM
// points per classify / scatter CTA for a batch of n: one 1024-thread CTA per SM, so that the scatter's
// open output lines (148 CTAs x 4096 buckets x 128 B = 77 MB) stay in L2 until they are complete
inline long long pts_per_cta(long long n) {
  long long p = (n + 147) / 148;
  p = (p + 1023) / 1024 * 1024;
  return p < 1024 ? 1024 : p;
}
constexpr int kChunkPts = 2048;                 // points per evaluator work item (one bucket's slice)
constexpr int kLocalBits = 11;                  // in-chunk counting sort on key bits [1, 12)
constexpr int kPiece = 16384;                   // absolute coefficient pieces: a window is cut at multiples
                                                // of kPiece (relative to k_min) and the piece partials are
                                                // combined top-down, so results never depend on the batch

// A point's record in bucket / sorted order: index, sort key, window [l, r] (absolute).
struct __align__(16) PtRec {
  int32_t idx;
  uint32_t key;
  int32_t l, r;
};

// A group: 32*NP consecutive points of the sorted permutation, evaluated by one warp (NP points per
// lane) over the union [lo, hi] of their windows (relative to k_min; hi < lo: no finite point).
struct GroupDesc {
  uint32_t p0;      // first position in the permutation
  int32_t count;    // points in the group
  int32_t lo, hi;   // union of the windows
  uint32_t slot;    // first scratch slot (multi-piece groups evaluated in parallel)
  int32_t npieces;  // > 1: the pieces lo/kPiece .. hi/kPiece are separate work items
};

// Planner outputs (k_plan) consumed by the evaluator.
struct Plan {
  GroupDesc* desc;        // [max_groups]
  uint32_t* gcnt;         // [max_groups] finished pieces of a multi-piece group
  uint2* items;           // [cap] (group, piece) of the parallel pieces; group = ~0u: unused slot
  uint32_t* ctrs;         // [0] multi fetch, [1] group fetch, [2] slots reserved
  void* scratch;          // [cap][32*NP] piece partials (working complex type)
  uint32_t cap;           // scratch slots
  int gsize;              // points per group (32*NP)
  uint32_t ngroups;       // ceil(n / gsize)
};

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
// bucket starts + item table (k_bucket_scan), records in bucket order (k_bucket_scatter), the records
// sorted in place, their windows (written over lr) and points (zs) in sorted order (k_chunk_sort), and the
// work plan (k_plan)
void bucket_finish(const uint2* keys, int2* lr, long long n, long long ppc, const uint32_t* gcount,
                   const uint32_t* cta_base, uint32_t* bstart, uint32_t* istart, PtRec* rec, int pk,
                   const void* pts, double2* zs, long long k_min, const Plan& plan, cudaStream_t s);
inline long long max_chunks(long long n) { return (n + kChunkPts - 1) / kChunkPts + kBuckets; }
inline long long max_groups(long long n) { return (n + 63) / 64; }   // groups of >= 64 points
}  // namespace fpe
