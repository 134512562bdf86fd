// sort.cuh -- work bucketing by a lambda-monotone key (sort.cu).
#pragma once
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

namespace fpe {
constexpr int kCoarseBits = 15;                 // buckets: the top 15 of the 23 key bits (sign, exponent and
constexpr int kBuckets = 1 << kCoarseBits;      // 8 mantissa bits of an estimate of lambda); groups of
                                                // consecutive points of a bucket share their windows
// Bucket bits for a batch of n points: 15 from 2^20 points up, fewer for small batches (~32 points per
// bucket), so that the per-CTA histograms, slice claims and the bucket scan do not dominate them.
__host__ __device__ __forceinline__ int coarse_bits(long long n) {
  int b = 10;
  while (b < kCoarseBits && (1ll << (b + 5)) < n) ++b;
  return b;
}
constexpr int kScatterThreads = 1024;           // classify CTA size: one CTA per SM
// points per classify CTA for a batch of n: one 1024-thread CTA per SM
inline long long pts_per_cta(long long n) {
  long long p = (n + 147) / 148;
  p = (p + 1023) / 1024 * 1024;
  return p < 1024 ? 1024 : p;
}
#ifndef FPE_KPIECE
#define FPE_KPIECE 16384
#endif
constexpr int kPiece = FPE_KPIECE;                  // absolute coefficient pieces: a window is cut at multiples
                                                // of kPiece (relative to k_min) and the piece partials are
                                                // combined top-down, so results never depend on the batch

// A point's record in bucket order: index, sort key, window [l, r] (absolute), z as doubles -- one
// aligned 32-byte sector, so the classifier's random writes are whole sectors.
struct __align__(32) PtRec {
  int32_t idx;
  uint32_t key;
  int32_t l, r;
  double x, y;
};
// The evaluator stages each point's accumulator at the point's input index (one whole 32-byte sector per
// point, so the random writes need no read-modify-write); k_unsort streams them back in the caller's order
// and applies the epilogue.
struct __align__(32) PtOut {
  double re, im;   // the point's accumulator acc (eval_tiled.cu stage_acc)
  long long E;     // an extra binary exponent of acc (wide handles), else 0
  long long n;     // value = acc 2^E z^n (k_unsort applies the power: finalize); -1: nothing accumulated
};

// A group: 32*NP consecutive points of the sorted permutation, evaluated by one warp (NP points per
// lane) over the union [lo, hi] of their windows (relative to k_min; hi < lo: no finite point).
struct GroupDesc {
  uint32_t p0;      // first position in the permutation
  int32_t count;    // points in the group
  int32_t lo, hi;   // union of the windows
  uint32_t slot;    // first scratch slot (multi-piece groups evaluated in parallel)
  int32_t npieces;  // > 1: the pieces lo/kPiece .. hi/kPiece are separate work items
  int32_t mma_p0;   // first kPiece-aligned piece some point covers whole (tensor cores, k_eval_mma)
  int32_t mma_np;   // number of such pieces (0: none, or the DMMA scratch was exhausted)
  uint32_t mma_slot;  // their first slot in the DMMA scratch
  int32_t listed;   // 1: in Plan::long_groups (evaluated first, skipped in the bucket-order pass)
};

// Tensor-core coverage (k_eval_mma): point (window [wl, wr] relative to k_min, z = x + iy) has piece p
// evaluated on the FP64 tensor cores iff its window covers the whole kPiece-aligned piece and
// 2^-3 <= max(|x|, |y|) < 2^3 (the range of the chunk powers u^i <= z^(256 - P), w = z^256).  A property of
// the point alone, so every point's arithmetic is independent of the batch.
__host__ __device__ __forceinline__ bool mma_covers(int wl, int wr, double x, double y, int p) {
  if (!(wl <= wr) || wl > p * kPiece || wr < p * kPiece + kPiece - 1) return false;
  const double m = fmax(fabs(x), fabs(y));
  long long b;
  memcpy(&b, &m, sizeof(b));
  const int e = (int)((b >> 52) & 0x7ff) - 1023;
  return e >= -3 && e <= 2;
}

// Planner outputs (k_plan) consumed by the evaluator.
struct Plan {
  GroupDesc* desc;        // [max_groups]
  uint32_t* gcnt;         // [max_groups] finished pieces of a multi-piece group
  uint2* items;           // [cap] (group, piece) of the parallel pieces; group = ~0u: unused slot
  uint32_t* ctrs;         // [0] multi fetch, [1] group fetch, [2] slots reserved, [3] long groups listed
  uint32_t* long_groups;  // [max_groups] single-item groups with a union window longer than kLongWin: the
                          // longest class from the front (count ctrs[3]), the other from the back (ctrs[8])
  void* scratch;          // [cap][32*NP] piece partials (working complex type)
  uint32_t cap;           // scratch slots
  int gsize;              // points per group (32*NP)
  uint32_t ngroups;       // ceil(n / gsize)
  // tensor-core pieces (complex fp64 coefficients only)
  int mma_on;             // 1: plan them
  uint2* mma_items;       // [mma_cap] (group, piece)
  uint32_t* mma_ctrs;     // [0] slots reserved, [1] items fetched, [2] overflow groups, [3] ... fetched
  uint32_t* ovf_groups;   // [max_groups] groups whose items did not fit the scratch (k_eval_overflow)
  double2* mma_scratch;   // [mma_cap][gsize] partial sums of covered points, origin = piece start
  uint32_t mma_cap;
  unsigned long long* stats;   // the call's counters (workspace header, kStat*)
};

// bucket starts from the bucket totals (k_bucket_scan); the work plan of the records in bucket order (k_plan)
void bucket_scan(const uint32_t* gcount, uint32_t* bstart, long long n, cudaStream_t s);
// bwin[b] = {l, r} bounds (relative to k_min) of the windows of bucket b's points, and whether the bucket's
// points are all below (z) / all above (w) the |z| range of tensor-core pieces (k_bucket_windows)
void plan_groups(long long n, const uint32_t* bstart, const int4* bwin, const Plan& plan, cudaStream_t s);
#ifndef FPE_LONG_FIRST
#define FPE_LONG_FIRST 1
#endif
#ifndef FPE_LONG_WIN
#define FPE_LONG_WIN 4096
#endif
#ifndef FPE_LONG_WIN2
#define FPE_LONG_WIN2 0   // > 0: the listed groups longer than this go first (a second size class)
#endif
constexpr int kLongWin = FPE_LONG_WIN;   // groups with longer union windows are evaluated first (FPE_LONG_FIRST)
inline long long max_groups(long long n) { return (n + 63) / 64; }   // groups of >= 64 points
}  // namespace fpe
