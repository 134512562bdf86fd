// eval_mma.cu -- the window evaluator's whole kPiece-aligned pieces on the FP64 tensor cores (k_eval_mma).
#include <cuda_runtime.h>
#include <cstdint>
#include "fpe_internal.h"
#include "fpe_math.cuh"
#include "sort.cuh"
#include "tma.cuh"
#include "eval_tiled.cuh"
#include "mma_piece.cuh"

namespace fpe {

// ------------------------------------------------------------------------------------------------
// Whole kPiece-aligned pieces on the FP64 tensor cores (complex fp64 coefficients).
//
// A DFMA that reads three fresh register pairs issues at 2/3 of the fp64 rate on B200 and ptxas's
// schedule of the complex Horner step leaves most DFMAs without a reused operand: the vector Horner tops
// out near 72% of the pipe.  mma.sync DMMA runs the same datapath from its fragments at 99.7%
// (profiles/r01_dmma_vs_dfma.json).  Over whole 256-coefficient chunks the Horner sum is a dense
// contraction once split by phase k mod P (P = kMmaPhases = 32):
//   sum_{k in piece} a_k z^{k-k0} = sum_{m<P} z^m R_m,  R_m = sum_{q,i} a_{k0+256q+Pi+m} u^i w^q,
// u = z^P, w = z^256, and each chunk q (in increasing order) is C += A_q V_q with A_q[m][i] = a_{256q+Pi+m}
// (P x 256/P, straight from the staged chunk), V_q[i][p] = u_p^i w_p^q and C[m][p] = R_m at point p
// (mma_piece.cuh): 4 real m16n8k4 DMMAs per 4 powers and 8 points for the complex product.  One CTA (8 warps x 16 points = a group) per item
// (group, piece), the piece's 64 chunks staged once per CTA by TMA into a 4-stage ring shared by the
// warps.  A point's column is active iff mma_covers (its window covers the whole piece), so every value
// is relative to the piece start, which lies in the point's window; u, u^4, w are
// rounded once from double-double squarings (w carries 1 ulp per chunk, the chunk powers ~11 ulp).
#ifndef FPE_MMA_MINB
#define FPE_MMA_MINB 2     // CTAs per SM the register budget is sized for (16 warps: 7.16 vs 7.35 ms with 1)
#endif
#ifndef FPE_MMA_STAGES
#define FPE_MMA_STAGES 6   // 6 vs 4: 7.30 vs 7.36 ms at cfg3
#endif
constexpr int kMmaWarps = 8;
constexpr int kMmaStages = FPE_MMA_STAGES;
constexpr int kPieceChunks = kMmaPieceChunks;

__global__ void __launch_bounds__(kMmaWarps * 32, FPE_MMA_MINB) k_eval_mma(long long n, const double2* __restrict__ coef,
                                                                int kmin, const PtRec* __restrict__ rec, Plan plan) {
  __shared__ __align__(128) double2 ring[kMmaStages][kChunk];
  __shared__ uint64_t full[kMmaStages], empty[kMmaStages];
  __shared__ uint2 item_sh, next_sh;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kMmaStages; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, kMmaWarps); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t n_items = min(plan.mma_ctrs[0], plan.mma_cap);
  uint32_t t_seq = 0;      // chunks consumed by this CTA (every warp consumes every chunk)
  uint32_t t_issued = 0;   // chunks issued (thread 0)
  auto issue = [&](int piece_chunk) {   // thread 0: next chunk into the ring
    const int s = (int)(t_issued % kMmaStages);
    if (t_issued >= (uint32_t)kMmaStages) mbar_wait(empty + s, ((t_issued / kMmaStages) - 1) & 1u);
    fence_proxy_async();
    mbar_expect_tx(full + s, kChunk * sizeof(double2));
    tma_load_1d(ring[s], coef + (size_t)piece_chunk * kChunk, kChunk * sizeof(double2), full + s);
    ++t_issued;
  };
  // Thread 0 claims items one ahead and streams the next item's first chunks into the ring while the warps
  // finish the current one, so the ring does not drain at item boundaries (short items pay for it otherwise).
  auto fetch = [&]() -> uint2 {   // thread 0: the next valid item, or the end marker
    for (;;) {
      const uint32_t it = atomicAdd(plan.mma_ctrs + 1, 1u);
      if (it >= n_items) return make_uint2(0xfffffffeu, 0u);
      const uint2 v = plan.mma_items[it];
      if (v.x != ~0u) return v;
    }
  };
  if (tid == 0) {
    const uint2 c = fetch();
    if (c.x != 0xfffffffeu)
      for (int i = 0; i < kMmaStages; ++i) issue((int)c.y * kPieceChunks + i);
    item_sh = c;
    next_sh = c.x != 0xfffffffeu ? fetch() : c;
  }
  __syncthreads();
  for (;;) {
    const uint2 item = item_sh, nxt = next_sh;
    __syncthreads();
    if (item.x == 0xfffffffeu) break;
    const uint32_t grp = item.x;
    const int p = (int)item.y;
    const int q0 = p * kPieceChunks;   // chunks ascend from q0 (mma_piece.cuh)
    // this warp's 16 points: lanes [0, 16) own point 16 w + lane (lanes 16..31 mirror them)
    const int q = 16 * w + (lane & 15);
    const long long pos = (long long)grp * plan.gsize + q;
    double x = 0.0, y = 0.0;
    int wl = 1, wr = 0;
    if (pos < n) {
      const int4 h = __ldg(reinterpret_cast<const int4*>(rec + pos));
      const double2 z = __ldg(reinterpret_cast<const double2*>(rec + pos) + 1);
      x = z.x; y = z.y;
      if (h.w >= h.z) { wl = h.z - kmin; wr = h.w - kmin; }
    }
    const int act = mma_covers(wl, wr, x, y, p) ? 1 : 0;
    MmaFrag F;
    mma_setup(F, x, y, act);
    const bool busy = __any_sync(0xffffffffu, act);   // a warp without covering points only keeps the ring going
    for (int k = 0; k < kPieceChunks; ++k) {
      const int s = (int)(t_seq % kMmaStages);
      mbar_wait(full + s, (t_seq / kMmaStages) & 1u);
      if (busy) mma_chunk(F, ring[s]);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      ++t_seq;
      if (tid == 0) {
        const int j = k + kMmaStages;
        if (j < kPieceChunks) issue(q0 + j);
        else if (nxt.x != 0xfffffffeu) issue((int)nxt.y * kPieceChunks + (j - kPieceChunks));
      }
      __syncwarp();
    }
    double orr, oi;
    mma_finish(F, x, y, orr, oi);
    if (lane < 16 && act) {
      const GroupDesc d = plan.desc[grp];
      plan.mma_scratch[(size_t)(d.mma_slot + (p - d.mma_p0)) * plan.gsize + q] = make_double2(orr, oi);
    }
    if (tid == 0) {
      item_sh = nxt;
      next_sh = nxt.x != 0xfffffffeu ? fetch() : nxt;
    }
    __syncthreads();
  }
}

int launch_eval_mma(long long n, const PolyDev& P, const PtRec* rec, const Plan& plan, cudaStream_t s) {
  const int grid = persistent_grid(reinterpret_cast<const void*>(k_eval_mma), kMmaWarps * 32, 0);
  k_eval_mma<<<grid, kMmaWarps * 32, 0, s>>>(n, static_cast<const double2*>(P.coef), (int)P.k_min, rec, plan);
  return 1;
}

}  // namespace fpe
