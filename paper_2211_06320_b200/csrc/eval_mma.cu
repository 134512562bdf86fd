// eval_mma.cu -- the window evaluator's whole kPiece-aligned pieces on the FP64 tensor cores (k_eval_mma).
#include <cuda_runtime.h>
#include <cstdint>
#include "fpe_internal.h"
#include "fpe_math.cuh"
#include "sort.cuh"
#include "tma.cuh"
#include "eval_tiled.cuh"

namespace fpe {

// ------------------------------------------------------------------------------------------------
// Whole kPiece-aligned pieces on the FP64 tensor cores (complex fp64 coefficients).
//
// A DFMA that reads three fresh register pairs issues at 2/3 of the fp64 rate on B200 and ptxas's
// schedule of the complex Horner step leaves most DFMAs without a reused operand: the vector Horner tops
// out near 72% of the pipe.  mma.sync DMMA runs the same datapath from its fragments at 99.7%
// (profiles/r01_dmma_vs_dfma.json).  Over whole 256-coefficient chunks the Horner sum is a dense
// contraction once split by phase k mod 16:
//   sum_{k in piece} a_k z^{k-k0} = sum_{m<16} z^m R_m,  R_m = sum_t a_{k0+16t+m} u^t,  u = z^16,
// and each chunk q is C <- C (.) w + A V with A[m][i] = a_{256q+16i+m} (16 x 16, straight from the staged
// chunk), V[i][p] = u_p^i, w_p = u_p^16 = z_p^256 and C[m][p] = R_m at point p: 4 real m16n8k4 DMMAs per
// 4 powers and 8 points for the complex product.  One CTA (8 warps x 16 points = a group) per item
// (group, piece), the piece's 64 chunks staged once per CTA by TMA into a 4-stage ring shared by the
// warps.  A point's column is active iff mma_covers (its window covers the whole piece), so every value
// is relative to the piece start, which lies in the point's window; u, u^4, w are
// rounded once from double-double squarings (w carries 1 ulp per chunk, the chunk powers ~11 ulp).
#ifndef FPE_MMA_MINB
#define FPE_MMA_MINB 2     // CTAs per SM the register budget is sized for (16 warps: 7.16 vs 7.35 ms with 1)
#endif
#ifndef FPE_MMA_STAGES
#define FPE_MMA_STAGES 4
#endif
constexpr int kMmaWarps = 8;
constexpr int kMmaStages = FPE_MMA_STAGES;
constexpr int kPieceChunks = kPiece / kChunk;

__device__ __forceinline__ void cmul(double& r, double& i, double ar, double ai, double br, double bi) {
  const double t = fma(ar, br, -ai * bi);
  i = fma(ar, bi, ai * br);
  r = t;
}
__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void dd_sqr_c(xc_t& v) {
  xc_sqr(v);
  const dd_t r = two_sum(v.hr, v.er), i = two_sum(v.hi, v.ei);
  v.hr = r.hi; v.er = r.lo; v.hi = i.hi; v.ei = i.lo;
}

__global__ void __launch_bounds__(kMmaWarps * 32, FPE_MMA_MINB) k_eval_mma(long long n, const double2* __restrict__ coef,
                                                                int kmin, const PtRec* __restrict__ rec, Plan plan) {
  __shared__ __align__(128) double2 ring[kMmaStages][kChunk];
  __shared__ uint64_t full[kMmaStages], empty[kMmaStages];
  __shared__ uint2 item_sh;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, c = lane & 3;
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
  for (;;) {
    if (tid == 0) {
      const uint32_t it = atomicAdd(plan.mma_ctrs + 1, 1u);
      item_sh = it < n_items ? plan.mma_items[it] : make_uint2(0xfffffffeu, 0u);
    }
    __syncthreads();
    const uint2 item = item_sh;
    __syncthreads();
    if (item.x == 0xfffffffeu) break;
    if (item.x == ~0u) continue;
    const uint32_t grp = item.x;
    const int p = (int)item.y;
    const int q0 = p * kPieceChunks + kPieceChunks - 1;   // chunks descend from q0
    if (tid == 0)
      for (int i = 0; i < kMmaStages; ++i) issue(q0 - i);
    __syncwarp();
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
    // u = z^16, u^4, w = z^256 of the lane's point (double-double squarings, one rounding each)
    double ur, ui, u4r, u4i, wwr, wwi;
    {
      xc_t v{act ? x : 1.0, act ? y : 0.0, 0.0, 0.0, 0};
#pragma unroll
      for (int i = 0; i < 4; ++i) dd_sqr_c(v);
      ur = v.hr + v.er; ui = v.hi + v.ei;
      dd_sqr_c(v); dd_sqr_c(v);
      u4r = v.hr + v.er; u4i = v.hi + v.ei;
      dd_sqr_c(v); dd_sqr_c(v);
      wwr = v.hr + v.er; wwi = v.hi + v.ei;
    }
    double vr[2][4], vi[2][4], cwr[2][2], cwi[2][2], cr[2][4], ci[2][4];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int src = 8 * t + g;                   // the point of B column g
      const double qr = __shfl_sync(0xffffffffu, ur, src), qi = __shfl_sync(0xffffffffu, ui, src);
      const double q4r = __shfl_sync(0xffffffffu, u4r, src), q4i = __shfl_sync(0xffffffffu, u4i, src);
      const int on = __shfl_sync(0xffffffffu, act, src);
      double pr = 1.0, pi = 0.0;                   // u^c
#pragma unroll
      for (int i = 0; i < 3; ++i)
        if (i < c) cmul(pr, pi, pr, pi, qr, qi);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {             // B row c of k-step ks: u^(4 ks + c); inactive column: 0
        if (ks) cmul(pr, pi, pr, pi, q4r, q4i);
        vr[t][ks] = on ? pr : 0.0;
        vi[t][ks] = on ? pi : 0.0;
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {                // w of the C columns 2c, 2c + 1
        const int s2 = 8 * t + 2 * c + e;
        cwr[t][e] = __shfl_sync(0xffffffffu, wwr, s2);
        cwi[t][e] = __shfl_sync(0xffffffffu, wwi, s2);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) { cr[t][e] = 0.0; ci[t][e] = 0.0; }
    }
    const bool busy = __any_sync(0xffffffffu, act);   // a warp without covering points only keeps the ring going
    for (int k = 0; k < kPieceChunks; ++k) {
      const int s = (int)(t_seq % kMmaStages);
      mbar_wait(full + s, (t_seq / kMmaStages) & 1u);
      const double2* cb = ring[s];
      if (!busy) {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
        ++t_seq;
        if (tid == 0 && k + kMmaStages < kPieceChunks) issue(q0 - k - kMmaStages);
        __syncwarp();
        continue;
      }
      if (k) {
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int e = 0; e < 4; ++e) cmul(cr[t][e], ci[t][e], cr[t][e], ci[t][e], cwr[t][e & 1], cwi[t][e & 1]);
      }
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const double2 a0 = cb[64 * ks + 16 * c + g], a1 = cb[64 * ks + 16 * c + g + 8];   // A[g|g+8][4ks + c]
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          dmma(cr[t], a0.x, a1.x, vr[t][ks]);      // Re: ar vr - ai vi
          dmma(cr[t], -a0.y, -a1.y, vi[t][ks]);
          dmma(ci[t], a0.x, a1.x, vi[t][ks]);      // Im: ar vi + ai vr
          dmma(ci[t], a0.y, a1.y, vr[t][ks]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      ++t_seq;
      if (tid == 0 && k + kMmaStages < kPieceChunks) issue(q0 - k - kMmaStages);
      __syncwarp();
    }
    // sum_m z^m R_m: rows g and g + 8 in the thread, then a tree over g (lane bits 2..4)
    double hr[2][2], hi[2][2];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int src = 8 * t + 2 * c + e;
        const double zr = __shfl_sync(0xffffffffu, x, src), zi = __shfl_sync(0xffffffffu, y, src);
        double z2r, z2i, z4r, z4i, z8r, z8i;
        cmul(z2r, z2i, zr, zi, zr, zi);
        cmul(z4r, z4i, z2r, z2i, z2r, z2i);
        cmul(z8r, z8i, z4r, z4i, z4r, z4i);
        double pr = cr[t][e], pi = ci[t][e];
        pr = fma(cr[t][e + 2], z8r, fma(-ci[t][e + 2], z8i, pr));
        pi = fma(cr[t][e + 2], z8i, fma(ci[t][e + 2], z8r, pi));
        double nr = __shfl_xor_sync(0xffffffffu, pr, 4), ni = __shfl_xor_sync(0xffffffffu, pi, 4);
        pr = fma(nr, zr, fma(-ni, zi, pr)); pi = fma(nr, zi, fma(ni, zr, pi));
        nr = __shfl_xor_sync(0xffffffffu, pr, 8); ni = __shfl_xor_sync(0xffffffffu, pi, 8);
        pr = fma(nr, z2r, fma(-ni, z2i, pr)); pi = fma(nr, z2i, fma(ni, z2r, pi));
        nr = __shfl_xor_sync(0xffffffffu, pr, 16); ni = __shfl_xor_sync(0xffffffffu, pi, 16);
        pr = fma(nr, z4r, fma(-ni, z4i, pr)); pi = fma(nr, z4i, fma(ni, z4r, pi));
        hr[t][e] = pr; hi[t][e] = pi;              // valid in lanes 0..3 (g = 0)
      }
    double orr = 0.0, oi = 0.0;
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double a = __shfl_sync(0xffffffffu, hr[t][e], (lane & 7) >> 1);
        const double b = __shfl_sync(0xffffffffu, hi[t][e], (lane & 7) >> 1);
        if (((lane >> 3) & 1) == t && (lane & 1) == e) { orr = a; oi = b; }
      }
    if (lane < 16 && act) {
      const GroupDesc d = plan.desc[grp];
      plan.mma_scratch[(size_t)(d.mma_slot + (p - d.mma_p0)) * plan.gsize + q] = make_double2(orr, oi);
    }
  }
}

int launch_eval_mma(long long n, const PolyDev& P, const PtRec* rec, const Plan& plan, cudaStream_t s) {
  const int grid = persistent_grid(reinterpret_cast<const void*>(k_eval_mma), kMmaWarps * 32, 0);
  k_eval_mma<<<grid, kMmaWarps * 32, 0, s>>>(n, static_cast<const double2*>(P.coef), (int)P.k_min, rec, plan);
  return 1;
}

}  // namespace fpe
