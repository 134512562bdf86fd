// mma_piece.cuh -- the per-warp arithmetic of a whole kPiece piece on the FP64 tensor cores, shared by
// k_eval_mma (eval_mma.cu: CTA-shared TMA ring, one warp per 16 points) and the vector evaluator's
// in-warp fallback (eval_tiled.cu: a group whose tensor-core items did not fit the DMMA scratch runs the
// same functions over its private ring).  Both call exactly these functions with the same per-point
// inputs, so a point's piece partial is bitwise the same whichever kernel computed it: results stay a
// pure function of (z, handle), whatever the batch (fpe.h).
//
// Phase split: over whole 256-coefficient chunks the piece sum is, with P phases (k mod P),
//   sum_{k in piece} a_k z^{k-k0} = sum_{m<P} z^m R_m,  R_m = sum_q sum_i a_{k0+256q+Pi+m} u^i w^q,
// u = z^P, w = z^256.  The chunks are fed in increasing q and each is one accumulation C += A_q V_q with
// A_q[m][i] = a_{k0+256q+Pi+m} (straight from the staged chunk) and V_q[i][p] = u_p^i w_p^q, the B
// fragment advanced by V_{q+1} = V_q (.) w after the chunk's DMMAs are issued -- so the per-chunk power
// update does not wait on the accumulators (a Horner over chunks, C <- C (.) w + A V, would put a complex
// multiply of every accumulator between consecutive chunks' DMMAs).
// Lane layout (m16n8k4 fragments): lanes 0..15 own the warp's 16 points (lanes 16..31 mirror them);
// thread (g = lane >> 2, c = lane & 3) holds B rows c of the two 8-point column tiles t and C columns 2c, 2c+1.
#pragma once
#include <cuda_runtime.h>
#include "fpe_math.cuh"
#include "fpe_internal.h"
#include "sort.cuh"

namespace fpe {

constexpr int kMmaPieceChunks = kPiece / kCoefPad;   // 256-coefficient chunks per piece
// GroupDesc::mma_slot of a group whose tensor-core items did not fit the DMMA scratch: the vector
// evaluator runs them in-warp (eval_tiled.cu mma_pass_inwarp)
constexpr uint32_t kMmaInWarp = 0xffffffffu;

// Phases P of the split (k mod P): a chunk is A (P x 256/P) times V (256/P x 16 points).  The per-chunk update
// V <- V (.) w costs one complex multiply per V entry, i.e. 1/P of the chunk's tensor work on the same fp64
// datapath: 32 phases halve it against 16 (C doubles, V halves).
#ifndef FPE_MMA_PHASES
#define FPE_MMA_PHASES 32
#endif
constexpr int kMmaPhases = FPE_MMA_PHASES;
constexpr int kMmaLogPhases = kMmaPhases == 16 ? 4 : 5;
static_assert(kMmaPhases == 16 || kMmaPhases == 32, "16 or 32 phases");
constexpr int kMmaI = kCoefPad / kMmaPhases;      // powers u^i per chunk (u = z^P)
constexpr int kMmaKs = kMmaI / 4;               // m16n8k4 k-steps per chunk
constexpr int kMmaMt = kMmaPhases / 16;         // m16 tiles of phases
constexpr int kMmaMaxBPow = kCoefPad - kMmaPhases;   // the largest B power, u^(I-1) = z^(256 - P)

__device__ __forceinline__ void mma_cmul(double& r, double& i, double ar, double ai, double br, double bi) {
  const double t = fma(ar, br, -ai * bi);
  i = fma(ar, bi, ai * br);
  r = t;
}
__device__ __forceinline__ void mma_dmma(double (&c)[4], double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void mma_dd_sqr_c(xc_t& v) {
  xc_sqr(v);
  const dd_t r = two_sum(v.hr, v.er), i = two_sum(v.hi, v.ei);
  v.hr = r.hi; v.er = r.lo; v.hi = i.hi; v.ei = i.lo;
}

// Fragments of one warp's 16 points for one piece.
struct MmaFrag {
  double vr[2][kMmaKs], vi[2][kMmaKs];   // B: u^(4 ks + c) w^q of the column tiles (0 for inactive columns)
  double cwr[2], cwi[2];                 // w = z^256 of the B columns g, 8 + g
  double cr[kMmaMt][2][4], ci[kMmaMt][2][4];   // C: Re / Im of R_m (m = 16 mt + g, + 8; columns 2c, 2c + 1)
};

// (x, y, act): the point of lane & 15 (act: it covers the piece, mma_covers).  u = z^P, u^4, w = z^256 by
// double-double squarings, rounded once each.
__device__ __forceinline__ void mma_setup(MmaFrag& F, double x, double y, int act) {
  const int lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
  double ur, ui, u4r, u4i, wwr, wwi;
  {
    xc_t v{act ? x : 1.0, act ? y : 0.0, 0.0, 0.0, 0};
#pragma unroll
    for (int i = 0; i < kMmaLogPhases; ++i) mma_dd_sqr_c(v);
    ur = v.hr + v.er; ui = v.hi + v.ei;
    mma_dd_sqr_c(v); mma_dd_sqr_c(v);
    u4r = v.hr + v.er; u4i = v.hi + v.ei;
#pragma unroll
    for (int i = kMmaLogPhases + 2; i < 8; ++i) mma_dd_sqr_c(v);
    wwr = v.hr + v.er; wwi = v.hi + v.ei;
  }
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int src = 8 * t + g;                   // the point of B column g
    const double qr = __shfl_sync(0xffffffffu, ur, src), qi = __shfl_sync(0xffffffffu, ui, src);
    const double q4r = __shfl_sync(0xffffffffu, u4r, src), q4i = __shfl_sync(0xffffffffu, u4i, src);
    const int on = __shfl_sync(0xffffffffu, act, src);
    double pr = 1.0, pi = 0.0;                   // u^c
#pragma unroll
    for (int i = 0; i < 3; ++i)
      if (i < c) mma_cmul(pr, pi, pr, pi, qr, qi);
#pragma unroll
    for (int ks = 0; ks < kMmaKs; ++ks) {        // B row c of k-step ks: u^(4 ks + c); inactive column: 0
      if (ks) mma_cmul(pr, pi, pr, pi, q4r, q4i);
      F.vr[t][ks] = on ? pr : 0.0;
      F.vi[t][ks] = on ? pi : 0.0;
    }
    F.cwr[t] = __shfl_sync(0xffffffffu, wwr, src);   // w of the B column g of tile t
    F.cwi[t] = __shfl_sync(0xffffffffu, wwi, src);
#pragma unroll
    for (int mt = 0; mt < kMmaMt; ++mt)
#pragma unroll
      for (int e = 0; e < 4; ++e) { F.cr[mt][t][e] = 0.0; F.ci[mt][t][e] = 0.0; }
  }
}

// One 256-coefficient chunk (cb: its first coefficient; chunks are fed in increasing q): C += A_q V_q, then
// V <- V (.) w for the next chunk.  A_q[m][i] = a_{256 q + P i + m}.
__device__ __forceinline__ void mma_chunk(MmaFrag& F, const double2* cb) {
  const int lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
#pragma unroll
  for (int ks = 0; ks < kMmaKs; ++ks) {
#pragma unroll
    for (int mt = 0; mt < kMmaMt; ++mt) {
      const int ia = kMmaPhases * (4 * ks + c) + 16 * mt + g;
      const double2 a0 = cb[ia], a1 = cb[ia + 8];   // A[16 mt + g | + 8][4 ks + c]
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        mma_dmma(F.cr[mt][t], a0.x, a1.x, F.vr[t][ks]);      // Re: ar vr - ai vi
        mma_dmma(F.cr[mt][t], -a0.y, -a1.y, F.vi[t][ks]);
        mma_dmma(F.ci[mt][t], a0.x, a1.x, F.vi[t][ks]);      // Im: ar vi + ai vr
        mma_dmma(F.ci[mt][t], a0.y, a1.y, F.vr[t][ks]);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int ks = 0; ks < kMmaKs; ++ks) mma_cmul(F.vr[t][ks], F.vi[t][ks], F.vr[t][ks], F.vi[t][ks], F.cwr[t], F.cwi[t]);
}

// Exact power-of-two rescaling hooks (k_horner_mma): B columns by sb[t], C columns 2c + e of tile t by sc[t][e].
__device__ __forceinline__ void mma_scale_b(MmaFrag& F, const double (&sb)[2]) {
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int ks = 0; ks < kMmaKs; ++ks) { F.vr[t][ks] *= sb[t]; F.vi[t][ks] *= sb[t]; }
}
__device__ __forceinline__ void mma_scale_c(MmaFrag& F, const double (&sc)[2][2]) {
#pragma unroll
  for (int mt = 0; mt < kMmaMt; ++mt)
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) { F.cr[mt][t][e] *= sc[t][e & 1]; F.ci[mt][t][e] *= sc[t][e & 1]; }
}

// sum_m z^m R_m for the warp's 16 points: rows 16 mt + g, + 8 in the thread (z^8, then z^16 across the
// m-tiles), then a tree over g (lane bits 2..4).  (x, y): the point of lane & 15.  The result of point
// lane is returned in lanes 0..15.
__device__ __forceinline__ void mma_finish(const MmaFrag& F, double x, double y, double& orr, double& oi) {
  const int lane = threadIdx.x & 31, c = lane & 3;
  double hr[2][2], hi[2][2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int src = 8 * t + 2 * c + e;
      const double zr = __shfl_sync(0xffffffffu, x, src), zi = __shfl_sync(0xffffffffu, y, src);
      double z2r, z2i, z4r, z4i, z8r, z8i;
      mma_cmul(z2r, z2i, zr, zi, zr, zi);
      mma_cmul(z4r, z4i, z2r, z2i, z2r, z2i);
      mma_cmul(z8r, z8i, z4r, z4i, z4r, z4i);
      double pr = 0.0, pi = 0.0;
#pragma unroll
      for (int mt = kMmaMt - 1; mt >= 0; --mt) {
        double qr = F.cr[mt][t][e], qi = F.ci[mt][t][e];
        qr = fma(F.cr[mt][t][e + 2], z8r, fma(-F.ci[mt][t][e + 2], z8i, qr));
        qi = fma(F.cr[mt][t][e + 2], z8i, fma(F.ci[mt][t][e + 2], z8r, qi));
        if (mt == kMmaMt - 1) { pr = qr; pi = qi; }
        else {   // p <- q + z^16 p
          double z16r, z16i;
          mma_cmul(z16r, z16i, z8r, z8i, z8r, z8i);
          const double nr = fma(pr, z16r, fma(-pi, z16i, qr));
          pi = fma(pr, z16i, fma(pi, z16r, qi));
          pr = nr;
        }
      }
      double nr = __shfl_xor_sync(0xffffffffu, pr, 4), ni = __shfl_xor_sync(0xffffffffu, pi, 4);
      pr = fma(nr, zr, fma(-ni, zi, pr)); pi = fma(nr, zi, fma(ni, zr, pi));
      nr = __shfl_xor_sync(0xffffffffu, pr, 8); ni = __shfl_xor_sync(0xffffffffu, pi, 8);
      pr = fma(nr, z2r, fma(-ni, z2i, pr)); pi = fma(nr, z2i, fma(ni, z2r, pi));
      nr = __shfl_xor_sync(0xffffffffu, pr, 16); ni = __shfl_xor_sync(0xffffffffu, pi, 16);
      pr = fma(nr, z4r, fma(-ni, z4i, pr)); pi = fma(nr, z4i, fma(ni, z4r, pi));
      hr[t][e] = pr; hi[t][e] = pi;              // valid in lanes 0..3 (g = 0)
    }
  orr = 0.0; oi = 0.0;
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const double a = __shfl_sync(0xffffffffu, hr[t][e], (lane & 7) >> 1);
      const double b = __shfl_sync(0xffffffffu, hi[t][e], (lane & 7) >> 1);
      if (((lane >> 3) & 1) == t && (lane & 1) == e) { orr = a; oi = b; }
    }
}

}  // namespace fpe
