// eval_tiled.cuh -- host entry of the bucketed tiled evaluator (eval_tiled.cu).
#pragma once
#include <cuda_runtime.h>
#include "fpe_internal.h"
#include "sort.cuh"

#ifndef FPE_NO_MMA_ITEMS
#define FPE_NO_MMA_ITEMS 0   // experiments: 1 keeps every piece on the vector Horner
#endif

namespace fpe {
constexpr int kChunk = kCoefPad;   // coefficients per TMA bulk copy / ring stage (dense array padded to this)

size_t tiled_ws_bytes(long long n);
// classify + sort + plan + evaluate (dense handles); stats: the call's kStat* counters (device).  Returns
// the number of kernel launches or -1.
int run_tiled(int pk, const void* pts, long long n, const PolyDev& P, void* vals, long long* exps,
              fpe_diag* diag, void* ws, unsigned long long* stats, Stage& st, cudaStream_t s);
// full Horner (dense handles) with the streaming evaluator; ctr: one device uint32 of scratch
// (complex fp64 coefficients with ws_bytes >= 256 + 4 n: on the FP64 tensor cores, k_horner_mma)
bool run_horner_tiled(int pk, const void* pts, long long n, const PolyDev& P, uint32_t* ctr, void* vals,
                      long long* exps, cudaStream_t s, size_t ws_bytes);
// whole kPiece pieces some point covers, on the FP64 tensor cores (eval_mma.cu); before the vector evaluator
int launch_eval_mma(long long n, const PolyDev& P, const PtRec* rec, const Plan& plan, cudaStream_t s);
}  // namespace fpe
