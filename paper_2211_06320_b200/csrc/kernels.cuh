// kernels.cuh -- launchers of kernels.cu (host side).
#pragma once
#include <cuda_runtime.h>
#include "fpe_internal.h"

namespace fpe {
constexpr int kSmemHullMax = 6144;   // cover vertices staged in shared memory (48 KiB)
constexpr int kSmemHullDbl = 1536;   // ... also as doubles (36 KiB) by the bucketing classifier

void launch_classify(int pk, const void* pts, long long n, const PolyDev& P, int2* lr, fpe_diag* diag,
                     unsigned long long* hard, cudaStream_t s);
constexpr int kSparseTab = 4096;   // buckets of the sparse evaluator's good-index table (int32[kSparseTab + 1])
// tab: device scratch of (kSparseTab + 2) int32 (the table and a work-queue counter), written by the call
bool launch_eval_sparse(int pk, const void* pts, long long n, const PolyDev& P, const int2* lr, int* tab, void* vals,
                        long long* exps, cudaStream_t s);
// fpe_diag::cancel from the outputs (after an evaluation); ok = fpe_dtype of the values
void launch_confidence(int ok, long long n, const PolyDev& P, const void* vals, const long long* exps,
                       fpe_diag* diag, cudaStream_t s);
// z - Q1/Q2 from extended-range values (fpe_newton_step)
void launch_newton(int pk, int ok, long long n, const void* pts, const void* v1, const long long* e1, const void* v2,
                   const long long* e2, void* out, void* incr, cudaStream_t s);
bool launch_horner(int pk, const void* pts, long long n, const PolyDev& P, void* vals, long long* exps,
                   cudaStream_t s);
}  // namespace fpe
