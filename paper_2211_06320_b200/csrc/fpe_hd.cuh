// fpe_hd.cuh -- host/device wrappers for the correctly rounded fp64 primitives used by the
// FPE math (fpe_math.cuh, fpe_polar.cuh).  On the device they are the _rn intrinsics, which
// nvcc never contracts into FMAs; on the host (CPU unit tests of the device math, built with
// -ffp-contract=off) they are plain IEEE operations.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>
#include "log_table.h"

#ifdef __CUDACC__
#define FPE_HD __host__ __device__ __forceinline__
#else
#define FPE_HD inline
#endif

namespace fpe {

FPE_HD double fpe_add(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
FPE_HD double fpe_sub(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
FPE_HD double fpe_mul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
FPE_HD double fpe_div(double a, double b) {
#ifdef __CUDA_ARCH__
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}
FPE_HD double fpe_fma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
FPE_HD double fpe_bits2d(long long b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(b);
#else
  double d;
  std::memcpy(&d, &b, sizeof d);
  return d;
#endif
}
FPE_HD long long fpe_d2bits(double d) {
#ifdef __CUDA_ARCH__
  return __double_as_longlong(d);
#else
  long long b;
  std::memcpy(&b, &d, sizeof b);
  return b;
#endif
}
FPE_HD int fpe_clzll(long long n) {
#ifdef __CUDA_ARCH__
  return __clzll(n);
#else
  return n == 0 ? 64 : __builtin_clzll((unsigned long long)n);
#endif
}
FPE_HD int fpe_d2i_rn(double x) {
#ifdef __CUDA_ARCH__
  return __double2int_rn(x);
#else
  return (int)std::nearbyint(x);
#endif
}
FPE_HD double fpe_logtab(int i, int j) {
#ifdef __CUDA_ARCH__
  return __ldg(&fpe_logtab_d[i][j]);
#else
  return fpe_logtab_h[i][j];
#endif
}
FPE_HD double fpe_atantab(int i, int j) {
#ifdef __CUDA_ARCH__
  return __ldg(&fpe_atantab_d[i][j]);
#else
  return fpe_atantab_h[i][j];
#endif
}

}  // namespace fpe
