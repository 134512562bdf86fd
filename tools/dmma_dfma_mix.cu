// dmma_dfma_mix.cu -- do DMMA (mma.sync f64) and DFMA share the fp64 datapath on B200?  Warps of one kernel
// run either a DMMA loop or a DFMA loop (mode 0: all DMMA, 1: all DFMA, 2: even warps DMMA / odd DFMA);
// the combined FMA rate of mode 2 against modes 0 and 1 answers it.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dmma_dfma_mix tools/dmma_dfma_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_mix(double* out, long long it_m, long long it_f, int mode, double y, double z) {
  const int w = threadIdx.x >> 5;
  const bool mma = mode == 0 || (mode == 2 && (w & 1) == 0);
  double s = 0;
  if (mma) {
    double a0 = 1.0 + 1e-9 * threadIdx.x, a1 = 1.0 - 1e-9 * threadIdx.x, b = 1.0 - 2e-9 * threadIdx.x;
    double c[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 2 * i; c[i][3] = 1; }
    for (long long t = 0; t < it_m; ++t) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  } else {
    double x[8];   // y, z: kernel parameters (uniform registers: the DFMA runs at the full rate)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = 1.0 + i * 1e-7;
    for (long long t = 0; t < it_f; ++t) {
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[i]) : "d"(y), "d"(z));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
  }
  if (s == 1.2345) out[0] = s;
}

int main() {
  double* d; cudaMalloc(&d, 8);
  const int blocks = 148 * 2, threads = 512;   // 32 warps per SM
  const long long it_m = 4096, it_f = 4096 * 16;   // per warp: 8*512*it_m FMA (DMMA) = 8*32*it_f FMA (DFMA)
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    k_mix<<<blocks, threads>>>(d, it_m, it_f, mode, 1.0 - 1e-12, 1e-9);
    cudaEventRecord(e0);
    k_mix<<<blocks, threads>>>(d, it_m, it_f, mode, 1.0 - 1e-12, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)blocks * threads / 32;
    const double fma = warps * 8.0 * 512.0 * it_m;   // the same per warp in every mode
    printf("mode %d (%s): %.3f ms, %.2f T FMA/s\n", mode, mode == 0 ? "all DMMA" : mode == 1 ? "all DFMA" : "half DMMA + half DFMA",
           ms, fma / (ms * 1e-3) / 1e12);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
