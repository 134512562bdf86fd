// fp64_peak.cu -- measures the sustained fp64 / fp32 FMA rate of this B200 (roofline denominator check).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CHAINS>
__global__ void fma_loop(T* out, long long iters, T a, T b) {
  T x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = (T)(threadIdx.x + c);
  for (long long i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == (T)12345.678) out[0] = s;
}

template <typename T>
double run(int blocks_per_sm, int threads, long long iters, float* ms_out) {
  T* d;
  cudaMalloc(&d, sizeof(T));
  int dev; cudaGetDevice(&dev);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int grid = p.multiProcessorCount * blocks_per_sm;
  fma_loop<T, 8><<<grid, threads>>>(d, iters / 10, (T)0.999999, (T)1e-7);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) fma_loop<T, 8><<<grid, threads>>>(d, iters, (T)0.999999, (T)1e-7);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  *ms_out = ms;
  double fmas = 5.0 * grid * threads * iters * 8.0;
  cudaFree(d);
  return fmas / (ms * 1e-3);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d", p.name, p.multiProcessorCount, clk);
  float ms;
  double f64 = run<double>(8, 256, 1 << 16, &ms);
  printf(", \"fp64_fma_per_s\": %.4e, \"fp64_ms\": %.2f", f64, ms);
  double f32 = run<float>(8, 256, 1 << 17, &ms);
  printf(", \"fp32_fma_per_s\": %.4e, \"fp32_ms\": %.2f", f32, ms);
  double nominal64 = (double)p.multiProcessorCount * 64 * 1.965e9;
  printf(", \"fp64_nominal_fma_per_s\": %.4e}\n", nominal64);
  return 0;
}
