// dfma_bench2.cu -- which DFMA operand patterns reach the fp64 pipe peak on B200 (register-file
// bandwidth study for the Horner step).  Prints one JSON object of FMA/s per pattern.
#include <cstdio>
#include <cuda_runtime.h>

#define CH 8
// V_u: 1 vector operand + 2 uniform (the fp64_peak pattern)
__global__ void v_uniform(double* out, long long it, double y, double z) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  for (long long i = 0; i < it; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], y, z);
  double t = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) t += x[c];
  if (t == 1.2345) out[0] = t;
}
// V_shared: y, z per-thread registers shared by all chains (B and C reusable)
__global__ void v_shared(double* out, long long it, double s) {
  double x[CH];
  const double y = s + 1e-9 * threadIdx.x, z = 1e-7 * threadIdx.x;
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  for (long long i = 0; i < it; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], y, z);
  double t = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) t += x[c];
  if (t == 1.2345) out[0] = t;
}
// V_yc: y per chain, z shared
__global__ void v_yc(double* out, long long it, double s) {
  double x[CH], y[CH];
  const double z = 1e-7 * threadIdx.x;
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x + c; y[c] = s + 1e-9 * (threadIdx.x + c); }
  for (long long i = 0; i < it; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], y[c], z);
  double t = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) t += x[c];
  if (t == 1.2345) out[0] = t;
}
// V_yu: y per chain (vector), z uniform
__global__ void v_yu(double* out, long long it, double s, double z) {
  double x[CH], y[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x + c; y[c] = s + 1e-9 * (threadIdx.x + c); }
  for (long long i = 0; i < it; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], y[c], z);
  double t = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) t += x[c];
  if (t == 1.2345) out[0] = t;
}
// complex Horner step, 4 points per lane, z per point in registers, coefficient from smem broadcast
__global__ void v_horner4(double* out, long long it, double s) {
  __shared__ double2 cf[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) cf[i] = make_double2(1e-3 * i, -1e-3 * i);
  __syncthreads();
  double zr[4], zi[4], br[4], bi[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) { zr[j] = s + 1e-9 * (threadIdx.x + j); zi[j] = 0.1 * s - 1e-9 * threadIdx.x * j; br[j] = 0; bi[j] = 0; }
  for (long long i = 0; i < it; ++i) {
#pragma unroll 4
    for (int k = 255; k >= 0; --k) {
      double2 a = cf[k];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double t = fma(br[j], zr[j], fma(-bi[j], zi[j], a.x));
        bi[j] = fma(br[j], zi[j], fma(bi[j], zr[j], a.y));
        br[j] = t;
      }
    }
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) t += br[j] + bi[j];
  if (t == 1.2345) out[0] = t;
}

template <typename F>
double timeit(F launch, double fmas) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch(); cudaDeviceSynchronize();
  cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return fmas / (ms * 1e-3);
}

int main() {
  double* d; cudaMalloc(&d, 8);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount, grid = sms * 4, thr = 256;
  const long long it = 1 << 16;
  const double base = (double)grid * thr * it * CH;
  printf("{\"uniform_yz\": %.4e", timeit([&] { v_uniform<<<grid, thr>>>(d, it, 0.999999, 1e-7); }, base));
  printf(", \"shared_yz\": %.4e", timeit([&] { v_shared<<<grid, thr>>>(d, it, 0.999999); }, base));
  printf(", \"y_per_chain_z_shared\": %.4e", timeit([&] { v_yc<<<grid, thr>>>(d, it, 0.999999); }, base));
  printf(", \"y_per_chain_z_uniform\": %.4e", timeit([&] { v_yu<<<grid, thr>>>(d, it, 0.999999, 1e-7); }, base));
  const long long ith = 64;
  printf(", \"horner_4pt\": %.4e", timeit([&] { v_horner4<<<grid, thr>>>(d, ith, 0.999); }, (double)grid * thr * ith * 256 * 16));
  printf(", \"nominal\": %.4e}\n", (double)sms * 64 * 1.965e9);
  return 0;
}
