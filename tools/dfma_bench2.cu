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

// 2 points, source order arranged for operand reuse (I1 p0, I1 p1, I3 p1, I3 p0, I2 p0, I4 p0, I2 p1, I4 p1)
__global__ void v_order2(double* out, long long it, double s) {
  __shared__ double2 cf[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) cf[i] = make_double2(1e-3 * i, -1e-3 * i);
  __syncthreads();
  const double u0 = 1e-9 * threadIdx.x;
  double zr0 = s + u0, zi0 = 0.1 * s - u0, zr1 = 0.3 * s + 2 * u0, zi1 = -0.2 * s + u0;
  double br0 = 0, bi0 = 0, br1 = 0, bi1 = 0;
  for (long long i = 0; i < it; ++i) {
#pragma unroll 8
    for (int k = 255; k >= 0; --k) {
      const double2 a = cf[k];
      const double u_0 = fma(-bi0, zi0, a.x);
      const double u_1 = fma(-bi1, zi1, a.x);
      const double v_1 = fma(bi1, zr1, a.y);
      const double v_0 = fma(bi0, zr0, a.y);
      const double nr0 = fma(br0, zr0, u_0);
      const double ni0 = fma(br0, zi0, v_0);
      const double nr1 = fma(br1, zr1, u_1);
      const double ni1 = fma(br1, zi1, v_1);
      br0 = nr0; bi0 = ni0; br1 = nr1; bi1 = ni1;
    }
  }
  if (br0 + bi0 + br1 + bi1 == 1.2345) out[0] = br0;
}
// 1 point per lane (4 DFMA per coefficient load)
__global__ void v_np1(double* out, long long it, double s) {
  __shared__ double2 cf[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) cf[i] = make_double2(1e-3 * i, -1e-3 * i);
  __syncthreads();
  const double u0 = 1e-9 * threadIdx.x;
  double zr0 = s + u0, zi0 = 0.1 * s - u0;
  double br0 = 0, bi0 = 0;
  for (long long i = 0; i < it; ++i) {
#pragma unroll 8
    for (int k = 255; k >= 0; --k) {
      const double2 a = cf[k];
      const double t = fma(br0, zr0, fma(-bi0, zi0, a.x));
      bi0 = fma(br0, zi0, fma(bi0, zr0, a.y));
      br0 = t;
    }
  }
  if (br0 + bi0 == 1.2345) out[0] = br0;
}
// 2 points, real-arithmetic split: the coefficient pair is reused across both points
__global__ void v_horner2(double* out, long long it, double s) {
  __shared__ double2 cf[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) cf[i] = make_double2(1e-3 * i, -1e-3 * i);
  __syncthreads();
  const double u0 = 1e-9 * threadIdx.x;
  double zr0 = s + u0, zi0 = 0.1 * s - u0, zr1 = 0.3 * s + 2 * u0, zi1 = -0.2 * s + u0;
  double br0 = 0, bi0 = 0, br1 = 0, bi1 = 0;
  for (long long i = 0; i < it; ++i) {
#pragma unroll 8
    for (int k = 255; k >= 0; --k) {
      const double2 a = cf[k];
      double t = fma(br0, zr0, fma(-bi0, zi0, a.x)); bi0 = fma(br0, zi0, fma(bi0, zr0, a.y)); br0 = t;
      t = fma(br1, zr1, fma(-bi1, zi1, a.x)); bi1 = fma(br1, zi1, fma(bi1, zr1, a.y)); br1 = t;
    }
  }
  if (br0 + bi0 + br1 + bi1 == 1.2345) out[0] = br0;
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
  printf(", \"order2\": %.4e", timeit([&] { v_order2<<<grid, thr>>>(d, ith, 0.999); }, (double)grid * thr * ith * 256 * 8));
  printf(", \"horner2\": %.4e", timeit([&] { v_horner2<<<grid, thr>>>(d, ith, 0.999); }, (double)grid * thr * ith * 256 * 8));
  printf(", \"np1\": %.4e", timeit([&] { v_np1<<<grid, thr>>>(d, ith, 0.999); }, (double)grid * thr * ith * 256 * 4));
  printf(", \"nominal\": %.4e}\n", (double)sms * 64 * 1.965e9);
  return 0;
}
