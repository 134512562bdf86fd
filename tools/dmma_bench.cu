// dmma_bench.cu -- FP64 tensor-core (mma.sync DMMA) throughput on B200 vs the DFMA pipe.
// Shapes m8n8k4 (sm_80+) and m16n8k4 / m16n8k8 / m16n8k16 (sm_90+); CH independent accumulators per warp.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_m8n8k4(double* out, long long it) {
  double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (long long t = 0; t < it; ++t) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
template <int CH>
__global__ void k_m16n8k4(double* out, long long it) {
  double a0 = 1.0 + 1e-9 * threadIdx.x, a1 = 1.0 - 1e-9 * threadIdx.x, b = 1.0 - 2e-9 * threadIdx.x;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 2 * i; c[i][3] = 1; }
  for (long long t = 0; t < it; ++t) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1.2345) out[0] = s;
}
template <int CH>
__global__ void k_m16n8k8(double* out, long long it) {
  double a[4], b[2];
#pragma unroll
  for (int j = 0; j < 4; ++j) a[j] = 1.0 + 1e-9 * (threadIdx.x + j);
  b[0] = 1.0 - 1e-9 * threadIdx.x; b[1] = 1.0 + 3e-9 * threadIdx.x;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 2 * i; c[i][3] = 1; }
  for (long long t = 0; t < it; ++t) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1.2345) out[0] = s;
}
template <int CH>
__global__ void k_m16n8k16(double* out, long long it) {
  double a[8], b[4];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = 1.0 + 1e-9 * (threadIdx.x + j);
#pragma unroll
  for (int j = 0; j < 4; ++j) b[j] = 1.0 - 1e-9 * (threadIdx.x + j);
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 2 * i; c[i][3] = 1; }
  for (long long t = 0; t < it; ++t) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1.2345) out[0] = s;
}

template <typename K>
double timeit(K launch, double fmas) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch(); cudaDeviceSynchronize();
  cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("\"err\": \"%s\", ", cudaGetErrorString(e)); return 0; }
  return fmas / (ms * 1e-3);
}

int main() {
  double* d; cudaMalloc(&d, 8);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  const long long it = 1 << 14;
  printf("{");
  for (int wpb : {4, 8, 16}) {
    const int grid = sms * 2, thr = 32 * wpb;
    const double warps = (double)grid * wpb;
    printf("\"m8n8k4_w%d\": %.4e, ", wpb, timeit([&] { k_m8n8k4<8><<<grid, thr>>>(d, it); }, warps * it * 8 * 256));
    printf("\"m16n8k4_w%d\": %.4e, ", wpb, timeit([&] { k_m16n8k4<8><<<grid, thr>>>(d, it); }, warps * it * 8 * 512));
    printf("\"m16n8k8_w%d\": %.4e, ", wpb, timeit([&] { k_m16n8k8<8><<<grid, thr>>>(d, it); }, warps * it * 8 * 1024));
    printf("\"m16n8k16_w%d\": %.4e, ", wpb, timeit([&] { k_m16n8k16<4><<<grid, thr>>>(d, it); }, warps * it * 4 * 2048));
  }
  printf("\"dfma_nominal_fma_per_s\": %.4e}\n", (double)sms * 64 * 1.965e9);
  return 0;
}
