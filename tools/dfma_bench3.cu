// dfma_bench3.cu -- complex Horner step formulations vs the fp64 pipe (operand reuse study, B200).
// Each kernel: NP points per lane, coefficients broadcast from shared memory (8 hoisted per step as in
// k_eval_tiled), 4 DFMA per coefficient per point.  Prints FMA/s per formulation as JSON.
#include <cstdio>
#include <cuda_runtime.h>

// current evaluator step: pairs of points, u/v then nr/ni (horner_step2_c64)
struct FCur {
  template <int NP>
  __device__ static void step(double (&br)[NP], double (&bi)[NP], const double (&zr)[NP], const double (&zi)[NP], double2 a) {
#pragma unroll
    for (int j = 0; j < NP; j += 2) {
      const double u0 = fma(-bi[j], zi[j], a.x), u1 = fma(-bi[j + 1], zi[j + 1], a.x);
      const double v1 = fma(bi[j + 1], zr[j + 1], a.y), v0 = fma(bi[j], zr[j], a.y);
      const double nr0 = fma(br[j], zr[j], u0), ni0 = fma(br[j], zi[j], v0);
      const double nr1 = fma(br[j + 1], zr[j + 1], u1), ni1 = fma(br[j + 1], zi[j + 1], v1);
      br[j] = nr0; bi[j] = ni0; br[j + 1] = nr1; bi[j + 1] = ni1;
    }
  }
};
// t1 = br zr + ar, t2 = bi zr + ai (coefficient shared as C across points), then nr = t1 - bi zi,
// ni = t2 + br zi (z_i shared as B within a point)
struct FT12 {
  template <int NP>
  __device__ static void step(double (&br)[NP], double (&bi)[NP], const double (&zr)[NP], const double (&zi)[NP], double2 a) {
    double t1[NP], t2[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) t1[j] = fma(br[j], zr[j], a.x);
#pragma unroll
    for (int j = 0; j < NP; ++j) t2[j] = fma(bi[j], zr[j], a.y);
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const double nr = fma(-bi[j], zi[j], t1[j]);
      const double ni = fma(br[j], zi[j], t2[j]);
      br[j] = nr; bi[j] = ni;
    }
  }
};
// per point: t1, t2 (B = zr shared), nr, ni (B = zi shared)
struct FT12i {
  template <int NP>
  __device__ static void step(double (&br)[NP], double (&bi)[NP], const double (&zr)[NP], const double (&zi)[NP], double2 a) {
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const double t1 = fma(br[j], zr[j], a.x);
      const double t2 = fma(bi[j], zr[j], a.y);
      const double nr = fma(-bi[j], zi[j], t1);
      const double ni = fma(br[j], zi[j], t2);
      br[j] = nr; bi[j] = ni;
    }
  }
};
// plain (compiler's choice)
struct FPlain {
  template <int NP>
  __device__ static void step(double (&br)[NP], double (&bi)[NP], const double (&zr)[NP], const double (&zi)[NP], double2 a) {
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const double t = fma(br[j], zr[j], fma(-bi[j], zi[j], a.x));
      bi[j] = fma(br[j], zi[j], fma(bi[j], zr[j], a.y));
      br[j] = t;
    }
  }
};

template <typename F, int NP>
__global__ void __launch_bounds__(128, 3) k_horner(double* out, long long it, double s) {
  __shared__ double2 cf[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) cf[i] = make_double2(1e-3 * i, -1e-3 * i);
  __syncthreads();
  double zr[NP], zi[NP], br[NP], bi[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    zr[j] = s + 1e-9 * (threadIdx.x + 3 * j); zi[j] = 0.1 * s - 1e-9 * threadIdx.x * (j + 1); br[j] = 0; bi[j] = 0;
  }
  for (long long i = 0; i < it; ++i) {
    for (int k = 255; k >= 7; k -= 8) {
      double2 a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = cf[k - u];
#pragma unroll
      for (int u = 0; u < 8; ++u) F::template step<NP>(br, bi, zr, zi, a[u]);
    }
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < NP; ++j) t += br[j] + bi[j];
  if (t == 1.2345) out[0] = t;
}

template <typename K>
double timeit(K launch, double fmas) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch(); cudaDeviceSynchronize();
  cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return fmas / (ms * 1e-3);
}

int main() {
  double* d; cudaMalloc(&d, 8);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount, grid = sms * 3, thr = 128;
  const long long it = 256;
  auto F = [&](int np) { return (double)grid * thr * it * 256 * 4 * np; };
  printf("{\"cur_np4\": %.4e", timeit([&] { k_horner<FCur, 4><<<grid, thr>>>(d, it, 0.999); }, F(4)));
  printf(", \"t12_np4\": %.4e", timeit([&] { k_horner<FT12, 4><<<grid, thr>>>(d, it, 0.999); }, F(4)));
  printf(", \"t12i_np4\": %.4e", timeit([&] { k_horner<FT12i, 4><<<grid, thr>>>(d, it, 0.999); }, F(4)));
  printf(", \"plain_np4\": %.4e", timeit([&] { k_horner<FPlain, 4><<<grid, thr>>>(d, it, 0.999); }, F(4)));
  printf(", \"t12_np2\": %.4e", timeit([&] { k_horner<FT12, 2><<<grid, thr>>>(d, it, 0.999); }, F(2)));
  printf(", \"cur_np2\": %.4e", timeit([&] { k_horner<FCur, 2><<<grid, thr>>>(d, it, 0.999); }, F(2)));
  printf(", \"t12_np6\": %.4e", timeit([&] { k_horner<FT12, 6><<<grid, thr>>>(d, it, 0.999); }, F(6)));
  printf(", \"t12_np8\": %.4e", timeit([&] { k_horner<FT12, 8><<<grid, thr>>>(d, it, 0.999); }, F(8)));
  printf(", \"nominal\": %.4e}\n", (double)sms * 64 * 1.965e9);
  return 0;
}
