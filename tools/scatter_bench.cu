// Bucket-scatter microbenchmark (tools/, not part of the library): 2^26 points, 148 source ranges x
// 32768 buckets (the k_classify_bucket / k_bucket_scatter layout), positions precomputed on the host.
//   a) 32-byte record scatter  rec[pos[i]] = {i, key, l, r, x, y}       (what k_bucket_scatter does)
//   b) 4-byte index scatter    idx[pos[i]] = i
//   c) bucket-order gather of lr (8 B) + point (16 B) through idx        (what an evaluator would then read)
//   d) sequential read of the 32-byte records                             (what the evaluator reads today)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/scatter_bench tools/scatter_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

struct __align__(32) Rec { int32_t idx; uint32_t key; int32_t l, r; double x, y; };

__global__ void k_rec(const uint32_t* pos, const double2* pts, const int2* lr, long long n, Rec* rec) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double2 z = pts[i]; const int2 w = lr[i];
    rec[pos[i]] = Rec{(int32_t)i, 0u, w.x, w.y, z.x, z.y};
  }
}
__global__ void k_idx(const uint32_t* pos, long long n, uint32_t* idx) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    idx[pos[i]] = (uint32_t)i;
}
__global__ void k_gather(const uint32_t* idx, const double2* pts, const int2* lr, long long n, double* out) {
  double s = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint32_t j = idx[i];
    const double2 z = pts[j]; const int2 w = lr[j];
    s += z.x + z.y + w.x + w.y;
  }
  if (s == 12345.678) out[0] = s;
}
__global__ void k_seq(const Rec* rec, long long n, double* out) {
  double s = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const Rec r = rec[i];
    s += r.x + r.y + r.l + r.r;
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  const long long n = 1ll << 26;
  const int nb = 32768, nc = 148;
  const long long ppc = (n + nc - 1) / nc;
  std::vector<uint32_t> key(n), cnt((size_t)nc * nb, 0), tot(nb, 0), start(nb + 1, 0);
  uint64_t st = 88172645463325252ull;
  for (long long i = 0; i < n; ++i) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    key[i] = (uint32_t)(st % nb);
    ++tot[key[i]];
  }
  for (int b = 0; b < nb; ++b) start[b + 1] = start[b] + tot[b];
  std::vector<uint32_t> base((size_t)nc * nb), pos(n);
  {
    std::vector<uint32_t> run(start.begin(), start.end() - 1);
    for (int c = 0; c < nc; ++c) {
      std::vector<uint32_t> loc(nb, 0);
      for (long long i = c * ppc; i < std::min(n, (c + 1) * ppc); ++i) ++loc[key[i]];
      for (int b = 0; b < nb; ++b) { base[(size_t)c * nb + b] = run[b]; run[b] += loc[b]; }
      std::fill(loc.begin(), loc.end(), 0);
      for (long long i = c * ppc; i < std::min(n, (c + 1) * ppc); ++i) pos[i] = base[(size_t)c * nb + key[i]] + loc[key[i]]++;
    }
  }
  uint32_t *dpos, *didx; double2* dpts; int2* dlr; Rec* drec; double* dout;
  cudaMalloc(&dpos, n * 4); cudaMalloc(&didx, n * 4); cudaMalloc(&dpts, n * 16); cudaMalloc(&dlr, n * 8);
  cudaMalloc(&drec, n * 32); cudaMalloc(&dout, 8);
  cudaMemcpy(dpos, pos.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemset(dpts, 0, n * 16); cudaMemset(dlr, 0, n * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = 148 * 8, blk = 256;
  auto tm = [&](const char* name, auto f, double bytes) {
    for (int w = 0; w < 3; ++w) f();
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) f();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
    printf("%-48s %7.3f ms  %6.2f TB/s (algorithmic)\n", name, ms, bytes / ms / 1e9);
  };
  tm("a) 32-B record scatter", [&] { k_rec<<<grid, blk>>>(dpos, dpts, dlr, n, drec); }, n * (4 + 16 + 8 + 32.0));
  tm("b) 4-B index scatter", [&] { k_idx<<<grid, blk>>>(dpos, n, didx); }, n * 8.0);
  tm("c) gather lr + point by index (bucket order)", [&] { k_gather<<<grid, blk>>>(didx, dpts, dlr, n, dout); }, n * 28.0);
  tm("d) sequential 32-B record read", [&] { k_seq<<<grid, blk>>>(drec, n, dout); }, n * 32.0);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
