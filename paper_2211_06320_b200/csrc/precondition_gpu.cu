// precondition_gpu.cu -- lines 2-4 of Algorithm FPE_p on the device (SURVEY.md
// §8(f) row 3: "device-side preconditioner: parallel scales, per-block hulls merged, G_p runs").
//
//   k_pre_scales      s(a_k) per coefficient (exact: frexp, and for complex a_k the 128-bit test
//                     x'^2 + y'^2 >= 1 on the significands), finiteness, k_min / k_max
//   k_pre_hull_chunk  Andrew's monotone chain over each chunk of 1024 consecutive indices (one thread
//                     per chunk; the points arrive sorted by abscissa)
//   k_pre_hull_merge  the same chain over the vertices of 32 consecutive partial covers, repeated until
//                     one cover is left: every vertex of the canonical cover of all points is a vertex of
//                     the cover of any subset containing it, so the merged chain is the canonical cover
//                     (collinear points dropped, as on the host)
//   k_pre_good        G_p: s_k >= cover(k) - D by exact integer cross-multiplication (eq:threshold,
//                     PAPER.md:1512-1521), |G_p|, min scale over G_p, max cover height
//   k_pre_fill        the flat buffer: coefficients a_k 2^-shift (0 outside G_p), prefix counts or the
//                     compact (index, coefficient) list, from an exclusive scan of the G_p flags
//
// The buffer is byte-identical to precondition.cpp's (tests/test_gpu_parity.py compares them).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>
#include "fpe_internal.h"

namespace fpe {

namespace {

constexpr int32_t kNegInf = INT32_MIN;
constexpr int kHullChunk = 1024;   // indices per first-level partial cover
constexpr int kMergeFan = 32;      // partial covers merged per thread and level
constexpr int kScanBlock = 1024;

struct PreStats {
  unsigned int nonfinite;
  int pad;
  long long k_min, k_max;
  long long n_good;
  int smin, hmax;
  long long nv;
};

__device__ __forceinline__ void load_coef(int dt, const void* c, long long k, double& re, double& im) {
  switch (dt) {
    case FPE_R64: re = static_cast<const double*>(c)[k]; im = 0.0; break;
    case FPE_C64: re = static_cast<const double*>(c)[2 * k]; im = static_cast<const double*>(c)[2 * k + 1]; break;
    case FPE_R32: re = static_cast<const float*>(c)[k]; im = 0.0; break;
    default: re = static_cast<const float*>(c)[2 * k]; im = static_cast<const float*>(c)[2 * k + 1]; break;
  }
}

__device__ __forceinline__ int32_t scale_real_d(double a) {
  if (a == 0.0) return kNegInf;
  int e;
  (void)frexp(a, &e);
  return e;
}

// s(x + iy) = e + [x'^2 + y'^2 >= 1], e the larger exponent, decided exactly on the
// 53-bit significands with 128-bit integers (the host's scale_complex, restated for the device).
__device__ __forceinline__ int32_t scale_complex_d(double re, double im) {
  double ax = fabs(re), ay = fabs(im);
  if (ay > ax) { const double t = ax; ax = ay; ay = t; }
  if (ax == 0.0) return kNegInf;
  int ex, ey;
  const double fx = frexp(ax, &ex);
  if (ay == 0.0) return ex;
  const double fy = frexp(ay, &ey);
  const int k = ex - ey;
  if (k >= 53) return ex;
  const unsigned __int128 Mx = (unsigned __int128)(unsigned long long)ldexp(fx, 53);
  const unsigned __int128 My = (unsigned __int128)(unsigned long long)ldexp(fy, 53);
  const unsigned __int128 D = ((unsigned __int128)1 << 106) - Mx * Mx;
  if ((D >> (106 - 2 * k)) != 0) return ex;
  return ex + ((My * My >= (D << (2 * k))) ? 1 : 0);
}

__global__ void k_pre_scales(int dt, const void* __restrict__ coef, long long n, int32_t* __restrict__ s,
                             PreStats* st) {
  long long kmin = 0x7fffffffffffffffll, kmax = -1;
  bool bad = false;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    double re, im;
    load_coef(dt, coef, k, re, im);
    bad = bad || !isfinite(re) || !isfinite(im);
    const int32_t v = (dt == FPE_C64 || dt == FPE_C32) ? scale_complex_d(re, im) : scale_real_d(re);
    s[k] = v;
    if (v != kNegInf) { kmin = min(kmin, k); kmax = max(kmax, k); }
  }
  // warp-aggregated
  for (int o = 16; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  bad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicOr(&st->nonfinite, 1u);
    if (kmax >= 0) {
      atomicMin(reinterpret_cast<unsigned long long*>(&st->k_min), (unsigned long long)kmin);
      atomicMax(reinterpret_cast<unsigned long long*>(&st->k_max), (unsigned long long)kmax);
    }
  }
}

// Push (k, h) onto the chain hk/hh[base..base+m) (canonical: pop while the turn is not strictly right).
__device__ __forceinline__ void chain_push(int2* v, int& m, int k, int h) {
  while (m >= 2) {
    const int2 o = v[m - 2], a = v[m - 1];
    const long long cross = (long long)(a.x - o.x) * (long long)(h - o.y) - (long long)(a.y - o.y) * (long long)(k - o.x);
    if (cross >= 0) --m; else break;
  }
  v[m++] = make_int2(k, h);
}

// First level: chunk c covers indices [k_min + c*kHullChunk, ...) ∩ [k_min, k_max]; its cover goes to
// v[c*kHullChunk ...], its vertex count to cnt[c].
__global__ void k_pre_hull_chunk(const int32_t* __restrict__ s, long long k_min, long long k_max, int2* v,
                                 int* cnt, int nchunks) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const long long k0 = k_min + (long long)c * kHullChunk;
  const long long k1 = min(k_max + 1, k0 + kHullChunk);
  int2* out = v + (size_t)c * kHullChunk;
  int m = 0;
  for (long long k = k0; k < k1; ++k) {
    const int32_t h = s[k];
    if (h != kNegInf) chain_push(out, m, (int)k, h);
  }
  cnt[c] = m;
}

// Merge level: partial covers g*kMergeFan .. of the previous level (stored at stride `stride` in src,
// counts in cnt_src) into one cover per group at dst + g*stride*kMergeFan (in place: the group's own
// first slot), counts into cnt_dst[g].
__global__ void k_pre_hull_merge(int2* v, const int* cnt_src, int* cnt_dst, int nsrc, long long stride) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int first = g * kMergeFan;
  if (first >= nsrc) return;
  const int last = min(nsrc, first + kMergeFan);
  int2* out = v + (size_t)first * stride;
  int m = cnt_src[first];                       // the first partial cover is already in place
  for (int c = first + 1; c < last; ++c) {
    const int2* in = v + (size_t)c * stride;
    const int nc = cnt_src[c];
    for (int i = 0; i < nc; ++i) {
      const int2 p = in[i];
      chain_push(out, m, p.x, p.y);
    }
  }
  cnt_dst[g] = m;
}

// G_p flags (relative index k - k_min), |G_p|, min scale over G_p, max cover height.
__global__ void k_pre_good(const int32_t* __restrict__ s, long long k_min, long long k_max, const int2* __restrict__ hull,
                           int nv, int drop, uint8_t* __restrict__ good, PreStats* st) {
  extern __shared__ int2 sh[];
  const bool staged = nv <= 4096;
  if (staged) {
    for (int i = threadIdx.x; i < nv; i += blockDim.x) sh[i] = hull[i];
    __syncthreads();
  }
  const int2* hv = staged ? sh : hull;
  long long ng = 0;
  int smin = INT32_MAX;
  const long long n = k_max - k_min + 1;
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const long long k = k_min + r;
    const int32_t h = s[k];
    bool g = false;
    if (h != kNegInf) {
      if (nv == 1) {
        g = true;
      } else {
        // segment j: the last j <= nv - 2 with hk[j] <= k
        int a = 0, b = nv - 2;
        while (a < b) { const int mid = (a + b + 1) >> 1; if (hv[mid].x <= k) a = mid; else b = mid - 1; }
        const int2 A = hv[a], B = hv[a + 1];
        const long long dk = (long long)B.x - A.x, dh = (long long)B.y - A.y;
        g = ((long long)h + drop - A.y) * dk >= dh * (k - A.x);
      }
    }
    good[r] = g ? 1 : 0;
    if (g) { ++ng; smin = min(smin, (int)h); }
  }
  for (int o = 16; o > 0; o >>= 1) {
    ng += __shfl_xor_sync(0xffffffffu, ng, o);
    smin = min(smin, __shfl_xor_sync(0xffffffffu, smin, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (ng) atomicAdd(reinterpret_cast<unsigned long long*>(&st->n_good), (unsigned long long)ng);
    atomicMin(&st->smin, smin);
  }
  if (blockIdx.x == 0) {
    int hm = INT32_MIN;
    for (int i = threadIdx.x; i < nv; i += blockDim.x) hm = max(hm, hv[i].y);
    for (int o = 16; o > 0; o >>= 1) hm = max(hm, __shfl_xor_sync(0xffffffffu, hm, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&st->hmax, hm);
  }
}

// Exclusive scan of the G_p flags into int32 counts: per-block totals, their scan, then the blocks.
__global__ void k_scan_block_sums(const uint8_t* __restrict__ f, long long n, int* __restrict__ sums) {
  __shared__ int w[32];
  const long long i = (long long)blockIdx.x * kScanBlock + threadIdx.x;
  int v = i < n ? f[i] : 0;
  v = __reduce_add_sync(0xffffffffu, (unsigned)v);
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    int t = __reduce_add_sync(0xffffffffu, (unsigned)w[threadIdx.x]);
    if (threadIdx.x == 0) sums[blockIdx.x] = t;
  }
}
__global__ void k_scan_sums(int* sums, int nb) {   // one block: exclusive scan in place
  __shared__ int w[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int v = i < nb ? sums[i] : 0;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, x, o); if ((threadIdx.x & 31) >= o) x += y; }
    if ((threadIdx.x & 31) == 31) w[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      int z = w[threadIdx.x];
      for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, z, o); if (threadIdx.x >= o) z += y; }
      w[threadIdx.x] = z;
    }
    __syncthreads();
    const int excl = carry + (threadIdx.x >= 32 ? w[(threadIdx.x >> 5) - 1] : 0) + x - v;
    if (i < nb) sums[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
}

// The coefficient section (and prefix counts / compact list) of the flat buffer.
__global__ void k_pre_fill(int dt, const void* __restrict__ coef, long long k_min, long long n_rel,
                           const uint8_t* __restrict__ good, const int* __restrict__ bsum, int shift, int sparse,
                           uint8_t* __restrict__ out_coef, int32_t* __restrict__ prefix, int32_t* __restrict__ sidx) {
  __shared__ int w[32];
  const long long r = (long long)blockIdx.x * kScanBlock + threadIdx.x;
  const int g = r < n_rel ? good[r] : 0;
  // exclusive rank inside the block
  const unsigned ball = __ballot_sync(0xffffffffu, g);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) w[wid] = __popc(ball);
  __syncthreads();
  if (threadIdx.x < 32) {
    int x = w[threadIdx.x], v = x;
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, x, o); if (threadIdx.x >= o) x += y; }
    w[threadIdx.x] = x - v;
  }
  __syncthreads();
  const int rank = bsum[blockIdx.x] + w[wid] + __popc(ball & ((1u << lane) - 1));
  if (r >= n_rel) return;
  if (prefix) prefix[r] = rank;
  const bool cplx = (dt == FPE_C64 || dt == FPE_C32), f32 = (dt == FPE_R32 || dt == FPE_C32);
  double re = 0.0, im = 0.0;
  if (g) load_coef(dt, coef, k_min + r, re, im);
  re = ldexp(re, -shift); im = ldexp(im, -shift);
  if (sparse) {
    if (!g) return;
    sidx[rank] = (int32_t)(k_min + r);
  }
  const long long slot = sparse ? rank : r;
  if (f32) {
    float* c = reinterpret_cast<float*>(out_coef);
    if (cplx) { c[2 * slot] = (float)re; c[2 * slot + 1] = (float)im; } else c[slot] = (float)re;
  } else {
    double* c = reinterpret_cast<double*>(out_coef);
    if (cplx) { c[2 * slot] = re; c[2 * slot + 1] = im; } else c[slot] = re;
  }
}

int32_t bit_length(long long d) {
  int32_t b = 0;
  while (d > 0) { ++b; d >>= 1; }
  return b;
}
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

// The preconditioner's temporaries (scales, cover, G_p flags, scan sums) come from a library-private
// stream-ordered pool that keeps its memory: cudaMalloc / cudaFree of tens of MiB per call cost more than
// the kernels (cfg3 wall time 3-12 ms, the kernels ~2 ms).  The handle's buffer stays a plain cudaMalloc.
static cudaMemPool_t scratch_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    unsigned long long keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    pools[dev] = pool;
  }
  return pools[dev];
}
static cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
  cudaMemPool_t pool = scratch_pool();
  if (!pool) return cudaMalloc(p, bytes);
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}
// frees on the stream the temporaries were used on (the callers synchronise it before returning)
static void scratch_free(void* p, cudaStream_t s) {
  if (!p) return;
  if (scratch_pool()) cudaFreeAsync(p, s);
  else cudaFree(p);
}

namespace {
struct DevBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  ~DevBuf() { scratch_free(p, s); }
};
}  // namespace

#define PRE_CUDA(x)                                                                                  \
  do {                                                                                               \
    cudaError_t e_ = (x);                                                                            \
    if (e_ != cudaSuccess) { set_error("%s: %s", #x, cudaGetErrorString(e_)); return FPE_ERR_CUDA; } \
  } while (0)

// Stage 1 (independent of p, PAPER.md:1529-1537 remark rem:partialpreproc): scales and the canonical cover.
fpe_status cover_build(const void* coeffs, int64_t n, fpe_dtype dt, cudaStream_t s, CoverDev& cv) {
  cv.coeffs = coeffs; cv.n = n; cv.dt = dt;
  const long long nchunks_max = (n + kHullChunk - 1) / kHullChunk;
  const size_t sz_s = align256((size_t)n * 4), sz_v = align256((size_t)nchunks_max * kHullChunk * sizeof(int2));
  const size_t sz_c = align256((size_t)(nchunks_max + 1) * 4 * 2);
  if (scratch_alloc(&cv.scales, sz_s, s) != cudaSuccess) { cudaGetLastError(); cv.scales = nullptr; set_error("device allocation of %zu bytes failed", sz_s); return FPE_ERR_OOM; }
  DevBuf scratch;
  scratch.s = s;
  const size_t total = sz_v + sz_c + align256(sizeof(PreStats));
  if (scratch_alloc(&scratch.p, total, s) != cudaSuccess) { cudaGetLastError(); scratch.p = nullptr; set_error("device allocation of %zu bytes failed", total); return FPE_ERR_OOM; }
  char* q = static_cast<char*>(scratch.p);
  int32_t* d_s = static_cast<int32_t*>(cv.scales);
  int2* d_v = reinterpret_cast<int2*>(q); q += sz_v;
  int* d_cnt = reinterpret_cast<int*>(q); q += sz_c;
  PreStats* d_st = reinterpret_cast<PreStats*>(q);

  PreStats init{};
  // unsigned atomics on k_min / k_max: k_min left at its initial value <=> every coefficient is zero
  init.k_min = 0x7fffffffffffffffll; init.k_max = 0; init.smin = INT32_MAX; init.hmax = INT32_MIN;
  PRE_CUDA(cudaMemcpyAsync(d_st, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  const int grid = (int)std::min<long long>((n + 255) / 256, 148 * 16);
  k_pre_scales<<<grid, 256, 0, s>>>(dt, coeffs, n, d_s, d_st);
  PreStats st;
  PRE_CUDA(cudaMemcpyAsync(&st, d_st, sizeof(st), cudaMemcpyDeviceToHost, s));
  PRE_CUDA(cudaStreamSynchronize(s));
  if (st.nonfinite) { set_error("a coefficient is not finite"); return FPE_ERR_NONFINITE_COEFF; }
  if (st.k_min == 0x7fffffffffffffffll) { set_error("all %lld coefficients are zero", (long long)n); return FPE_ERR_ZERO_POLY; }
  cv.k_min = st.k_min; cv.k_max = st.k_max;
  const long long d_eff = cv.k_max - cv.k_min;

  // cover: chunk chains, then merges of kMergeFan partial covers until one is left
  int nparts = (int)((d_eff + kHullChunk) / kHullChunk);
  k_pre_hull_chunk<<<(nparts + 127) / 128, 128, 0, s>>>(d_s, cv.k_min, cv.k_max, d_v, d_cnt, nparts);
  long long stride = kHullChunk;
  int* cnt_a = d_cnt;
  int* cnt_b = d_cnt + (nchunks_max + 1);
  while (nparts > 1) {
    const int ng = (nparts + kMergeFan - 1) / kMergeFan;
    k_pre_hull_merge<<<(ng + 127) / 128, 128, 0, s>>>(d_v, cnt_a, cnt_b, nparts, stride);
    std::swap(cnt_a, cnt_b);
    stride *= kMergeFan;
    nparts = ng;
  }
  int nv_i = 0;
  PRE_CUDA(cudaMemcpyAsync(&nv_i, cnt_a, sizeof(int), cudaMemcpyDeviceToHost, s));
  PRE_CUDA(cudaStreamSynchronize(s));
  cv.nv = nv_i;
  if (scratch_alloc(&cv.hull, cv.nv * sizeof(int2), s) != cudaSuccess) { cudaGetLastError(); cv.hull = nullptr; set_error("device allocation failed"); return FPE_ERR_OOM; }
  PRE_CUDA(cudaMemcpyAsync(cv.hull, d_v, cv.nv * sizeof(int2), cudaMemcpyDeviceToDevice, s));
  std::vector<int2> hv(cv.nv);
  PRE_CUDA(cudaMemcpyAsync(hv.data(), d_v, cv.nv * sizeof(int2), cudaMemcpyDeviceToHost, s));
  PRE_CUDA(cudaStreamSynchronize(s));
  cv.hk.resize(cv.nv); cv.hh.resize(cv.nv);
  for (long long i = 0; i < cv.nv; ++i) { cv.hk[i] = hv[i].x; cv.hh[i] = hv[i].y; }
  return FPE_OK;
}

// Stage 2 (for a given p, O(d)): G_p, the shift, the layout and the flat buffer.
fpe_status cover_finish(const CoverDev& cv, int32_t p_bits, int32_t drop_override, cudaStream_t s, void** dbuf,
                        Header& hdr, std::vector<int32_t>& hk, std::vector<int32_t>& hh) {
  const fpe_dtype dt = cv.dt;
  const int64_t n = cv.n;
  const bool cplx = (dt == FPE_C64 || dt == FPE_C32);
  const bool f32 = (dt == FPE_R32 || dt == FPE_C32);
  const long long k_min = cv.k_min, k_max = cv.k_max, d_eff = k_max - k_min, nv = cv.nv;
  const long long nblocks_scan = (d_eff + kScanBlock) / kScanBlock;
  const size_t sz_g = align256((size_t)(d_eff + 1)), sz_b = align256((size_t)(nblocks_scan + 1) * 4);
  DevBuf scratch;
  scratch.s = s;
  const size_t total = sz_g + sz_b + align256(sizeof(PreStats));
  if (scratch_alloc(&scratch.p, total, s) != cudaSuccess) { cudaGetLastError(); scratch.p = nullptr; set_error("device allocation of %zu bytes failed", total); return FPE_ERR_OOM; }
  char* q = static_cast<char*>(scratch.p);
  uint8_t* d_good = reinterpret_cast<uint8_t*>(q); q += sz_g;
  int* d_bsum = reinterpret_cast<int*>(q); q += sz_b;
  PreStats* d_st = reinterpret_cast<PreStats*>(q);
  PreStats init{};
  init.smin = INT32_MAX; init.hmax = INT32_MIN;
  PRE_CUDA(cudaMemcpyAsync(d_st, &init, sizeof(init), cudaMemcpyHostToDevice, s));

  // D and G_p
  const int32_t p = p_bits > 0 ? p_bits : (f32 ? 24 : 53);
  const int32_t drop = drop_override > 0 ? drop_override : p + (d_eff >= 1 ? bit_length(d_eff) : 0) + 3;
  const size_t shm = nv <= 4096 ? (size_t)nv * sizeof(int2) : 0;
  k_pre_good<<<(int)std::min<long long>((d_eff + 256) / 256, 148 * 8), 256, shm, s>>>(
      static_cast<const int32_t*>(cv.scales), k_min, k_max, static_cast<const int2*>(cv.hull), (int)nv, drop, d_good, d_st);
  PreStats st;
  PRE_CUDA(cudaMemcpyAsync(&st, d_st, sizeof(st), cudaMemcpyDeviceToHost, s));
  PRE_CUDA(cudaStreamSynchronize(s));
  hk = cv.hk; hh = cv.hh;
  const long long n_good = st.n_good;
  const bool all_good = (n_good == d_eff + 1);
  const bool sparse = (n_good * 32 < d_eff + 1);
  const int32_t limit = f32 ? 100 : 1000;   // as precondition_host: "wide" handles keep shift 0
  const bool wide = ((long long)st.hmax - st.smin > limit || drop + 30 > (f32 ? 120 : 1000));
  const int32_t shift = wide ? 0 : st.hmax;

  // layout (as precondition_host)
  const size_t csz = f32 ? (cplx ? 8 : 4) : (cplx ? 16 : 8);
  const long long n_coef = sparse ? n_good : d_eff + 1;
  const long long n_coef_alloc = sparse ? n_coef : (n_coef + kCoefPad - 1) / kCoefPad * kCoefPad;
  std::memset(&hdr, 0, sizeof(hdr));
  hdr.magic = kMagic; hdr.version = kVersion; hdr.dtype = dt;
  hdr.n_coeffs = n; hdr.k_min = k_min; hdr.k_max = k_max; hdr.n_hull = nv; hdr.n_good = n_good;
  hdr.p = p; hdr.drop = drop; hdr.shift = shift; hdr.sparse = sparse; hdr.all_good = all_good;
  hdr.wide = wide;
  size_t off = align256(sizeof(Header));
  hdr.off_hull = off; off = align256(off + nv * sizeof(int2));
  hdr.off_coef = off; off = align256(off + n_coef_alloc * csz);
  hdr.off_prefix = 0;
  if (!sparse && !all_good) { hdr.off_prefix = off; off = align256(off + (d_eff + 2) * sizeof(int32_t)); }
  hdr.off_sidx = 0;
  if (sparse) { hdr.off_sidx = off; off = align256(off + n_good * sizeof(int32_t)); }
  hdr.bytes = off;

  void* buf = nullptr;
  if (cudaMalloc(&buf, off) != cudaSuccess) { cudaGetLastError(); set_error("cudaMalloc(%zu) failed", off); return FPE_ERR_OOM; }
  struct BufGuard { void* p; ~BufGuard() { if (p) cudaFree(p); } } guard{buf};
  char* b = static_cast<char*>(buf);
  PRE_CUDA(cudaMemsetAsync(b, 0, off, s));
  PRE_CUDA(cudaMemcpyAsync(b, &hdr, sizeof(hdr), cudaMemcpyHostToDevice, s));
  PRE_CUDA(cudaMemcpyAsync(b + hdr.off_hull, cv.hull, nv * sizeof(int2), cudaMemcpyDeviceToDevice, s));
  const long long n_rel = d_eff + 1;
  const int nb = (int)((n_rel + kScanBlock - 1) / kScanBlock);
  k_scan_block_sums<<<nb, kScanBlock, 0, s>>>(d_good, n_rel, d_bsum);
  k_scan_sums<<<1, 1024, 0, s>>>(d_bsum, nb);
  int32_t* prefix = hdr.off_prefix ? reinterpret_cast<int32_t*>(b + hdr.off_prefix) : nullptr;
  int32_t* sidx = hdr.off_sidx ? reinterpret_cast<int32_t*>(b + hdr.off_sidx) : nullptr;
  k_pre_fill<<<nb, kScanBlock, 0, s>>>(dt, cv.coeffs, k_min, n_rel, d_good, d_bsum, shift, sparse ? 1 : 0,
                                       reinterpret_cast<uint8_t*>(b + hdr.off_coef), prefix, sidx);
  if (prefix) {   // prefix[d_eff + 1] = |G_p|
    const int32_t tot = (int32_t)n_good;
    PRE_CUDA(cudaMemcpyAsync(prefix + d_eff + 1, &tot, sizeof(tot), cudaMemcpyHostToDevice, s));
  }
  PRE_CUDA(cudaGetLastError());
  PRE_CUDA(cudaStreamSynchronize(s));
  guard.p = nullptr;
  *dbuf = buf;
  return FPE_OK;
}

void CoverDev::release() {
  // pool memory; every use of it ended with a synchronisation of its stream (cover_build / cover_finish),
  // and the caller's stream may be gone by now, so it is freed on the legacy default stream
  scratch_free(scales, nullptr);
  scratch_free(hull, nullptr);
  if (owned) cudaFree(owned);
  scales = hull = owned = nullptr;
}

fpe_status precondition_device(const void* coeffs, int64_t n, fpe_dtype dt, int32_t p_bits, int32_t drop_override,
                               cudaStream_t s, void** dbuf, Header& hdr, std::vector<int32_t>& hk,
                               std::vector<int32_t>& hh) {
  CoverDev cv;
  fpe_status st = cover_build(coeffs, n, dt, s, cv);
  if (st == FPE_OK) st = cover_finish(cv, p_bits, drop_override, s, dbuf, hdr, hk, hh);
  cv.release();
  return st;
}

}  // namespace fpe
