// api.cu -- the C ABI of include/fpe.h.
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>
#include "fpe_internal.h"
#include "fpe_math.cuh"
#include "kernels.cuh"
#include "eval_tiled.cuh"

static_assert(sizeof(fpe_diag) == 48, "fpe_diag layout (paper_2211_06320_b200/_lib.py DIAG_BYTES)");

namespace fpe {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

#define FPE_CUDA(call)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      fpe::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return FPE_ERR_CUDA;                                                                  \
    }                                                                                       \
  } while (0)

static size_t dtype_size(int dt) {
  switch (dt) { case FPE_R64: return 8; case FPE_C64: return 16; case FPE_R32: return 4; case FPE_C32: return 8; }
  return 0;
}
static bool dtype_ok(int dt) { return dt >= FPE_R64 && dt <= FPE_C32; }
static bool is_f32(int dt) { return dt == FPE_R32 || dt == FPE_C32; }

// RAII device guard
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) { cudaGetDevice(&prev); if (prev != dev) cudaSetDevice(dev); }
  ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

// internal batch: the radix scan handles up to 2^28 points at a time
constexpr long long kMaxBatch = 1ll << 28;

// workspace = kWsHeader bytes of counters (kStat*) + the path's scratch
static size_t ws_bytes_for(long long n) {
  long long b = n < kMaxBatch ? n : kMaxBatch;
  size_t naive = (((size_t)b * sizeof(int2) + 255) & ~size_t(255)) + (kSparseTab + 2) * sizeof(int);   // lr + table + queue counter
  size_t tiled = tiled_ws_bytes(b);
  return kWsHeader + (naive > tiled ? naive : tiled);
}

// The calling thread's last evaluation (fpe_last_stats): which workspaces hold its counters, the stream
// to synchronise, and the number of library kernels it launched.  Thread-local, so the handle itself is
// never written by fpe_evaluate / fpe_horner (fpe.h: concurrent calls on one handle with distinct
// workspaces are safe).
struct LastCall {
  const void* ws[fpe_poly_s::kHostSlots] = {};
  int nws = 0;
  void* stream = nullptr;
  int device = 0;
  long long launches = 0;
};
static thread_local LastCall g_last;

// Profiling events are recorded only on a handle with fpe_set_profiling on (a debugging mode that writes
// the handle: not for concurrent calls).
Stage::Stage(fpe_poly h_, void* s_) : h(h_), stream(s_) {
  if (!h->profiling) return;
  h->n_stages = 0;
  h->prof_stream = s_;
  cudaEventRecord(static_cast<cudaEvent_t>(h->prof_events[0]), static_cast<cudaStream_t>(s_));
}
void Stage::mark(const char* name) {
  if (!h->profiling) return;
  if (h->n_stages < 15) {
    h->stage_names[h->n_stages] = name;
    ++h->n_stages;
    cudaEventRecord(static_cast<cudaEvent_t>(h->prof_events[h->n_stages]), static_cast<cudaStream_t>(stream));
  }
}

}  // namespace fpe

fpe::PolyDev fpe_poly_s::view() const {
  fpe::PolyDev P;
  const char* b = static_cast<const char*>(dbuf);
  P.hull = reinterpret_cast<const int2*>(b + hdr.off_hull);
  P.coef = b + hdr.off_coef;
  P.prefix = hdr.off_prefix ? reinterpret_cast<const int32_t*>(b + hdr.off_prefix) : nullptr;
  P.sidx = hdr.off_sidx ? reinterpret_cast<const int32_t*>(b + hdr.off_sidx) : nullptr;
  P.k_min = hdr.k_min; P.k_max = hdr.k_max; P.n_good = hdr.n_good;
  P.nv = (int)hdr.n_hull; P.drop = hdr.drop; P.shift = hdr.shift;
  P.sparse = hdr.sparse; P.all_good = hdr.all_good; P.cdt = hdr.dtype; P.wide = hdr.wide;
  long long hmin = 0, hmax = 0;
  for (size_t i = 0; i < hh.size(); ++i) {
    hmin = i ? std::min<long long>(hmin, hh[i]) : hh[i];
    hmax = i ? std::max<long long>(hmax, hh[i]) : hh[i];
  }
  const long long deff = hdr.k_max - hdr.k_min;
  P.dbl_ok = deff < (1ll << 26) && (2 * (hmax - hmin) + hdr.drop) * (deff + 1) < (1ll << 52);
  return P;
}

using namespace fpe;

static fpe_status finish_handle(fpe_poly h) {
  (void)h;
  return FPE_OK;
}

extern "C" {

const char* fpe_status_string(fpe_status s) {
  switch (s) {
    case FPE_OK: return "FPE_OK";
    case FPE_ERR_INVALID_ARG: return "FPE_ERR_INVALID_ARG";
    case FPE_ERR_ZERO_POLY: return "FPE_ERR_ZERO_POLY";
    case FPE_ERR_NONFINITE_COEFF: return "FPE_ERR_NONFINITE_COEFF";
    case FPE_ERR_UNSUPPORTED: return "FPE_ERR_UNSUPPORTED";
    case FPE_ERR_OOM: return "FPE_ERR_OOM";
    case FPE_ERR_CUDA: return "FPE_ERR_CUDA";
  }
  return "FPE_ERR_UNKNOWN";
}

const char* fpe_last_error_detail(void) { return g_err; }

void fpe_destroy(fpe_poly h) {
  if (!h) return;
  DeviceGuard g(h->device);
  if (h->dbuf) cudaFree(h->dbuf);
  if (h->st_dev) cudaFree(h->st_dev);
  for (void* s : h->st_streams) if (s) cudaStreamDestroy(static_cast<cudaStream_t>(s));
  for (void* e : h->st_events) if (e) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  for (void* e : h->prof_events) if (e) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  delete h;
}

fpe_status fpe_precondition(const void* coeffs, int64_t n_coeffs, fpe_dtype dt, int32_t p_bits,
                            int32_t drop_override, int device, void* stream, fpe_poly* out) {
  if (!coeffs || !out || n_coeffs < 1 || !dtype_ok(dt) || p_bits < 0 || drop_override < 0) {
    set_error("fpe_precondition: invalid argument");
    return FPE_ERR_INVALID_ARG;
  }
  if (n_coeffs > (1ll << 31) - 2) { set_error("fpe_precondition: n_coeffs > 2^31-2"); return FPE_ERR_UNSUPPORTED; }
  *out = nullptr;
  int ndev = 0;
  FPE_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) { set_error("fpe_precondition: bad device %d", device); return FPE_ERR_INVALID_ARG; }
  DeviceGuard g(device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // host copy of the coefficients (they may live on the device)
  const size_t nbytes = (size_t)n_coeffs * dtype_size(dt);
  std::vector<uint8_t> host;
  const void* src = coeffs;
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, coeffs) == cudaSuccess &&
      (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged)) {
    host.resize(nbytes);
    FPE_CUDA(cudaMemcpyAsync(host.data(), coeffs, nbytes, cudaMemcpyDeviceToHost, s));
    FPE_CUDA(cudaStreamSynchronize(s));
    src = host.data();
  }
  cudaGetLastError();  // clear a benign error from cudaPointerGetAttributes on plain host memory
  fpe_poly h = new (std::nothrow) fpe_poly_s();
  if (!h) { set_error("out of host memory"); return FPE_ERR_OOM; }
  h->device = device;
  std::vector<uint8_t> flat;
  fpe_status st = precondition_host(src, n_coeffs, dt, p_bits, drop_override, flat, h->hdr, h->hk, h->hh);
  if (st != FPE_OK) { delete h; return st; }
  if (cudaMalloc(&h->dbuf, flat.size()) != cudaSuccess) {
    cudaGetLastError();
    set_error("cudaMalloc(%zu) failed", flat.size());
    delete h;
    return FPE_ERR_OOM;
  }
  cudaError_t e = cudaMemcpyAsync(h->dbuf, flat.data(), flat.size(), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) { set_error("upload failed: %s", cudaGetErrorString(e)); fpe_destroy(h); return FPE_ERR_CUDA; }
  st = finish_handle(h);
  if (st != FPE_OK) { fpe_destroy(h); return st; }
  *out = h;
  return FPE_OK;
}

fpe_status fpe_precondition_gpu(const void* coeffs, int64_t n_coeffs, fpe_dtype dt, int32_t p_bits,
                                int32_t drop_override, int device, void* stream, fpe_poly* out) {
  if (!coeffs || !out || n_coeffs < 1 || !dtype_ok(dt) || p_bits < 0 || drop_override < 0) {
    set_error("fpe_precondition_gpu: invalid argument");
    return FPE_ERR_INVALID_ARG;
  }
  if (n_coeffs > (1ll << 31) - 2) { set_error("fpe_precondition_gpu: n_coeffs > 2^31-2"); return FPE_ERR_UNSUPPORTED; }
  *out = nullptr;
  int ndev = 0;
  FPE_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) { set_error("fpe_precondition_gpu: bad device %d", device); return FPE_ERR_INVALID_ARG; }
  DeviceGuard g(device);
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, coeffs) != cudaSuccess ||
      !(attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) || attr.device != device) {
    cudaGetLastError();
    set_error("fpe_precondition_gpu: coeffs must be device memory of device %d", device);
    return FPE_ERR_INVALID_ARG;
  }
  fpe_poly h = new (std::nothrow) fpe_poly_s();
  if (!h) { set_error("out of host memory"); return FPE_ERR_OOM; }
  h->device = device;
  fpe_status st = precondition_device(coeffs, n_coeffs, dt, p_bits, drop_override, static_cast<cudaStream_t>(stream),
                                      &h->dbuf, h->hdr, h->hk, h->hh);
  if (st != FPE_OK) { delete h; return st; }
  st = finish_handle(h);
  if (st != FPE_OK) { fpe_destroy(h); return st; }
  *out = h;
  return FPE_OK;
}

// -analyse (host): exact classification of a lambda on the handle's cover (the evaluator's predicates,
// by linear scans: intended for low degrees).
namespace {
struct HostClass { int32_t istar, l, r; };
HostClass classify_host(const std::vector<int32_t>& hk, const std::vector<int32_t>& hh, int drop, double lam) {
  const int nv = (int)hk.size(), m = nv - 1;
  int is = m;
  for (int i = 0; i < m; ++i)
    if (fpe::sign_lin(lam, (long long)hk[i + 1] - hk[i], (long long)hh[i + 1] - hh[i]) <= 0) { is = i; break; }
  auto in_band = [&](long long k) {   // cover(k) + lam (k - hk_i*) - hh_i* + D >= 0, exactly
    int sgm = 0;
    while (sgm + 1 < m && hk[sgm + 1] <= k) ++sgm;
    if (m == 0) return true;
    const long long dk = (long long)hk[sgm + 1] - hk[sgm], dh = (long long)hh[sgm + 1] - hh[sgm];
    const long long J = ((long long)hh[sgm] - hh[is] + drop) * dk + dh * (k - hk[sgm]);
    const long long I = (k - hk[is]) * dk;
    return fpe::sign_lin(lam, I, J) >= 0;
  };
  long long l = hk[is], r = hk[is];
  while (l - 1 >= hk[0] && in_band(l - 1)) --l;   // the band is an interval containing hk_i*
  while (r + 1 <= hk[m] && in_band(r + 1)) ++r;
  return HostClass{is, (int32_t)l, (int32_t)r};
}
}  // namespace

fpe_status fpe_analyse(fpe_poly h, double lam_lo, double lam_hi, fpe_interval* out, int64_t cap, int64_t* n) {
  if (!h || !n || !(lam_lo < lam_hi) || !std::isfinite(lam_lo) || !std::isfinite(lam_hi) || cap < 0) {
    set_error("fpe_analyse: invalid argument");
    return FPE_ERR_INVALID_ARG;
  }
  const auto& hk = h->hk;
  const auto& hh = h->hh;
  const int nv = (int)hk.size(), m = nv - 1, drop = h->hdr.drop;
  const long long d_eff = h->hdr.k_max - h->hdr.k_min;
  if ((double)(d_eff + 1) * nv > (double)(1 << 26)) { set_error("fpe_analyse: d_eff * |cover| too large"); return FPE_ERR_UNSUPPORTED; }
  // G_p membership for the kept counts (prefix counts, compact list, or all good)
  DeviceGuard g(h->device);
  std::vector<int32_t> aux;
  if (!h->hdr.all_good) {
    const bool sp = h->hdr.sparse;
    const size_t cnt = sp ? (size_t)h->hdr.n_good : (size_t)(d_eff + 2);
    aux.resize(cnt);
    FPE_CUDA(cudaMemcpy(aux.data(), static_cast<char*>(h->dbuf) + (sp ? h->hdr.off_sidx : h->hdr.off_prefix),
                        cnt * sizeof(int32_t), cudaMemcpyDeviceToHost));
  }
  auto kept = [&](long long l, long long r) -> int32_t {
    if (h->hdr.all_good) return (int32_t)(r - l + 1);
    if (!h->hdr.sparse) return aux[r + 1 - h->hdr.k_min] - aux[l - h->hdr.k_min];
    return (int32_t)(std::upper_bound(aux.begin(), aux.end(), (int32_t)r) - std::lower_bound(aux.begin(), aux.end(), (int32_t)l));
  };
  // candidate breakpoints: slopes, and per region i the band entry/exit values of every index
  std::vector<double> bp;
  for (int i = 0; i < m; ++i) bp.push_back(-(double)(hh[i + 1] - hh[i]) / (double)(hk[i + 1] - hk[i]));
  for (int i = 0; i <= m; ++i) {
    for (int sgm = 0; sgm < std::max(m, 1); ++sgm) {
      const long long k0 = hk[sgm], k1 = m ? hk[sgm + 1] : hk[0];
      for (long long k = k0; k <= k1; ++k) {
        if (k == hk[i]) continue;
        const long long dk = m ? (long long)hk[sgm + 1] - hk[sgm] : 1, dh = m ? (long long)hh[sgm + 1] - hh[sgm] : 0;
        const long long J = ((long long)hh[sgm] - hh[i] + drop) * dk + dh * (k - hk[sgm]);
        const long long I = (k - hk[i]) * dk;
        const double b = -(double)J / (double)I;
        if (b > lam_lo && b < lam_hi) bp.push_back(b);
      }
    }
  }
  bp.push_back(lam_lo);
  bp.push_back(lam_hi);
  std::sort(bp.begin(), bp.end());
  bp.erase(std::unique(bp.begin(), bp.end()), bp.end());
  std::vector<fpe_interval> iv;
  for (size_t j = 0; j + 1 < bp.size(); ++j) {
    const double a = std::max(bp[j], lam_lo), b = std::min(bp[j + 1], lam_hi);
    if (!(a < b)) continue;
    const HostClass c = classify_host(hk, hh, drop, 0.5 * (a + b));
    if (!iv.empty() && iv.back().region == c.istar && iv.back().l == c.l && iv.back().r == c.r) {
      iv.back().lam_hi = b;
    } else {
      iv.push_back(fpe_interval{a, b, c.istar, c.l, c.r, kept(c.l, c.r)});
    }
  }
  *n = (int64_t)iv.size();
  if (out) {
    if (cap < (int64_t)iv.size()) { set_error("fpe_analyse: need %zu intervals", iv.size()); return FPE_ERR_INVALID_ARG; }
    std::copy(iv.begin(), iv.end(), out);
  }
  return FPE_OK;
}

fpe_status fpe_cover_build(const void* coeffs, int64_t n_coeffs, fpe_dtype dt, int device, void* stream,
                           fpe_cover* out) {
  if (!coeffs || !out || n_coeffs < 1 || !dtype_ok(dt)) { set_error("fpe_cover_build: invalid argument"); return FPE_ERR_INVALID_ARG; }
  if (n_coeffs > (1ll << 31) - 2) { set_error("fpe_cover_build: n_coeffs > 2^31-2"); return FPE_ERR_UNSUPPORTED; }
  *out = nullptr;
  int ndev = 0;
  FPE_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) { set_error("fpe_cover_build: bad device %d", device); return FPE_ERR_INVALID_ARG; }
  DeviceGuard g(device);
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, coeffs) != cudaSuccess ||
      !(attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) || attr.device != device) {
    cudaGetLastError();
    set_error("fpe_cover_build: coeffs must be device memory of device %d", device);
    return FPE_ERR_INVALID_ARG;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  fpe_cover c = new (std::nothrow) fpe_cover_s();
  if (!c) { set_error("out of host memory"); return FPE_ERR_OOM; }
  c->cv.device = device;
  const size_t nbytes = (size_t)n_coeffs * dtype_size(dt);
  if (cudaMalloc(&c->cv.owned, nbytes) != cudaSuccess) { cudaGetLastError(); delete c; set_error("cudaMalloc(%zu) failed", nbytes); return FPE_ERR_OOM; }
  cudaError_t e = cudaMemcpyAsync(c->cv.owned, coeffs, nbytes, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) { set_error("copy failed: %s", cudaGetErrorString(e)); c->cv.release(); delete c; return FPE_ERR_CUDA; }
  fpe_status st = cover_build(c->cv.owned, n_coeffs, dt, s, c->cv);
  if (st != FPE_OK) { c->cv.release(); delete c; return st; }
  *out = c;
  return FPE_OK;
}

fpe_status fpe_cover_finish(fpe_cover c, int32_t p_bits, int32_t drop_override, void* stream, fpe_poly* out) {
  if (!c || !out || p_bits < 0 || drop_override < 0) { set_error("fpe_cover_finish: invalid argument"); return FPE_ERR_INVALID_ARG; }
  *out = nullptr;
  DeviceGuard g(c->cv.device);
  fpe_poly h = new (std::nothrow) fpe_poly_s();
  if (!h) { set_error("out of host memory"); return FPE_ERR_OOM; }
  h->device = c->cv.device;
  fpe_status st = cover_finish(c->cv, p_bits, drop_override, static_cast<cudaStream_t>(stream), &h->dbuf, h->hdr,
                               h->hk, h->hh);
  if (st != FPE_OK) { delete h; return st; }
  st = finish_handle(h);
  if (st != FPE_OK) { fpe_destroy(h); return st; }
  *out = h;
  return FPE_OK;
}

void fpe_cover_destroy(fpe_cover c) {
  if (!c) return;
  DeviceGuard g(c->cv.device);
  c->cv.release();
  delete c;
}

fpe_status fpe_precondition_host(const void* coeffs, int64_t n_coeffs, fpe_dtype dt, int32_t p_bits,
                                 int32_t drop_override, void* buf, size_t cap, size_t* bytes) {
  if (!coeffs || !bytes || n_coeffs < 1 || !dtype_ok(dt) || p_bits < 0 || drop_override < 0) {
    set_error("fpe_precondition_host: invalid argument");
    return FPE_ERR_INVALID_ARG;
  }
  if (n_coeffs > (1ll << 31) - 2) { set_error("fpe_precondition_host: n_coeffs > 2^31-2"); return FPE_ERR_UNSUPPORTED; }
  std::vector<uint8_t> flat;
  Header hdr;
  std::vector<int32_t> hk, hh;
  fpe_status st = precondition_host(coeffs, n_coeffs, dt, p_bits, drop_override, flat, hdr, hk, hh);
  if (st != FPE_OK) return st;
  *bytes = flat.size();
  if (!buf || cap < flat.size()) { set_error("fpe_precondition_host: need %zu bytes", flat.size()); return FPE_ERR_INVALID_ARG; }
  std::memcpy(buf, flat.data(), flat.size());
  return FPE_OK;
}

fpe_status fpe_poly_export(fpe_poly h, void* dst, size_t cap, void* stream) {
  if (!h || !dst || cap < h->hdr.bytes) { set_error("fpe_poly_export: invalid argument"); return FPE_ERR_INVALID_ARG; }
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  FPE_CUDA(cudaMemcpyAsync(dst, h->dbuf, h->hdr.bytes, cudaMemcpyDefault, s));
  FPE_CUDA(cudaStreamSynchronize(s));
  return FPE_OK;
}

fpe_status fpe_poly_get_info(fpe_poly h, fpe_poly_info* out) {
  if (!h || !out) { set_error("fpe_poly_get_info: invalid argument"); return FPE_ERR_INVALID_ARG; }
  out->d = h->hdr.n_coeffs - 1;
  out->k_min = h->hdr.k_min; out->k_max = h->hdr.k_max;
  out->n_hull = h->hdr.n_hull; out->n_good = h->hdr.n_good;
  out->p = h->hdr.p; out->drop = h->hdr.drop; out->shift = h->hdr.shift;
  out->sparse = h->hdr.sparse; out->dtype = h->hdr.dtype; out->reserved = 0;
  out->bytes = h->hdr.bytes;
  return FPE_OK;
}

fpe_status fpe_poly_get_hull(fpe_poly h, int32_t* hk, int32_t* hh, int64_t cap, int64_t* n) {
  if (!h || !n) { set_error("fpe_poly_get_hull: invalid argument"); return FPE_ERR_INVALID_ARG; }
  *n = (int64_t)h->hk.size();
  if (cap < *n || !hk || !hh) { set_error("fpe_poly_get_hull: capacity %lld < %lld", (long long)cap, (long long)*n); return FPE_ERR_INVALID_ARG; }
  std::copy(h->hk.begin(), h->hk.end(), hk);
  std::copy(h->hh.begin(), h->hh.end(), hh);
  return FPE_OK;
}

fpe_status fpe_poly_device_buffer(fpe_poly h, const void** dptr, size_t* bytes) {
  if (!h || !dptr || !bytes) { set_error("fpe_poly_device_buffer: invalid argument"); return FPE_ERR_INVALID_ARG; }
  *dptr = h->dbuf;
  *bytes = h->hdr.bytes;
  return FPE_OK;
}

// A header received from elsewhere (another rank, a file): every field the library indexes with must be in
// range and every section inside the buffer, so that no later read leaves it.
static bool header_valid(const Header& H, size_t bytes) {
  if (H.magic != kMagic || H.version != kVersion || H.bytes != bytes) return false;
  if (!dtype_ok(H.dtype) || H.n_coeffs < 1 || H.n_coeffs > (1ll << 31) - 2) return false;
  if (H.k_min < 0 || H.k_min > H.k_max || H.k_max >= H.n_coeffs) return false;
  const long long d_eff = H.k_max - H.k_min;
  if (H.n_hull < 1 || H.n_hull > d_eff + 1 || H.n_good < 1 || H.n_good > d_eff + 1) return false;
  if (H.p < 1 || H.drop < 1 || (H.sparse != 0 && H.sparse != 1) || (H.all_good != 0 && H.all_good != 1) ||
      (H.wide != 0 && H.wide != 1)) return false;
  auto inside = [&](uint64_t off, uint64_t len) { return off >= sizeof(Header) && off <= bytes && len <= bytes - off; };
  const uint64_t csz = dtype_size(H.dtype);
  const uint64_t n_coef = H.sparse ? (uint64_t)H.n_good : (uint64_t)(d_eff + 1 + kCoefPad - 1) / kCoefPad * kCoefPad;
  if (!inside(H.off_hull, (uint64_t)H.n_hull * sizeof(int2)) || !inside(H.off_coef, n_coef * csz)) return false;
  if (!H.sparse && !H.all_good && !inside(H.off_prefix, (uint64_t)(d_eff + 2) * sizeof(int32_t))) return false;
  if (H.sparse && !inside(H.off_sidx, (uint64_t)H.n_good * sizeof(int32_t))) return false;
  return true;
}

fpe_status fpe_poly_from_device_buffer(const void* dptr, size_t bytes, int device, void* stream, fpe_poly* out) {
  if (!dptr || !out || bytes < sizeof(Header)) { set_error("fpe_poly_from_device_buffer: invalid argument"); return FPE_ERR_INVALID_ARG; }
  *out = nullptr;
  int ndev = 0;
  FPE_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) { set_error("fpe_poly_from_device_buffer: bad device %d", device); return FPE_ERR_INVALID_ARG; }
  DeviceGuard g(device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  fpe_poly h = new (std::nothrow) fpe_poly_s();
  if (!h) { set_error("out of host memory"); return FPE_ERR_OOM; }
  h->device = device;
  cudaError_t e = cudaMemcpyAsync(&h->hdr, dptr, sizeof(Header), cudaMemcpyDefault, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) { set_error("header read failed: %s", cudaGetErrorString(e)); delete h; return FPE_ERR_CUDA; }
  if (!header_valid(h->hdr, bytes)) {
    set_error("fpe_poly_from_device_buffer: not a valid fpe buffer (magic/version/size/section bounds)");
    delete h;
    return FPE_ERR_INVALID_ARG;
  }
  if (cudaMalloc(&h->dbuf, bytes) != cudaSuccess) { cudaGetLastError(); set_error("cudaMalloc failed"); delete h; return FPE_ERR_OOM; }
  std::vector<int2> hull;
  try {
    hull.resize(h->hdr.n_hull);
    h->hk.reserve(h->hdr.n_hull);
    h->hh.reserve(h->hdr.n_hull);
  } catch (const std::bad_alloc&) {
    set_error("out of host memory");
    fpe_destroy(h);
    return FPE_ERR_OOM;
  }
  e = cudaMemcpyAsync(h->dbuf, dptr, bytes, cudaMemcpyDefault, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hull.data(), static_cast<const char*>(dptr) + h->hdr.off_hull,
                                            hull.size() * sizeof(int2), cudaMemcpyDefault, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) { set_error("buffer copy failed: %s", cudaGetErrorString(e)); fpe_destroy(h); return FPE_ERR_CUDA; }
  for (auto v : hull) { h->hk.push_back(v.x); h->hh.push_back(v.y); }
  fpe_status st = finish_handle(h);
  if (st != FPE_OK) { fpe_destroy(h); return st; }
  *out = h;
  return FPE_OK;
}

fpe_status fpe_eval_workspace_size(fpe_poly h, int64_t n_points, size_t* bytes) {
  if (!h || !bytes || n_points < 0) { set_error("fpe_eval_workspace_size: invalid argument"); return FPE_ERR_INVALID_ARG; }
  *bytes = ws_bytes_for(n_points);
  return FPE_OK;
}

static fpe_status check_eval_args(fpe_poly h, const void* points, fpe_dtype pt_dt, int64_t n, void* values) {
  if (!h || n < 0 || !dtype_ok(pt_dt) || (n > 0 && (!points || !values))) {
    set_error("fpe_evaluate: invalid argument");
    return FPE_ERR_INVALID_ARG;
  }
  if (is_f32(pt_dt) != is_f32(h->hdr.dtype)) {
    set_error("fpe_evaluate: point precision (%s) must match the coefficient precision",
              is_f32(pt_dt) ? "fp32" : "fp64");
    return FPE_ERR_INVALID_ARG;
  }
  return FPE_OK;
}

// reset_stats: clear the workspace's counters first (fpe_evaluate); fpe_evaluate_host clears its staging
// slots' counters once and lets the chunks accumulate into them.  *launches receives the number of library
// kernels enqueued.
static fpe_status evaluate_impl(fpe_poly h, const void* points, fpe_dtype pt_dt, int64_t n_points,
                                void* values_out, int64_t* exps_out, fpe_diag* diag_out,
                                void* workspace, size_t ws_bytes, void* stream, bool reset_stats,
                                long long* launches_out) {
  *launches_out = 0;
  fpe_status st = check_eval_args(h, points, pt_dt, n_points, values_out);
  if (st != FPE_OK) return st;
  if (n_points == 0) return FPE_OK;
  if (!workspace || ws_bytes < ws_bytes_for(n_points)) {
    set_error("fpe_evaluate: workspace of %zu bytes < %zu", ws_bytes, ws_bytes_for(n_points));
    return FPE_ERR_INVALID_ARG;
  }
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PolyDev P = h->view();
  unsigned long long* stats = static_cast<unsigned long long*>(workspace);
  void* scratch = static_cast<char*>(workspace) + kWsHeader;
  if (reset_stats) FPE_CUDA(cudaMemsetAsync(stats, 0, kWsHeader, s));
  Stage stg(h, s);
  long long launches = 0;
  for (long long off = 0; off < n_points; off += kMaxBatch) {
    const long long m = std::min(kMaxBatch, n_points - off);
    const size_t in_sz = dtype_size(pt_dt);
    const bool cplx_out = (pt_dt == FPE_C64 || pt_dt == FPE_C32 || h->hdr.dtype == FPE_C64 || h->hdr.dtype == FPE_C32);
    const size_t out_sz = is_f32(pt_dt) ? (cplx_out ? 8 : 4) : (cplx_out ? 16 : 8);
    const int out_kind = is_f32(pt_dt) ? (cplx_out ? FPE_C32 : FPE_R32) : (cplx_out ? FPE_C64 : FPE_R64);
    const void* pp = static_cast<const char*>(points) + off * in_sz;
    void* vv = static_cast<char*>(values_out) + off * out_sz;
    long long* ee = exps_out ? reinterpret_cast<long long*>(exps_out) + off : nullptr;
    fpe_diag* dd = diag_out ? diag_out + off : nullptr;
    if (!P.sparse) {
      int l = run_tiled(pt_dt, pp, m, P, vv, ee, dd, scratch, stats, stg, s);
      if (l < 0) { set_error("fpe_evaluate: tiled path rejected the launch"); return FPE_ERR_INVALID_ARG; }
      launches += l;
      if (dd) { launch_confidence(out_kind, m, P, vv, ee, dd, s); launches += 1; }
    } else {
      int2* lr = static_cast<int2*>(scratch);
      launch_classify(pt_dt, pp, m, P, lr, dd, stats + kStatHard, s);
      stg.mark("classify");
      int* tab = reinterpret_cast<int*>(static_cast<char*>(scratch) + (((size_t)m * sizeof(int2) + 255) & ~size_t(255)));
      launch_eval_sparse(pt_dt, pp, m, P, lr, tab, vv, ee, s);
      stg.mark("eval_sparse");
      launches += 3;   // classify, good-index table, evaluation
      if (dd) { launch_confidence(out_kind, m, P, vv, ee, dd, s); launches += 1; }
    }
  }
  *launches_out = launches;       // kernels of this library (memsets not counted)
  FPE_CUDA(cudaGetLastError());
  return FPE_OK;
}

fpe_status fpe_evaluate(fpe_poly h, const void* points, fpe_dtype pt_dt, int64_t n_points,
                        void* values_out, int64_t* exps_out, fpe_diag* diag_out,
                        void* workspace, size_t ws_bytes, void* stream) {
  long long launches = 0;
  const fpe_status st = evaluate_impl(h, points, pt_dt, n_points, values_out, exps_out, diag_out, workspace, ws_bytes,
                                      stream, true, &launches);
  if (st == FPE_OK) {
    g_last = LastCall{};
    g_last.ws[0] = workspace; g_last.nws = n_points > 0 ? 1 : 0;
    g_last.stream = stream; g_last.device = h->device; g_last.launches = launches;
  }
  return st;
}

fpe_status fpe_horner(fpe_poly h, const void* points, fpe_dtype pt_dt, int64_t n_points,
                      void* values_out, int64_t* exps_out, void* workspace, size_t ws_bytes, void* stream) {
  fpe_status st = check_eval_args(h, points, pt_dt, n_points, values_out);
  if (st != FPE_OK) return st;
  if (n_points == 0) return FPE_OK;
  if (!h->hdr.sparse && (!workspace || ws_bytes < 256)) {
    set_error("fpe_horner: workspace of %zu bytes < 256", ws_bytes);
    return FPE_ERR_INVALID_ARG;
  }
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PolyDev P = h->view();
  Stage stg(h, s);
  if (h->hdr.sparse) {   // Horner over the nonzero terms with gap powers
    launch_horner(pt_dt, points, n_points, P, values_out, reinterpret_cast<long long*>(exps_out), s);
  } else {
    run_horner_tiled(pt_dt, points, n_points, P, static_cast<uint32_t*>(workspace), values_out,
                     reinterpret_cast<long long*>(exps_out), s, ws_bytes);
  }
  stg.mark("horner_full");
  g_last = LastCall{};
  g_last.stream = stream; g_last.device = h->device; g_last.launches = 1;
  FPE_CUDA(cudaGetLastError());
  return FPE_OK;
}

fpe_status fpe_evaluate_host(fpe_poly h, const void* points_host, fpe_dtype pt_dt, int64_t n_points,
                             void* values_host, int64_t* exps_host, void* stream) {
  fpe_status st = check_eval_args(h, points_host, pt_dt, n_points, values_host);
  if (st != FPE_OK) return st;
  if (n_points == 0) return FPE_OK;
  DeviceGuard g(h->device);
  (void)stream;
  const bool cplx_out = (pt_dt == FPE_C64 || pt_dt == FPE_C32 || h->hdr.dtype == FPE_C64 || h->hdr.dtype == FPE_C32);
  const size_t in_sz = dtype_size(pt_dt);
  const size_t out_sz = is_f32(pt_dt) ? (cplx_out ? 8 : 4) : (cplx_out ? 16 : 8);
  // Pipeline over kSlots staging slots: H2D of chunk c (one copy stream) -> classify/sort/evaluate on the
  // slot's own kernel stream -> D2H (one copy stream).  Consecutive chunks' kernels overlap, so one
  // chunk's evaluator tail (its last long-window groups) runs beside the next chunk's work; the chunks
  // stay large enough for the evaluator's window sharing (points of similar |z| per group), and the
  // first ones are smaller (a geometric ramp) so that the D2H stream -- the steady-state bound -- starts early.
  static const int kSlots = [] {
    const char* e = std::getenv("FPE_HOST_SLOTS");   // tuning experiments only
    return e ? std::max(2, std::min(fpe_poly_s::kHostSlots, std::atoi(e))) : 6;
  }();
  static const int lg_chunk = [] {
    const char* e = std::getenv("FPE_HOST_CHUNK_LOG2");   // tuning experiments only
    return e ? std::max(16, std::min(26, std::atoi(e))) : 22;
  }();
  static const int lg_first = [] {
    const char* e = std::getenv("FPE_HOST_FIRST_LOG2");   // tuning experiments only
    return e ? std::max(16, std::min(26, std::atoi(e))) : 20;
  }();
  const long long chunk = std::min<long long>(n_points, 1ll << lg_chunk);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t per = al(chunk * in_sz) + al(chunk * out_sz) + al(chunk * 8) + ws_bytes_for(chunk);
  if (h->st_bytes < kSlots * per) {
    if (h->st_dev) { cudaDeviceSynchronize(); cudaFree(h->st_dev); h->st_dev = nullptr; h->st_bytes = 0; }
    if (cudaMalloc(&h->st_dev, kSlots * per) != cudaSuccess) { cudaGetLastError(); set_error("staging cudaMalloc failed"); return FPE_ERR_OOM; }
    h->st_bytes = kSlots * per;
  }
  for (auto& sp : h->st_streams)
    if (!sp) {
      cudaStream_t ns;
      FPE_CUDA(cudaStreamCreateWithFlags(&ns, cudaStreamNonBlocking));
      sp = ns;
    }
  for (auto& e : h->st_events)
    if (!e) {
      cudaEvent_t ev;
      FPE_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      e = ev;
    }
  cudaStream_t s_in = static_cast<cudaStream_t>(h->st_streams[0]);
  cudaStream_t s_out = static_cast<cudaStream_t>(h->st_streams[1]);
  // the exponents' device->host copies on a second stream (a second copy engine), when FPE_HOST_SPLIT_D2H=1
  static const bool split_d2h = [] { const char* e = std::getenv("FPE_HOST_SPLIT_D2H"); return e && e[0] == '1'; }();
  cudaStream_t s_out2 = split_d2h ? static_cast<cudaStream_t>(h->st_streams[2 + fpe_poly_s::kHostSlots]) : s_out;
  auto slot_base = [&](int b) { return static_cast<char*>(h->st_dev) + b * per; };
  auto slot_ws = [&](int b) { return slot_base(b) + al(chunk * in_sz) + al(chunk * out_sz) + al(chunk * 8); };
  // chunk sizes ramp up geometrically from 2^lg_first to `chunk`, so that the first results start their way
  // back to the host early (the D2H stream is the steady-state bound)
  auto next_size = [&](long long cur) { return std::min(chunk, cur * 2); };
  int used = 0;
  {
    long long cur = std::min<long long>(chunk, 1ll << lg_first);
    for (long long off = 0; off < n_points && used < kSlots; off += cur, cur = next_size(cur)) ++used;
  }
  for (int b = 0; b < used; ++b) FPE_CUDA(cudaMemsetAsync(slot_ws(b), 0, kWsHeader, s_in));   // counters, before every chunk
  auto ev = [&](int slot, int kind) { return static_cast<cudaEvent_t>(h->st_events[slot * 4 + kind]); };
  long long launches = 0;
  static const bool trace = std::getenv("FPE_HOST_TRACE") != nullptr;   // debugging: per-chunk timeline
  std::vector<cudaEvent_t> tev;
  cudaEvent_t t0 = nullptr;
  if (trace) { cudaEventCreate(&t0); cudaEventRecord(t0, s_in); }
  auto mark = [&](cudaStream_t st_) {
    if (!trace) return;
    cudaEvent_t e; cudaEventCreate(&e); cudaEventRecord(e, st_); tev.push_back(e);
  };
  auto release_trace = [&]() {
    for (auto e : tev) cudaEventDestroy(e);
    tev.clear();
    if (t0) { cudaEventDestroy(t0); t0 = nullptr; }
  };
  // On an error after work was enqueued, wait for every stream of the pipeline before returning: copies
  // still queued point at the caller's host buffers.
  auto fail = [&](fpe_status e) {
    for (auto sp : h->st_streams) if (sp) cudaStreamSynchronize(static_cast<cudaStream_t>(sp));
    release_trace();
    return e;
  };
#define FPE_CUDA_P(call)                                                                           \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) {                                                                       \
      fpe::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return fail(FPE_ERR_CUDA);                                                                   \
    }                                                                                              \
  } while (0)
  long long next = std::min<long long>(chunk, 1ll << lg_first);
  for (long long off = 0, c = 0, m = 0; off < n_points; off += m, ++c) {
    m = std::min(next, n_points - off);
    next = next_size(next);
    const int b = (int)(c % kSlots);
    cudaStream_t s_ev = static_cast<cudaStream_t>(h->st_streams[2 + b]);
    char* base = slot_base(b);
    void* dp = base;
    void* dv = base + al(chunk * in_sz);
    long long* de = reinterpret_cast<long long*>(base + al(chunk * in_sz) + al(chunk * out_sz));
    void* wsp = slot_ws(b);
    if (c >= kSlots) {   // the slot's previous results copied out
      FPE_CUDA_P(cudaStreamWaitEvent(s_in, ev(b, 2), 0));
      if (split_d2h) FPE_CUDA_P(cudaStreamWaitEvent(s_in, ev(b, 3), 0));
    }
    mark(s_in);
    FPE_CUDA_P(cudaMemcpyAsync(dp, static_cast<const char*>(points_host) + off * in_sz, m * in_sz, cudaMemcpyHostToDevice, s_in));
    mark(s_in);
    FPE_CUDA_P(cudaEventRecord(ev(b, 0), s_in));
    FPE_CUDA_P(cudaStreamWaitEvent(s_ev, ev(b, 0), 0));
    mark(s_ev);
    long long l = 0;
    fpe_status est = evaluate_impl(h, dp, pt_dt, m, dv, exps_host ? reinterpret_cast<int64_t*>(de) : nullptr, nullptr,
                                   wsp, ws_bytes_for(chunk), s_ev, false, &l);
    mark(s_ev);
    if (est != FPE_OK) return fail(est);
    launches += l;
    FPE_CUDA_P(cudaEventRecord(ev(b, 1), s_ev));
    FPE_CUDA_P(cudaStreamWaitEvent(s_out, ev(b, 1), 0));
    mark(s_out);
    FPE_CUDA_P(cudaMemcpyAsync(static_cast<char*>(values_host) + off * out_sz, dv, m * out_sz, cudaMemcpyDeviceToHost, s_out));
    if (split_d2h) FPE_CUDA_P(cudaStreamWaitEvent(s_out2, ev(b, 1), 0));
    if (exps_host) FPE_CUDA_P(cudaMemcpyAsync(exps_host + off, de, m * 8, cudaMemcpyDeviceToHost, s_out2));
    mark(s_out);
    FPE_CUDA_P(cudaEventRecord(ev(b, 2), s_out));
    if (split_d2h) FPE_CUDA_P(cudaEventRecord(ev(b, 3), s_out2));
  }
#undef FPE_CUDA_P
  cudaError_t se = cudaStreamSynchronize(s_out);
  if (se == cudaSuccess && split_d2h) se = cudaStreamSynchronize(s_out2);
  if (se != cudaSuccess) {
    set_error("fpe_evaluate_host: %s", cudaGetErrorString(se));
    return fail(FPE_ERR_CUDA);
  }
  if (trace) {   // chunk: h2d [start, end], kernels [start, end], d2h [start, end] in ms from the call
    cudaDeviceSynchronize();
    for (size_t k = 0; k + 5 < tev.size() + 0; k += 6) {
      float v[6];
      for (int q = 0; q < 6; ++q) cudaEventElapsedTime(&v[q], t0, tev[k + q]);
      std::fprintf(stderr, "chunk %zu: h2d %.2f-%.2f  eval %.2f-%.2f  d2h %.2f-%.2f\n", k / 6, v[0], v[1], v[2], v[3],
                   v[4], v[5]);
    }
    release_trace();
  }
  g_last = LastCall{};
  for (int b = 0; b < used; ++b) g_last.ws[b] = slot_ws(b);
  g_last.nws = used;
  g_last.stream = s_out; g_last.device = h->device; g_last.launches = launches;
  return FPE_OK;
}

fpe_status fpe_precondition_derivative(const void* coeffs, int64_t n_coeffs, fpe_dtype dt, int32_t p_bits,
                                       int32_t drop_override, int device, void* stream, fpe_poly* out) {
  if (!coeffs || !out || n_coeffs < 1 || !dtype_ok(dt)) {
    set_error("fpe_precondition_derivative: invalid argument");
    return FPE_ERR_INVALID_ARG;
  }
  if (n_coeffs < 2) { set_error("fpe_precondition_derivative: P is constant"); return FPE_ERR_ZERO_POLY; }
  DeviceGuard g(device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t esz = dtype_size(dt);
  std::vector<uint8_t> src((size_t)n_coeffs * esz);
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, coeffs) == cudaSuccess &&
      (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged)) {
    FPE_CUDA(cudaMemcpyAsync(src.data(), coeffs, src.size(), cudaMemcpyDeviceToHost, s));
    FPE_CUDA(cudaStreamSynchronize(s));
  } else {
    cudaGetLastError();
    std::memcpy(src.data(), coeffs, src.size());
  }
  const int64_t m = n_coeffs - 1;
  std::vector<uint8_t> der((size_t)m * esz);
  for (int64_t j = 0; j < m; ++j) {
    const double f = (double)(j + 1);
    switch (dt) {
      case FPE_R64: reinterpret_cast<double*>(der.data())[j] = f * reinterpret_cast<const double*>(src.data())[j + 1]; break;
      case FPE_C64:
        for (int c = 0; c < 2; ++c)
          reinterpret_cast<double*>(der.data())[2 * j + c] = f * reinterpret_cast<const double*>(src.data())[2 * (j + 1) + c];
        break;
      case FPE_R32: reinterpret_cast<float*>(der.data())[j] = (float)(f * reinterpret_cast<const float*>(src.data())[j + 1]); break;
      default:
        for (int c = 0; c < 2; ++c)
          reinterpret_cast<float*>(der.data())[2 * j + c] = (float)(f * reinterpret_cast<const float*>(src.data())[2 * (j + 1) + c]);
        break;
    }
  }
  return fpe_precondition(der.data(), m, dt, p_bits, drop_override, device, stream, out);
}

fpe_status fpe_newton_workspace_size(fpe_poly P, fpe_poly dP, int64_t n_points, size_t* bytes) {
  if (!P || !dP || !bytes || n_points < 0) { set_error("fpe_newton_workspace_size: invalid argument"); return FPE_ERR_INVALID_ARG; }
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t osz = is_f32(P->hdr.dtype) ? 8 : 16;   // complex output is the largest
  *bytes = 2 * (al((size_t)n_points * osz) + al((size_t)n_points * 8)) + ws_bytes_for(n_points);
  return FPE_OK;
}

fpe_status fpe_newton_step(fpe_poly P, fpe_poly dP, const void* points, fpe_dtype pt_dt, int64_t n_points,
                           void* points_out, void* incr_out, void* workspace, size_t ws_bytes, void* stream) {
  fpe_status st = check_eval_args(P, points, pt_dt, n_points, points_out);
  if (st != FPE_OK) return st;
  if (!dP || dP->device != P->device || is_f32(dP->hdr.dtype) != is_f32(P->hdr.dtype)) {
    set_error("fpe_newton_step: P and P' must be handles of the same device and precision");
    return FPE_ERR_INVALID_ARG;
  }
  if (n_points == 0) return FPE_OK;
  size_t need = 0;
  fpe_newton_workspace_size(P, dP, n_points, &need);
  if (!workspace || ws_bytes < need) { set_error("fpe_newton_step: workspace of %zu bytes < %zu", ws_bytes, need); return FPE_ERR_INVALID_ARG; }
  DeviceGuard g(P->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  // both values in the output type of the complex-or-real evaluation of P
  const bool cplx = (pt_dt == FPE_C64 || pt_dt == FPE_C32 || P->hdr.dtype == FPE_C64 || P->hdr.dtype == FPE_C32 ||
                     dP->hdr.dtype == FPE_C64 || dP->hdr.dtype == FPE_C32);
  const size_t osz = is_f32(pt_dt) ? (cplx ? 8 : 4) : (cplx ? 16 : 8);
  char* p = static_cast<char*>(workspace);
  void* v1 = p; p += al((size_t)n_points * osz);
  int64_t* e1 = reinterpret_cast<int64_t*>(p); p += al((size_t)n_points * 8);
  void* v2 = p; p += al((size_t)n_points * osz);
  int64_t* e2 = reinterpret_cast<int64_t*>(p); p += al((size_t)n_points * 8);
  const size_t ws = ws_bytes_for(n_points);
  if (P->hdr.dtype != dP->hdr.dtype) {
    set_error("fpe_newton_step: P and P' must have the same coefficient type");
    return FPE_ERR_INVALID_ARG;
  }
  st = fpe_evaluate(P, points, pt_dt, n_points, v1, e1, nullptr, p, ws, stream);
  if (st != FPE_OK) return st;
  long long launches = g_last.launches;
  st = fpe_evaluate(dP, points, pt_dt, n_points, v2, e2, nullptr, p, ws, stream);
  if (st != FPE_OK) return st;
  launches += g_last.launches;
  const int ok = is_f32(pt_dt) ? (cplx ? FPE_C32 : FPE_R32) : (cplx ? FPE_C64 : FPE_R64);
  launch_newton(pt_dt, ok, n_points, points, v1, reinterpret_cast<const long long*>(e1), v2,
                reinterpret_cast<const long long*>(e2), points_out, incr_out, s);
  g_last.launches = launches + 1;   // counters: those of the P' evaluation (the workspace is reused)
  FPE_CUDA(cudaGetLastError());
  return FPE_OK;
}

fpe_status fpe_set_profiling(fpe_poly h, int enable) {
  if (!h) { set_error("fpe_set_profiling: invalid argument"); return FPE_ERR_INVALID_ARG; }
  DeviceGuard g(h->device);
  if (enable && !h->prof_events[0])
    for (auto& e : h->prof_events) {
      cudaEvent_t ev;
      FPE_CUDA(cudaEventCreate(&ev));
      e = ev;
    }
  h->profiling = enable != 0;
  return FPE_OK;
}

fpe_status fpe_last_stage_ms(fpe_poly h, float* ms, int cap, int* n) {
  if (!h || !n || (cap > 0 && !ms)) { set_error("fpe_last_stage_ms: invalid argument"); return FPE_ERR_INVALID_ARG; }
  *n = h->n_stages;
  if (!h->profiling) { set_error("fpe_last_stage_ms: profiling is off"); return FPE_ERR_INVALID_ARG; }
  DeviceGuard g(h->device);
  FPE_CUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(h->prof_events[h->n_stages])));
  for (int i = 0; i < h->n_stages && i < cap; ++i)
    FPE_CUDA(cudaEventElapsedTime(ms + i, static_cast<cudaEvent_t>(h->prof_events[i]),
                                  static_cast<cudaEvent_t>(h->prof_events[i + 1])));
  return FPE_OK;
}

const char* fpe_stage_name(fpe_poly h, int i) {
  if (!h || i < 0 || i >= h->n_stages) return nullptr;
  return h->stage_names[i];
}

static fpe_status read_counters(const void* ws, cudaStream_t s, unsigned long long* v) {
  FPE_CUDA(cudaStreamSynchronize(s));
  FPE_CUDA(cudaMemcpy(v, ws, kStatCount * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  return FPE_OK;
}

fpe_status fpe_workspace_stats(const void* workspace, void* stream, int64_t* stats, int cap, int* n) {
  if (!workspace || !n || (cap > 0 && !stats) || cap < 0) {
    set_error("fpe_workspace_stats: invalid argument");
    return FPE_ERR_INVALID_ARG;
  }
  unsigned long long v[kStatCount];
  fpe_status st = read_counters(workspace, static_cast<cudaStream_t>(stream), v);
  if (st != FPE_OK) return st;
  *n = kStatCount;
  for (int i = 0; i < kStatCount && i < cap; ++i) stats[i] = (int64_t)v[i];
  return FPE_OK;
}

fpe_status fpe_last_stats(fpe_poly h, int64_t* stats4) {
  if (!h || !stats4) { set_error("fpe_last_stats: invalid argument"); return FPE_ERR_INVALID_ARG; }
  DeviceGuard g(g_last.device);
  unsigned long long tot[kStatCount] = {};
  for (int b = 0; b < g_last.nws; ++b) {
    unsigned long long v[kStatCount];
    fpe_status st = read_counters(g_last.ws[b], static_cast<cudaStream_t>(g_last.stream), v);
    if (st != FPE_OK) return st;
    for (int i = 0; i < kStatCount; ++i) tot[i] += v[i];
  }
  stats4[0] = (int64_t)tot[kStatHard];
  stats4[1] = g_last.launches;
  stats4[2] = (int64_t)tot[kStatMmaItems];
  stats4[3] = (int64_t)tot[kStatMmaInWarp];
  return FPE_OK;
}

}  // extern "C"
