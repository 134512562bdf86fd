// precondition.cpp -- host preconditioner: lines 2-4 of Algorithm FPE_p.
//
//   scales s(a_k)            exact integer scales (R8)
//   concave cover            Andrew's monotone chain over (k, s_k), k increasing -- O(d)
//                            because the points arrive sorted by abscissa (the paper sorts
//                            by scale and inserts; same canonical cover)
//   G_p                      s_k >= cover(k) - D by exact integer cross-multiplication
//                            (eq:threshold)
//   buffers                  dense masked coefficients (+ prefix counts) or a compact
//                            good-index list when |G_p| << d
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include "fpe_internal.h"

namespace fpe {

namespace {

constexpr int32_t kNegInf = INT32_MIN;

int32_t scale_real(double a) {
  if (a == 0.0) return kNegInf;
  int e;
  (void)std::frexp(a, &e);
  return e;
}

// s(x + iy) = e + [x'^2 + y'^2 >= 1] with e = max exponent and x' = x 2^-e, y' = y 2^-e
// (equ:sz).  Decided exactly with 128-bit integers on the significands.
int32_t scale_complex(double re, double im) {
  double ax = std::fabs(re), ay = std::fabs(im);
  if (ay > ax) std::swap(ax, ay);
  if (ax == 0.0) return kNegInf;
  int ex;
  double fx = std::frexp(ax, &ex);                 // ax = fx 2^ex, fx in [1/2, 1)
  if (ay == 0.0) return ex;
  int ey;
  double fy = std::frexp(ay, &ey);
  int k = ex - ey;                                  // >= 0
  if (k >= 53) return ex;                           // y'^2 < 2^-106 < 1 - x'^2 (x' <= 1 - 2^-53)
  // x' = Mx 2^-53, y' = My 2^-(53+k):  x'^2 + y'^2 >= 1  <=>  My^2 >= (2^106 - Mx^2) 4^k
  unsigned __int128 Mx = (unsigned __int128)(uint64_t)std::ldexp(fx, 53);
  unsigned __int128 My = (unsigned __int128)(uint64_t)std::ldexp(fy, 53);
  unsigned __int128 D = ((unsigned __int128)1 << 106) - Mx * Mx;   // > 0
  if ((D >> (106 - 2 * k)) != 0) return ex;          // (2^106 - Mx^2) 4^k >= 2^106 > My^2
  return ex + ((My * My >= (D << (2 * k))) ? 1 : 0);
}

int32_t bit_length(int64_t d) {
  int32_t b = 0;
  while (d > 0) { ++b; d >>= 1; }
  return b;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

fpe_status precondition_host(const void* coeffs, int64_t n, fpe_dtype dt, int32_t p_bits,
                             int32_t drop_override, std::vector<uint8_t>& flat, Header& hdr,
                             std::vector<int32_t>& hk, std::vector<int32_t>& hh) {
  const bool cplx = (dt == FPE_C64 || dt == FPE_C32);
  const bool f32 = (dt == FPE_R32 || dt == FPE_C32);
  auto get = [&](int64_t k, double& re, double& im) {
    if (dt == FPE_R64) { re = static_cast<const double*>(coeffs)[k]; im = 0.0; }
    else if (dt == FPE_C64) { re = static_cast<const double*>(coeffs)[2 * k]; im = static_cast<const double*>(coeffs)[2 * k + 1]; }
    else if (dt == FPE_R32) { re = static_cast<const float*>(coeffs)[k]; im = 0.0; }
    else { re = static_cast<const float*>(coeffs)[2 * k]; im = static_cast<const float*>(coeffs)[2 * k + 1]; }
  };

  // 1. scales, finiteness, k_min / k_max
  std::vector<int32_t> s(n);
  int64_t k_min = -1, k_max = -1;
  for (int64_t k = 0; k < n; ++k) {
    double re, im;
    get(k, re, im);
    if (!std::isfinite(re) || !std::isfinite(im)) {
      set_error("coefficient a_%lld is not finite", (long long)k);
      return FPE_ERR_NONFINITE_COEFF;
    }
    s[k] = cplx ? scale_complex(re, im) : scale_real(re);
    if (s[k] != kNegInf) { if (k_min < 0) k_min = k; k_max = k; }
  }
  if (k_min < 0) { set_error("all %lld coefficients are zero", (long long)n); return FPE_ERR_ZERO_POLY; }
  const int64_t d_eff = k_max - k_min;

  // 2. canonical upper concave cover (monotone chain; collinear points dropped)
  hk.clear(); hh.clear();
  for (int64_t k = k_min; k <= k_max; ++k) {
    if (s[k] == kNegInf) continue;
    while (hk.size() >= 2) {
      size_t m = hk.size();
      int64_t ox = hk[m - 2], oy = hh[m - 2], ax = hk[m - 1], ay = hh[m - 1];
      int64_t cross = (ax - ox) * (int64_t)(s[k] - oy) - (ay - oy) * (k - ox);
      if (cross >= 0) { hk.pop_back(); hh.pop_back(); } else break;
    }
    hk.push_back((int32_t)k); hh.push_back(s[k]);
  }
  const int64_t nv = (int64_t)hk.size();

  // 3. D and G_p
  const int32_t p = p_bits > 0 ? p_bits : (f32 ? 24 : 53);
  const int32_t drop = drop_override > 0 ? drop_override : p + (d_eff >= 1 ? bit_length(d_eff) : 0) + 3;
  std::vector<uint8_t> good(d_eff + 1, 0);
  int64_t n_good = 0;
  {
    int64_t j = 0;
    for (int64_t k = k_min; k <= k_max; ++k) {
      if (s[k] == kNegInf) continue;
      if (nv == 1) { good[k - k_min] = 1; ++n_good; continue; }
      while (j + 1 < nv - 1 && hk[j + 1] <= k) ++j;
      int64_t dk = hk[j + 1] - hk[j], dh = hh[j + 1] - hh[j];
      bool g = ((int64_t)s[k] + drop - hh[j]) * dk >= dh * (k - hk[j]);
      good[k - k_min] = g;
      n_good += g;
    }
  }
  const bool all_good = (n_good == d_eff + 1);
  const bool sparse = (n_good * 32 < d_eff + 1);

  // 4. common power-of-two shift: the largest scale maps to 2^0 so that every Horner
  //    intermediate stays below K 2^D; the smallest good term must
  //    stay normal in the working format.
  int32_t hmax = kNegInf, smin = INT32_MAX;
  for (int64_t i = 0; i < nv; ++i) hmax = std::max(hmax, hh[i]);
  for (int64_t k = k_min; k <= k_max; ++k)
    if (good[k - k_min]) smin = std::min(smin, s[k]);
  // Beyond the format's range for one common shift (good scales spanning more than 1000 / 100 bits, or a
  // drop D too large for the K 2^D bound) the handle is "wide": the coefficients are stored as given
  // (shift 0) and evaluated with per-step exponent tracking (k_eval_wide; north_star "exponent-rescaled
  // Horner", PAPER.md:2361-2373 on the exponent range of hardware formats).
  const int32_t limit = f32 ? 100 : 1000;
  const bool wide = ((int64_t)hmax - smin > limit || drop + 30 > (f32 ? 120 : 1000));
  const int32_t shift = wide ? 0 : hmax;

  // 5. flat buffer
  const size_t csz = f32 ? (cplx ? 8 : 4) : (cplx ? 16 : 8);
  const int64_t n_coef = sparse ? n_good : d_eff + 1;
  const int64_t n_coef_alloc = sparse ? n_coef : (n_coef + kCoefPad - 1) / kCoefPad * kCoefPad;   // TMA chunks read whole
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
  flat.assign(off, 0);
  std::memcpy(flat.data(), &hdr, sizeof(hdr));
  int2* hull = reinterpret_cast<int2*>(flat.data() + hdr.off_hull);
  for (int64_t i = 0; i < nv; ++i) hull[i] = make_int2(hk[i], hh[i]);
  uint8_t* coef = flat.data() + hdr.off_coef;
  auto put = [&](int64_t slot, double re, double im) {
    re = std::ldexp(re, -shift); im = std::ldexp(im, -shift);
    if (f32) {
      float* c = reinterpret_cast<float*>(coef);
      if (cplx) { c[2 * slot] = (float)re; c[2 * slot + 1] = (float)im; } else c[slot] = (float)re;
    } else {
      double* c = reinterpret_cast<double*>(coef);
      if (cplx) { c[2 * slot] = re; c[2 * slot + 1] = im; } else c[slot] = re;
    }
  };
  int64_t slot = 0;
  int32_t* prefix = hdr.off_prefix ? reinterpret_cast<int32_t*>(flat.data() + hdr.off_prefix) : nullptr;
  int32_t* sidx = hdr.off_sidx ? reinterpret_cast<int32_t*>(flat.data() + hdr.off_sidx) : nullptr;
  int32_t cnt = 0;
  for (int64_t k = k_min; k <= k_max; ++k) {
    if (prefix) prefix[k - k_min] = cnt;
    bool g = good[k - k_min];
    cnt += g;
    double re = 0.0, im = 0.0;
    if (g) get(k, re, im);
    if (sparse) {
      if (g) { put(slot, re, im); sidx[slot] = (int32_t)k; ++slot; }
    } else {
      put(k - k_min, re, im);
    }
  }
  if (prefix) prefix[d_eff + 1] = cnt;
  return FPE_OK;
}

}  // namespace fpe
