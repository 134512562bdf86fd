// devmath_host.cu -- TEST HARNESS: the library's host/device math (fpe_math.cuh, fpe_polar.cuh)
// compiled as host code so that tests/test_devmath_host.py can check it on the CPU against
// the oracle and mpmath.  Built with -ffp-contract=off (the device side uses _rn intrinsics).
#include "../../paper_2211_06320_b200/csrc/fpe_polar.cuh"

using namespace fpe;

extern "C" {
void dm_lambda_fast(const double* xy, long long n, int cplx, double* lam, int* hard) {
  for (long long i = 0; i < n; ++i) lam[i] = lambda_fast(xy[2 * i], xy[2 * i + 1], cplx != 0, hard + i);
}
void dm_lambda_cr(const double* xy, long long n, int cplx, double* lam, int* hard) {
  for (long long i = 0; i < n; ++i) lam[i] = lambda_cr(xy[2 * i], xy[2 * i + 1], cplx != 0, hard + i);
}
void dm_log2abs(const double* xy, long long n, int cplx, double* hl) {
  for (long long i = 0; i < n; ++i) {
    dd_t v = log2abs_quick(xy[2 * i], xy[2 * i + 1], cplx != 0);
    hl[2 * i] = v.hi; hl[2 * i + 1] = v.lo;
  }
}
void dm_atan2_turns(const double* xy, long long n, double* hl) {
  for (long long i = 0; i < n; ++i) {
    dd_t v = atan2_turns(xy[2 * i], xy[2 * i + 1]);
    hl[2 * i] = v.hi; hl[2 * i + 1] = v.lo;
  }
}
// z^p[i] by the polar route: out = (re, im) mantissa, E
void dm_pow_polar(const double* xy, const long long* p, long long n, int cplx, double* out, long long* E) {
  for (long long i = 0; i < n; ++i) {
    const double x = xy[2 * i], y = xy[2 * i + 1];
    if (cplx) {
      polar_t P = polar_of<true>(x, y);
      xc_t v = pow_polar(P.lam, P.tau, p[i]);
      out[2 * i] = v.hr; out[2 * i + 1] = v.hi; E[i] = v.E;
    } else {
      polar_t P = polar_of<false>(x, 0.0);
      xr_t v = pow_polar_real(P.lam, P.neg, p[i]);
      out[2 * i] = v.h; out[2 * i + 1] = 0.0; E[i] = v.E;
    }
  }
}
}
extern "C" void dm_ln1p(const double* u, long long n, double* hl) {
  for (long long i = 0; i < n; ++i) {
    dd_t v = ln1p_series(dd_t{u[2 * i], u[2 * i + 1]});
    hl[2 * i] = v.hi; hl[2 * i + 1] = v.lo;
  }
}
// the classifier's enclosure of log2|z| (fpe_math.cuh lambda_enclosure): lo, hi, mid per point
// the work bucketing's sort key and the lambda-estimate range of a bucket (fpe_math.cuh)
extern "C" void dm_bucket_key(const double* xy, long long n, int cplx, unsigned int* key) {
  for (long long i = 0; i < n; ++i) key[i] = bucket_key(xy[2 * i], xy[2 * i + 1], cplx != 0);
}
extern "C" void dm_bucket_estimates(const unsigned int* b, long long n, int cb, double* lohi) {
  for (long long i = 0; i < n; ++i) bucket_estimates(b[i], cb, lohi[2 * i], lohi[2 * i + 1]);
}
extern "C" void dm_lambda_enclosure(const double* xy, long long n, int cplx, double* lmh) {
  for (long long i = 0; i < n; ++i)
    lambda_enclosure(xy[2 * i], xy[2 * i + 1], cplx != 0, lmh[3 * i], lmh[3 * i + 1], lmh[3 * i + 2]);
}
