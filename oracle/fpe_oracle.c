/*
 * oracle/fpe_oracle.c -- CPU ORACLE FOR THE FPE HOT PATH.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  The product (paper_2211_06320_b200/)
 * never links, imports or calls it, and shares no code, header, table or
 * constant with it.
 *
 * What it computes, step by step in the order and notation of Algorithm FPE_p
 * (label algo:fast), plus the plain definition
 * P(z) = sum_k a_k z^k (full Horner) as the reference value:
 *
 *   scales      s(a) = 1 + floor(log2|a|), s(0) = -inf      PAPER.md:509-532 (equ:dsz, eq:sigma)
 *   cover       concave cover of E_P(k) = s(a_k) by the     PAPER.md:1413-1509 (Lemma, sorted insertion)
 *               paper's sorted insertion, made canonical
 *   G_p         s(a_k) >= cover(k) - p - s(d) - 3           PAPER.md:1512-1521 (eq:threshold)
 *   lambda      log2|z|, rounded to nearest fp64            PAPER.md:1131 (eq:defLambda); SURVEY G4
 *   k_lambda    argmax(cover + lambda Id), smallest on ties PAPER.md:1543-1546; SURVEY G5
 *   [l, r]      largest integer interval around k_lambda    PAPER.md:1552-1559 (def:LRN); SURVEY G6
 *               with cover(k)+lambda k >= N - p - s(d) - 3
 *   Q_lambda    sum over G_p cap [l,r] of a_k z^k, as        PAPER.md:1253, 1287 (eq:reducedQlambda),
 *               z^l (binary powering) times Horner
 *   P(z)        full Horner over all coefficients           PAPER.md:111-113 (Horner's scheme)
 *
 * Arithmetic: IEEE binary128 (__float128, 113-bit significand) via libquadmath,
 * with a separate int64 binary exponent so that z^l and P(z) never overflow
 * (PAPER.md:2364-2366 -- fp64 cannot hold z^n for |z|>=2, n>1024).
 * Every extended value is renormalised after every operation.  Nothing is
 * blocked, fused or reordered beyond the algorithm as stated.
 *
 * Readings where the paper is silent: p = 53 for fp64
 * and 24 for fp32 (G1); buffer 3 and d := d_eff = k_max - k_min (G2, G3);
 * lambda := correctly rounded fp64 of the exact log2|z| (G4), hard-to-round
 * cases flagged (Ziv test, 2^-100 relative margin); ties in argmax -> smallest
 * vertex (G5); band inclusive (G6); canonical cover without collinear vertices
 * (G7); exact complex scale (G8); kept set is literally G_p cap [l, r] (G9);
 * insertion sentinel y_{s+1} = +inf (G19).
 *
 * Integer encoding of s(0) = -inf: INT32_MIN.
 */
#include <quadmath.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef __float128 f128;
#define OR_NEG_INF INT32_MIN

/* ------------------------------------------------------------------------ */
/* Scales.  s(z) = sigma  iff  2^(sigma-1) <= |z| < 2^sigma. */
/* ------------------------------------------------------------------------ */

/* Real: frexp gives a = m 2^e with |m| in [1/2, 1), i.e. 2^(e-1) <= |a| < 2^e,
 * so s(a) = e ("for floating-point numbers, the scale coincides with the exponent"). */
int32_t or_scale_real(double a)
{
    if (a == 0.0) return OR_NEG_INF;
    int e;
    (void)frexp(a, &e);
    return (int32_t)e;
}

/* Complex: with e = max(s(Re z), s(Im z)) (equ:sz), x = Re z 2^-e and
 * y = Im z 2^-e are exact, |z 2^-e| lies in [1/2, sqrt 2), and
 * s(z) = e + [x^2 + y^2 >= 1]  (eq:exact2pow).  The test x^2 + y^2 >= 1 is
 * done exactly in binary128 as y^2 >= 1 - x^2 (both sides exact: a square of a
 * 53-bit significand has 106 bits).  SURVEY G8. */
int32_t or_scale_complex(double re, double im)
{
    if (re == 0.0 && im == 0.0) return OR_NEG_INF;
    int ex = INT32_MIN, ey = INT32_MIN;
    if (re != 0.0) (void)frexp(re, &ex);
    if (im != 0.0) (void)frexp(im, &ey);
    int e = ex > ey ? ex : ey;
    f128 x = ldexpq((f128)re, -e);
    f128 y = ldexpq((f128)im, -e);
    f128 lhs = y * y;              /* exact */
    f128 rhs = (f128)1 - x * x;    /* exact: x*x exact, the difference fits 113 bits */
    return (int32_t)(e + (lhs >= rhs ? 1 : 0));
}

void or_scales(const double* a, int64_t n, int is_complex, int32_t* s_out)
{
    for (int64_t k = 0; k < n; ++k)
        s_out[k] = is_complex ? or_scale_complex(a[2 * k], a[2 * k + 1]) : or_scale_real(a[k]);
}

/* s(d) for an integer d >= 1: 1 + floor(log2 d) = bit length of d. */
int32_t or_scale_int(int64_t d)
{
    int32_t b = 0;
    while (d > 0) { ++b; d >>= 1; }
    return b;
}

/* Drop D = p + s(d) + 3 with d := d_eff. */
int32_t or_drop(int32_t p, int64_t d_eff)
{
    return p + (d_eff >= 1 ? or_scale_int(d_eff) : 0) + 3;
}

/* ------------------------------------------------------------------------ */
/* Concave cover by the paper's sorted insertion.          */
/* ------------------------------------------------------------------------ */

typedef struct { int64_t k; int32_t s; } or_pt;

/* "sort the values s_n = s(a_{k_n}) in decreasing order ... In case of equality,
 * k_n is chosen in increasing order". */
static int or_cmp_sorted(const void* pa, const void* pb)
{
    const or_pt* a = (const or_pt*)pa;
    const or_pt* b = (const or_pt*)pb;
    if (a->s != b->s) return a->s > b->s ? -1 : 1;
    return (a->k > b->k) - (a->k < b->k);
}

/* s <= (value at abscissa k of the line through (xa,ha), (xb,hb)), xa < xb, exactly. */
static int or_below_line(int64_t k, int64_t s, int64_t xa, int64_t ha, int64_t xb, int64_t hb)
{
    return (s - ha) * (xb - xa) <= (hb - ha) * (k - xa);
}

/*
 * Build the concave cover of the points (k, s[k]), s[k] != -inf, by the
 * Lemma's construction E_0, E_1, ..., E_d.  The graph of E_n is kept as its
 * vertex list X[lo..hi], H[lo..hi] inside a buffer with room on both sides.
 * Returns the number of vertices of the canonical cover written to hk/hh
 * (collinear vertices removed), 0 if all s are -inf, or -1 if the
 * construction produced a non-concave list (an internal error).
 */
int64_t or_hull(const int32_t* s, int64_t n, int32_t* hk, int32_t* hh)
{
    int64_t cnt = 0;
    for (int64_t k = 0; k < n; ++k) cnt += (s[k] != OR_NEG_INF);
    if (cnt == 0) return 0;
    or_pt* pts = (or_pt*)malloc((size_t)cnt * sizeof(or_pt));
    int64_t* X = (int64_t*)malloc((size_t)(2 * cnt + 2) * sizeof(int64_t));
    int64_t* H = (int64_t*)malloc((size_t)(2 * cnt + 2) * sizeof(int64_t));
    cnt = 0;
    for (int64_t k = 0; k < n; ++k)
        if (s[k] != OR_NEG_INF) { pts[cnt].k = k; pts[cnt].s = s[k]; ++cnt; }
    qsort(pts, (size_t)cnt, sizeof(or_pt), or_cmp_sorted);

    /* E_0: l_0 = r_0 = k_0, E_0(k_0) = s_0. */
    int64_t lo = cnt, hi = cnt;
    X[lo] = pts[0].k; H[lo] = pts[0].s;

    for (int64_t n1 = 1; n1 < cnt; ++n1) {
        int64_t k = pts[n1].k, sv = pts[n1].s;
        if (k > X[lo] && k < X[hi]) continue;           /* k in (l_n, r_n): E_{n+1} = E_n */
        if (k < X[lo]) {                                   /* left extension */
            if (hi > lo && !or_below_line(k, sv, X[lo], H[lo], X[lo + 1], H[lo + 1])) {
                /* s_{n+1} > E~_{n+1}(k_{n+1}): the lines Sigma_j (segment j = [X[lo+j],
                 * X[lo+j+1]]) evaluated at k give y_j increasing in j; binary search
                 * the j with s in (y_{j-1}, y_j]; sentinel y_{nseg} = +inf
                 * joins the new point to r_n. */
                int64_t nseg = hi - lo;
                int64_t a = 1, b = nseg;   /* y_0 < s known; find least j in [1, nseg] with s <= y_j */
                while (a < b) {
                    int64_t j = a + (b - a) / 2;
                    if (or_below_line(k, sv, X[lo + j], H[lo + j], X[lo + j + 1], H[lo + j + 1])) b = j;
                    else a = j + 1;
                }
                lo = lo + a;  /* l'_n = leftmost abscissa of Sigma_j (= r_n for the sentinel) */
            }
            --lo; X[lo] = k; H[lo] = sv;
        } else {                                           /* right extension (mirror image) */
            if (hi > lo && !or_below_line(k, sv, X[hi - 1], H[hi - 1], X[hi], H[hi])) {
                int64_t nseg = hi - lo;
                int64_t a = 1, b = nseg;   /* segment j counted from the right: [X[hi-j-1], X[hi-j]] */
                while (a < b) {
                    int64_t j = a + (b - a) / 2;
                    if (or_below_line(k, sv, X[hi - j - 1], H[hi - j - 1], X[hi - j], H[hi - j])) b = j;
                    else a = j + 1;
                }
                hi = hi - a;
            }
            ++hi; X[hi] = k; H[hi] = sv;
        }
    }

    /* Canonical form: drop vertices where the left and right slopes are equal. */
    int64_t m = 0;
    for (int64_t i = lo; i <= hi; ++i) {
        while (m >= 2) {
            int64_t x0 = hk[m - 2], h0 = hh[m - 2], x1 = hk[m - 1], h1 = hh[m - 1];
            if ((h1 - h0) * (X[i] - x1) == (H[i] - h1) * (x1 - x0)) --m; else break;
        }
        hk[m] = (int32_t)X[i]; hh[m] = (int32_t)H[i]; ++m;
    }
    int64_t ok = 1;
    for (int64_t i = 1; i + 1 < m; ++i) {   /* strictly decreasing slopes */
        int64_t l = (int64_t)(hh[i] - hh[i - 1]) * (hk[i + 1] - hk[i]);
        int64_t r = (int64_t)(hh[i + 1] - hh[i]) * (hk[i] - hk[i - 1]);
        if (!(l > r)) ok = 0;
    }
    free(pts); free(X); free(H);
    return ok ? m : -1;
}

/* Segment j of the cover containing k (hk[j] <= k <= hk[j+1]); nv >= 2. */
static int64_t or_segment(const int32_t* hk, int64_t nv, int64_t k)
{
    int64_t a = 0, b = nv - 2;
    while (a < b) {
        int64_t j = a + (b - a + 1) / 2;
        if (hk[j] <= k) a = j; else b = j - 1;
    }
    return a;
}

/* G_p (eq:threshold): good[k] = [a_k != 0 and s(a_k) >= cover(k) - drop].
 * With k in segment j: (s_k + drop - hh_j) dk_j >= dh_j (k - hk_j), exactly. */
void or_good(const int32_t* s, int64_t n, const int32_t* hk, const int32_t* hh, int64_t nv,
             int32_t drop, uint8_t* good)
{
    for (int64_t k = 0; k < n; ++k) {
        good[k] = 0;
        if (s[k] == OR_NEG_INF || nv == 0) continue;
        if (k < hk[0] || k > hk[nv - 1]) continue;
        if (nv == 1) { good[k] = 1; continue; }
        int64_t j = or_segment(hk, nv, k);
        int64_t dk = hk[j + 1] - hk[j], dh = hh[j + 1] - hh[j];
        good[k] = ((int64_t)s[k] + drop - hh[j]) * dk >= dh * (k - hk[j]);
    }
}

/* ------------------------------------------------------------------------ */
/* lambda = log2|z| (eq:defLambda), correctly rounded to fp64.       */
/* ------------------------------------------------------------------------ */

/* Round a binary128 approximation L (relative error << 2^-100) to fp64 and
 * flag it when L lies within 2^-100 |L| of a rounding boundary (Ziv test). */
static double or_round_checked(f128 L, int32_t* hard)
{
    double d = (double)L;            /* round to nearest */
    if (d == 0.0 || isinf(d)) return d;
    double up = nextafter(d, INFINITY), dn = nextafter(d, -INFINITY);
    f128 mid_up = ((f128)d + (f128)up) / 2, mid_dn = ((f128)d + (f128)dn) / 2;
    f128 margin = fminq(fabsq(mid_up - L), fabsq(L - mid_dn));
    f128 tol = fabsq(L) * 0x1p-100Q;
    if (tol < 0x1p-1180Q) tol = 0x1p-1180Q;
    if (margin <= tol) *hard = 1;
    return d;
}

/* Returns -inf for z = 0 (the lambda -> -inf limit) and NaN for a
 * non-finite z.  Complex case: v = x^2 + y^2 with |x| >= |y|.  Near |z| = 1
 * (v in [1/2, 2]) the relative accuracy of lambda needs t = v - 1 computed as
 * (x^2 - 1) + y^2, where x^2 - 1 is exact, so that lambda = log1p(t)/(2 ln 2);
 * elsewhere lambda = log2(v)/2.  Real case: t = |x| - 1 (exact). */
double or_lambda(double re, double im, int is_complex, int32_t* hard)
{
    *hard = 0;
    if (!isfinite(re) || !isfinite(im)) return NAN;
    if (!is_complex) im = 0.0;
    if (re == 0.0 && im == 0.0) return -INFINITY;
    f128 L;
    if (!is_complex || im == 0.0 || re == 0.0) {
        f128 x = fabsq((f128)(re != 0.0 ? re : im));
        if (x >= 0.5Q && x <= 2.0Q) L = log1pq(x - 1) / M_LN2q;
        else L = log2q(x);
    } else {
        f128 x = fabsq((f128)re), y = fabsq((f128)im);
        if (y > x) { f128 t = x; x = y; y = t; }
        f128 v = x * x + y * y;
        if (v >= 0.5Q && v <= 2.0Q) {
            f128 t = (x * x - 1) + y * y;
            L = log1pq(t) / (2 * M_LN2q);
        } else {
            L = log2q(v) / 2;
        }
    }
    return or_round_checked(L, hard);
}

/* ------------------------------------------------------------------------ */
/* Evaluation-phase searches, exact predicates.            */
/* ------------------------------------------------------------------------ */

/* sign of (lambda * I + J) exactly: lambda*I is exact in binary128 for |I| < 2^60
 * (53 + 60 bits), and rounding the sum preserves its sign. */
static int or_sign_lin(double lam, int64_t I, int64_t J)
{
    f128 v = (f128)lam * (f128)I + (f128)J;
    return (v > 0) - (v < 0);
}

/* f(k) >= 0 where f(k) = cover(k) + lambda k - (N - drop), N = hh_i* + lambda hk_i*.
 * With k in segment j, times dk_j > 0:
 *   (hh_j - hh_i* + drop) dk_j + dh_j (k - hk_j) + lambda (k - hk_i*) dk_j >= 0. */
static int or_in_band(const int32_t* hk, const int32_t* hh, int64_t nv, int64_t istar,
                      int32_t drop, double lam, int64_t k)
{
    if (nv == 1) return 1;
    int64_t j = or_segment(hk, nv, k);
    int64_t dk = hk[j + 1] - hk[j], dh = hh[j + 1] - hh[j];
    int64_t J = ((int64_t)hh[j] - hh[istar] + drop) * dk + dh * (k - hk[j]);
    int64_t I = (k - hk[istar]) * dk;
    return or_sign_lin(lam, I, J) >= 0;
}

/*
 * Per point: lambda, i* (index of the vertex k_lambda), l, r.
 * k_lambda = argmax(cover + lambda Id) (line 6): cover + lambda Id is concave
 * with segment slopes sigma_i + lambda decreasing, so the smallest maximiser is
 * vertex i* = min{i : lambda dk_i + dh_i <= 0} (m if none), found by binary
 * search.  [l, r] (line 8, def:LRN): the two monotone
 * branches around k_lambda are binary-searched for the extreme integers still in
 * the super-level set {f >= 0}, clipped to [k_min, k_max].
 * z = 0: region 0, l = r = k_min; non-finite z: i* = -1.
 */
static void or_search(double lam, const int32_t* hk, const int32_t* hh, int64_t nv, int32_t drop,
                      int32_t* istar_out, int64_t* l_out, int64_t* r_out)
{
    if (isnan(lam)) { *istar_out = -1; *l_out = -1; *r_out = -1; return; }
    if (isinf(lam) && lam < 0) { *istar_out = 0; *l_out = hk[0]; *r_out = hk[0]; return; }
    int64_t m = nv - 1;
    int64_t a = 0, b = m;   /* least i in [0, m) with lambda dk_i + dh_i <= 0, else m */
    while (a < b) {
        int64_t i = a + (b - a) / 2;
        if (or_sign_lin(lam, hk[i + 1] - hk[i], hh[i + 1] - hh[i]) <= 0) b = i; else a = i + 1;
    }
    int64_t istar = a, kst = hk[istar];
    /* l: least k in [k_min, k_lambda] with f(k) >= 0 (f(k_lambda) = drop >= 0) */
    int64_t lo = hk[0], hi = kst;
    while (lo < hi) {
        int64_t k = lo + (hi - lo) / 2;
        if (or_in_band(hk, hh, nv, istar, drop, lam, k)) hi = k; else lo = k + 1;
    }
    int64_t l = lo;
    /* r: greatest k in [k_lambda, k_max] with f(k) >= 0 */
    lo = kst; hi = hk[m];
    while (lo < hi) {
        int64_t k = lo + (hi - lo + 1) / 2;
        if (or_in_band(hk, hh, nv, istar, drop, lam, k)) lo = k; else hi = k - 1;
    }
    *istar_out = (int32_t)istar; *l_out = l; *r_out = lo;
}

void or_classify(const double* pts, int64_t npts, int is_complex,
                 const int32_t* hk, const int32_t* hh, int64_t nv, int32_t drop,
                 double* lam_out, int32_t* istar_out, int64_t* l_out, int64_t* r_out,
                 int32_t* hard_out)
{
    #pragma omp parallel for schedule(dynamic, 256)
    for (int64_t q = 0; q < npts; ++q) {
        double re = is_complex ? pts[2 * q] : pts[q];
        double im = is_complex ? pts[2 * q + 1] : 0.0;
        int32_t hard = 0;
        double lam = or_lambda(re, im, is_complex, &hard);
        lam_out[q] = lam; hard_out[q] = hard;
        or_search(lam, hk, hh, nv, drop, istar_out + q, l_out + q, r_out + q);
    }
}

/* The searches alone, for given lambda values (tests of ties at hull slopes). */
void or_classify_lambda(const double* lams, int64_t n, const int32_t* hk, const int32_t* hh,
                        int64_t nv, int32_t drop, int32_t* istar_out, int64_t* l_out, int64_t* r_out)
{
    #pragma omp parallel for schedule(dynamic, 256)
    for (int64_t q = 0; q < n; ++q)
        or_search(lams[q], hk, hh, nv, drop, istar_out + q, l_out + q, r_out + q);
}

/* ------------------------------------------------------------------------ */
/* Extended-range binary128 complex numbers: (re + i im) 2^e.                   */
/* ------------------------------------------------------------------------ */

typedef struct { f128 re, im; int64_t e; } or_x;

static or_x or_norm(or_x a)
{
    f128 m = fmaxq(fabsq(a.re), fabsq(a.im));
    if (m == 0) { a.e = 0; return a; }
    int ex;
    (void)frexpq(m, &ex);
    a.re = ldexpq(a.re, -ex); a.im = ldexpq(a.im, -ex); a.e += ex;
    return a;
}

static or_x or_from(double re, double im)
{
    or_x a = { (f128)re, (f128)im, 0 };
    return or_norm(a);
}

static or_x or_mul(or_x a, or_x b)
{
    or_x c = { a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re, a.e + b.e };
    return or_norm(c);
}

static f128 or_shift(f128 v, int64_t by)   /* v 2^by for mantissas in [1/2,1) */
{
    if (by < -20000) return 0;
    if (by > 20000) by = 20000;
    return ldexpq(v, (int)by);
}

static or_x or_add(or_x a, or_x b)
{
    if (a.re == 0 && a.im == 0) return b;
    if (b.re == 0 && b.im == 0) return a;
    int64_t e = a.e > b.e ? a.e : b.e;
    or_x c = { or_shift(a.re, a.e - e) + or_shift(b.re, b.e - e),
               or_shift(a.im, a.e - e) + or_shift(b.im, b.e - e), e };
    return or_norm(c);
}

/* z^n by binary powering: "z^(2^alpha) can be computed with alpha successive
 * squarings that can be kept in memory to compute z^beta". */
static or_x or_pow(or_x z, int64_t n)
{
    or_x res = { 1, 0, 0 };
    res = or_norm(res);
    or_x base = z;
    while (n > 0) {
        if (n & 1) res = or_mul(res, base);
        n >>= 1;
        if (n) base = or_mul(base, base);
    }
    return res;
}

static void or_store(or_x v, double* out4, int64_t* e_out)
{
    double rh = (double)v.re, ih = (double)v.im;
    out4[0] = rh; out4[1] = (double)(v.re - (f128)rh);
    out4[2] = ih; out4[3] = (double)(v.im - (f128)ih);
    *e_out = v.e;
}

static or_x or_coef(const double* a, int is_complex, int64_t k)
{
    return is_complex ? or_from(a[2 * k], a[2 * k + 1]) : or_from(a[k], 0.0);
}

static or_x or_point(const double* pts, int is_complex, int64_t q)
{
    return is_complex ? or_from(pts[2 * q], pts[2 * q + 1]) : or_from(pts[q], 0.0);
}

/*
 * Q_lambda(z) = sum_{k in G_p cap [l, r]} a_k z^k  (line 9, eq:reducedQlambda):
 * Horner over k = r, ..., l with the bad / zero indices contributing 0, then
 * times z^l by binary powering ("we compute z^l in 2 log2 l
 * steps and then use Horner's method to compute Q_lambda(z)").
 * out: 4 doubles per point (re_hi, re_lo, im_hi, im_lo) of the mantissa;
 * exps: its binary exponent.  Non-finite points (l < 0) give NaN.
 */
void or_fpe_eval(const double* a, const uint8_t* good, int is_complex,
                 const double* pts, int64_t npts, const int64_t* l, const int64_t* r,
                 double* out, int64_t* exps)
{
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t q = 0; q < npts; ++q) {
        if (l[q] < 0) { for (int i = 0; i < 4; ++i) out[4 * q + i] = NAN; exps[q] = 0; continue; }
        or_x z = or_point(pts, is_complex, q);
        or_x b = { 0, 0, 0 };
        if (z.re == 0 && z.im == 0) {   /* z = 0: P(0) = a_0 (term k_min = 0 only) */
            if (l[q] == 0 && good[0]) b = or_coef(a, is_complex, 0);
            or_store(b, out + 4 * q, exps + q);
            continue;
        }
        for (int64_t k = r[q]; k >= l[q]; --k) {
            b = or_mul(b, z);
            if (good[k]) b = or_add(b, or_coef(a, is_complex, k));
        }
        b = or_mul(b, or_pow(z, l[q]));
        or_store(b, out + 4 * q, exps + q);
    }
}

/* Reference P(z) by full Horner over k = k_max..k_min, times z^k_min. */
void or_horner(const double* a, int64_t kmin, int64_t kmax, int is_complex,
               const double* pts, int64_t npts, double* out, int64_t* exps)
{
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < npts; ++q) {
        or_x z = or_point(pts, is_complex, q);
        or_x b = { 0, 0, 0 };
        if (z.re == 0 && z.im == 0) {
            if (kmin == 0) b = or_coef(a, is_complex, 0);
            or_store(b, out + 4 * q, exps + q);
            continue;
        }
        for (int64_t k = kmax; k >= kmin; --k)
            b = or_add(or_mul(b, z), or_coef(a, is_complex, k));
        b = or_mul(b, or_pow(z, kmin));
        or_store(b, out + 4 * q, exps + q);
    }
}

/* Reference P(z) by full double-double Horner ("P_ref by full double-double Horner
 * with an exponent counter"), the plain definition P(z) = sum_k a_k z^k evaluated as
 * b <- b z + a_k for k = k_max .. k_min, then times z^k_min.  Each component of b is an unevaluated sum
 * hi + lo of two doubles (Dekker / Knuth error-free transformations: ~106-bit significand, relative error
 * ~2^-104 per step); b's value is (hi + lo) 2^E with E an int64, renormalised after every step so that
 * the larger component's hi lies in [1/2, 1); z = w 2^ez with the larger of |Re w|, |Im w| in [1/2, 1).
 * A faster plain reference than the binary128 or_horner for the full-size value checks (d up to 2^22). */
typedef struct { double hi, lo; } or_dd;
static or_dd dd_two_sum(double a, double b)
{
    double s = a + b, bb = s - a;
    or_dd r = { s, (a - (s - bb)) + (b - bb) };
    return r;
}
static or_dd dd_add(or_dd a, or_dd b)   /* accurate double-double addition */
{
    or_dd s = dd_two_sum(a.hi, b.hi), t = dd_two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = dd_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return dd_two_sum(s.hi, s.lo);
}
static or_dd dd_mul_d(or_dd a, double b)
{
    double p = a.hi * b;
    double e = fma(a.hi, b, -p) + a.lo * b;
    return dd_two_sum(p, e);
}
static or_dd dd_neg(or_dd a) { or_dd r = { -a.hi, -a.lo }; return r; }
static or_dd dd_ldexp(or_dd a, int64_t e)
{
    int s = e > 3000 ? 3000 : (e < -3000 ? -3000 : (int)e);
    or_dd r = { ldexp(a.hi, s), ldexp(a.lo, s) };
    return r;
}

void or_horner_dd(const double* a, int64_t kmin, int64_t kmax, int is_complex,
                  const double* pts, int64_t npts, double* out, int64_t* exps)
{
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < npts; ++q) {
        const double zr = is_complex ? pts[2 * q] : pts[q], zi = is_complex ? pts[2 * q + 1] : 0.0;
        or_dd br = { 0, 0 }, bi = { 0, 0 };
        int64_t E = 0;
        if (zr == 0 && zi == 0) {
            if (kmin == 0) { br.hi = is_complex ? a[0] : a[0]; bi.hi = is_complex ? a[1] : 0.0; }
            out[4 * q] = br.hi; out[4 * q + 1] = 0; out[4 * q + 2] = bi.hi; out[4 * q + 3] = 0; exps[q] = 0;
            continue;
        }
        int ez;
        (void)frexp(fabs(zr) > fabs(zi) ? zr : zi, &ez);
        const double wr = ldexp(zr, -ez), wi = ldexp(zi, -ez);   /* exact */
        for (int64_t k = kmax; k >= kmin; --k) {
            /* b <- b w (value times 2^ez) */
            or_dd nr = dd_add(dd_mul_d(br, wr), dd_neg(dd_mul_d(bi, wi)));
            or_dd ni = dd_add(dd_mul_d(br, wi), dd_mul_d(bi, wr));
            br = nr; bi = ni; E += ez;
            /* + a_k: align the two exponents (the smaller operand may underflow: it is then below the
             * larger one's rounding) */
            const double ar = is_complex ? a[2 * k] : a[k], ai = is_complex ? a[2 * k + 1] : 0.0;
            if (ar != 0 || ai != 0) {
                int ea;
                (void)frexp(fabs(ar) > fabs(ai) ? ar : ai, &ea);
                const int bz = (br.hi == 0 && bi.hi == 0);
                int eb = 0;
                if (!bz) (void)frexp(fabs(br.hi) > fabs(bi.hi) ? br.hi : bi.hi, &eb);
                if (bz || (int64_t)ea > E + eb) {      /* the coefficient is larger: work at its scale */
                    br = dd_ldexp(br, E - ea); bi = dd_ldexp(bi, E - ea); E = ea;
                }
                or_dd xr = { ldexp(ar, (int)(ea - E > -3000 ? ea - E : -3000) - ea), 0 };
                or_dd xi = { ldexp(ai, (int)(ea - E > -3000 ? ea - E : -3000) - ea), 0 };
                br = dd_add(br, xr); bi = dd_add(bi, xi);
            }
            /* renormalise: the larger component's hi in [1/2, 1) */
            const double m = fabs(br.hi) > fabs(bi.hi) ? br.hi : bi.hi;
            if (m != 0) {
                int e;
                (void)frexp(m, &e);
                br = dd_ldexp(br, -e); bi = dd_ldexp(bi, -e); E += e;
            } else {
                E = 0;
            }
        }
        /* times z^k_min: (w 2^ez)^k_min by binary powering in double-double */
        if (kmin > 0) {
            or_dd pr = { 1, 0 }, pi = { 0, 0 }, qr = { wr, 0 }, qi = { wi, 0 };
            int64_t pE = 0, qE = ez, n = kmin;
            while (n > 0) {
                if (n & 1) {
                    or_dd tr = dd_add(dd_mul_d(pr, qr.hi), dd_add(dd_mul_d(pr, qr.lo), dd_neg(dd_add(dd_mul_d(pi, qi.hi), dd_mul_d(pi, qi.lo)))));
                    or_dd ti = dd_add(dd_add(dd_mul_d(pr, qi.hi), dd_mul_d(pr, qi.lo)), dd_add(dd_mul_d(pi, qr.hi), dd_mul_d(pi, qr.lo)));
                    pr = tr; pi = ti; pE += qE;
                }
                n >>= 1;
                if (n) {
                    or_dd tr = dd_add(dd_add(dd_mul_d(qr, qr.hi), dd_mul_d(qr, qr.lo)), dd_neg(dd_add(dd_mul_d(qi, qi.hi), dd_mul_d(qi, qi.lo))));
                    or_dd ti = dd_add(dd_add(dd_mul_d(qr, qi.hi), dd_mul_d(qr, qi.lo)), dd_add(dd_mul_d(qi, qr.hi), dd_mul_d(qi, qr.lo)));
                    qr = tr; qi = ti; qE *= 2;
                }
                int e;
                double mp_ = fabs(pr.hi) > fabs(pi.hi) ? pr.hi : pi.hi;
                (void)frexp(mp_, &e); pr = dd_ldexp(pr, -e); pi = dd_ldexp(pi, -e); pE += e;
                double mq = fabs(qr.hi) > fabs(qi.hi) ? qr.hi : qi.hi;
                (void)frexp(mq, &e); qr = dd_ldexp(qr, -e); qi = dd_ldexp(qi, -e); qE += e;
            }
            or_dd tr = dd_add(dd_add(dd_mul_d(br, pr.hi), dd_mul_d(br, pr.lo)), dd_neg(dd_add(dd_mul_d(bi, pi.hi), dd_mul_d(bi, pi.lo))));
            or_dd ti = dd_add(dd_add(dd_mul_d(br, pi.hi), dd_mul_d(br, pi.lo)), dd_add(dd_mul_d(bi, pr.hi), dd_mul_d(bi, pr.lo)));
            br = tr; bi = ti; E += pE;
        }
        out[4 * q] = br.hi; out[4 * q + 1] = br.lo; out[4 * q + 2] = bi.hi; out[4 * q + 3] = bi.lo;
        exps[q] = E;
    }
}

/* Reference P(z) as the plain sum of monomials a_k z^k (each power by binary
 * powering) over an explicit list of nonzero terms (sparse polynomials). */
void or_direct_sum(const int64_t* idx, const double* vals, int64_t nnz, int is_complex,
                   const double* pts, int64_t npts, double* out, int64_t* exps)
{
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < npts; ++q) {
        or_x z = or_point(pts, is_complex, q);
        or_x s = { 0, 0, 0 };
        for (int64_t t = 0; t < nnz; ++t) {
            or_x c = or_coef(vals, is_complex, t);
            if (idx[t] == 0) s = or_add(s, c);
            else if (!(z.re == 0 && z.im == 0)) s = or_add(s, or_mul(c, or_pow(z, idx[t])));
        }
        or_store(s, out + 4 * q, exps + q);
    }
}

/* S(z) = sum_k |a_k| |z|^k (the tolerance scale of the north star), by Horner
 * on the absolute values (no cancellation).  out: mantissa (double), exps. */
void or_abs_sum(const double* a, int64_t kmin, int64_t kmax, int is_complex,
                const double* pts, int64_t npts, double* out, int64_t* exps)
{
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < npts; ++q) {
        double re = is_complex ? pts[2 * q] : pts[q];
        double im = is_complex ? pts[2 * q + 1] : 0.0;
        or_x z = { sqrtq((f128)re * re + (f128)im * im), 0, 0 };
        z = or_norm(z);
        or_x b = { 0, 0, 0 };
        for (int64_t k = kmax; k >= kmin; --k) {
            double ar = is_complex ? a[2 * k] : a[k];
            double ai = is_complex ? a[2 * k + 1] : 0.0;
            or_x c = { sqrtq((f128)ar * ar + (f128)ai * ai), 0, 0 };
            c = or_norm(c);
            b = or_add(or_mul(b, z), c);
        }
        if (z.re != 0) b = or_mul(b, or_pow(z, kmin));
        else if (kmin != 0) b.re = 0;
        b = or_norm(b);
        out[q] = (double)b.re;
        exps[q] = b.e;
    }
}

/* log2 M(z), M = max_k |a_k z^k| (eq:def_prec_loss), from precomputed log2|a_k|
 * (-inf for zeros) and the binary128 log2|z|.  Used by the T3 self-check. */
void or_log2_maxterm(const double* log2abs, int64_t n, const double* pts, int64_t npts,
                     int is_complex, double* out)
{
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < npts; ++q) {
        double re = is_complex ? pts[2 * q] : pts[q];
        double im = is_complex ? pts[2 * q + 1] : 0.0;
        f128 lz = log2q((f128)re * re + (f128)im * im) / 2;
        f128 best = -INFINITY;
        for (int64_t k = 0; k < n; ++k) {
            if (isinf(log2abs[k])) continue;
            f128 v = (f128)log2abs[k] + lz * (f128)k;
            if (v > best) best = v;
        }
        out[q] = (double)best;
    }
}

void or_log2abs(const double* a, int64_t n, int is_complex, double* out)
{
    for (int64_t k = 0; k < n; ++k) {
        double re = is_complex ? a[2 * k] : a[k];
        double im = is_complex ? a[2 * k + 1] : 0.0;
        if (re == 0.0 && im == 0.0) { out[k] = -INFINITY; continue; }
        out[k] = (double)(log2q((f128)re * re + (f128)im * im) / 2);
    }
}
