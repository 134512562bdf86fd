/*
 * fpe.h -- C ABI of the B200 Fast Polynomial Evaluator (libfpe.so).
 *
 * The calls follow the problem statement of Algorithm FPE_p:
 *   preconditioning  "Data: the list of coefficients a_0..a_d and the precision p"
 *                    (scales, concave cover, good indices G_p)
 *   evaluation       "Data: pre-conditioned P at precision p; finite subset Z of C*"
 *                    -> Q_lambda(z) for every z in Z
 * plus the full Horner scheme as the context baseline.
 *
 * Conventions
 *  - All entry points are extern "C", return fpe_status unless noted, and never
 *    throw.  On failure fpe_last_error_detail() (thread-local) says why.
 *  - Pointers are plain host or device pointers; stream arguments are
 *    cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Complex data are interleaved (re, im) pairs of the dtype's real type.
 *  - Results are returned in extended range: value = mantissa * 2^exp with
 *    max(|re|,|im|) of the mantissa in [1/2, 1) (or all zero with exp = 0),
 *    because z^d overflows any hardware float.
 *  - Results are a pure function of (handle, z): bitwise independent of the
 *    batch, its order, the sharding across GPUs and the run.  (Whole 16384-coefficient
 *    pieces of long windows run on the FP64 tensor cores; when a batch asks for more of
 *    them than its workspace's scratch holds, the excess runs the same tensor-core
 *    arithmetic inside the vector evaluator -- same bits, counted by fpe_workspace_stats.)
 *  - The handle is immutable: concurrent fpe_evaluate / fpe_horner calls on one handle
 *    are safe with distinct workspaces (except in profiling mode, fpe_set_profiling, and
 *    fpe_evaluate_host, which use per-handle state).
 */
#ifndef FPE_H_
#define FPE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FPE_OK = 0,
    FPE_ERR_INVALID_ARG = 1,      /* bad pointer / size / dtype; nothing enqueued            */
    FPE_ERR_ZERO_POLY = 2,        /* all coefficients are zero                               */
    FPE_ERR_NONFINITE_COEFF = 3,  /* a NaN or inf coefficient                                 */
    FPE_ERR_UNSUPPORTED = 4,      /* e.g. coefficient dynamic range beyond the fp64/fp32 path */
    FPE_ERR_OOM = 5,              /* device or host allocation failed                         */
    FPE_ERR_CUDA = 6              /* a CUDA runtime error (detail has the CUDA message)       */
} fpe_status;

typedef enum {
    FPE_R64 = 0,  /* double            */
    FPE_C64 = 1,  /* double re, im     */
    FPE_R32 = 2,  /* float             */
    FPE_C32 = 3   /* float re, im      */
} fpe_dtype;

/* Opaque, immutable preconditioned polynomial ("pre-conditioned P at precision p",
 * PAPER.md:1245).  Owns its device buffer until fpe_destroy. */
typedef struct fpe_poly_s* fpe_poly;

typedef struct {
    int64_t d;          /* n_coeffs - 1                                                  */
    int64_t k_min;      /* first nonzero index                                           */
    int64_t k_max;      /* last nonzero index; d_eff = k_max - k_min (R3)      */
    int64_t n_hull;     /* vertices of the canonical concave cover    */
    int64_t n_good;     /* |G_p| (eq:threshold)                      */
    int32_t p;          /* precision in bits (53 for fp64, 24 for fp32 by default)        */
    int32_t drop;       /* D = p + s(d_eff) + 3 unless overridden   */
    int32_t shift;      /* stored coefficients are a_k * 2^-shift (exact)                 */
    int32_t sparse;     /* 1: compact good-index list; 0: dense masked coefficient array  */
    int32_t dtype;      /* fpe_dtype of the coefficients                                   */
    int32_t reserved;
    size_t bytes;       /* size of the flat device buffer                                  */
} fpe_poly_info;

/* Per-point diagnostics of the evaluation phase (lines 5-8 of Algorithm FPE_p). */
typedef struct {
    double  lambda;     /* correctly rounded fp64 log2|z| (eq:defLambda); -inf for z = 0  */
    int32_t region;     /* index of the cover vertex k_lambda (smallest argmax); -1: non-finite z */
    int32_t l;          /* band [l, r] (def:LRN)                       */
    int32_t r;
    int32_t kept;       /* K = #(G_p cap [l, r])                                           */
    int32_t hard;       /* 1 if lambda was within 2^-96 |lambda| of an fp64 rounding boundary */
    int32_t cancel;     /* canceled bits c (eq:def_prec_loss): 0 if |Q| >= M, else
                           s(M) - s(Q), with s(M) estimated from above by ceil(N_lambda), N_lambda =
                           cover(k_lambda) + lambda k_lambda (log2 M lies in [N - 1, N)); the result
                           has about p - c correct bits (Theorem thm:equivAlgo); INT32_MIN when Q = 0
                           or z is non-finite                                                       */
    int32_t trusted;    /* conservative number of correct leading bits of the result (the errors file,
                           PAPER.md:2114-2118): clamp(s(Q) - err_exp, 0, p_w), p_w = 53 / 24 working
                           bits; 0 when Q = 0 or z is non-finite                                     */
    int32_t err_exp;    /* upper bound on the evaluation error: |value 2^exp - P(z)| <= 2^err_exp, with
                           err_exp = ceil(N) + ceil(log2(2K + 256)) + ceil(log2 K) + 1 - p_w: rounding
                           <= (2K + 256) u S over the K kept terms, S <= K 2^N, plus the truncation
                           < 2^(N-p-3); clamped to the int32 range; INT32_MIN
                           when z is non-finite                                                      */
    int32_t pad;
} fpe_diag;

/*
 * fpe_precondition -- lines 2-4 of Algorithm FPE_p.
 *   coeffs        a_0..a_d, n_coeffs = d+1 entries of dtype dt (host or device pointer;
 *                 read during the call only, then copied).
 *   p_bits        precision p; 0 selects 53 (R64/C64) or 24 (R32/C32).
 *   drop_override 0: D = p + s(d_eff) + 3; > 0: D = drop_override (tests only).
 *   device        CUDA device ordinal that will own the handle's buffer.
 *   stream        stream for the host->device upload (the call synchronises it).
 *   out           receives the handle.
 * Errors: INVALID_ARG (NULL pointers, n_coeffs < 1, bad dtype), ZERO_POLY,
 *         NONFINITE_COEFF, UNSUPPORTED (coefficient scales of the good terms span more
 *         than the working format can hold after a common power-of-two shift), OOM, CUDA.
 */
fpe_status fpe_precondition(const void* coeffs, int64_t n_coeffs, fpe_dtype dt,
                            int32_t p_bits, int32_t drop_override, int device,
                            void* stream, fpe_poly* out);

/*
 * fpe_precondition_gpu -- the same preconditioning computed on the device (
 * PAPER.md:1239-1243 with the scales PAPER.md:509-532, the cover PAPER.md:1413-1509 and G_p
 * PAPER.md:1512-1521): per-coefficient scales, per-chunk monotone chains merged level by level into the
 * canonical cover, G_p flags by exact integer tests, a scan for the prefix counts / compact list.
 * The flat buffer is byte-identical to fpe_precondition's.
 *   coeffs        device pointer on `device` to a_0..a_d (n_coeffs = d+1 entries of dtype dt); read
 *                 during the call only.
 *   other arguments as fpe_precondition; the call synchronises `stream`.  Temporary device memory:
 *   ~13 bytes per coefficient.
 * Errors: as fpe_precondition; INVALID_ARG also when coeffs is not device memory of `device`.
 */
fpe_status fpe_precondition_gpu(const void* coeffs, int64_t n_coeffs, fpe_dtype dt,
                                int32_t p_bits, int32_t drop_override, int device,
                                void* stream, fpe_poly* out);

/*
 * Partial preprocessing (remark rem:partialpreproc): lines 2-3 of FPE_p (the
 * scales and the concave cover) do not depend on p, so they can be computed once and G_p (line 4)
 * finished in O(d) for each precision p later.
 * fpe_cover_build   -- scales and canonical cover on the device from device coefficients (copied:
 *                      the caller's array is read during the call only); synchronises `stream`.
 *                      Errors: INVALID_ARG (bad arguments or coeffs not device memory of `device`),
 *                      ZERO_POLY, NONFINITE_COEFF, OOM, CUDA.
 * fpe_cover_finish  -- a handle for precision p_bits (0: 53 / 24 by dtype) and D = drop_override
 *                      (0: p + s(d_eff) + 3), byte-identical to fpe_precondition's; the cover object
 *                      stays valid.  Errors: INVALID_ARG, UNSUPPORTED, OOM, CUDA.
 * fpe_cover_destroy -- frees the cover (NULL is a no-op).
 */
typedef struct fpe_cover_s* fpe_cover;
fpe_status fpe_cover_build(const void* coeffs, int64_t n_coeffs, fpe_dtype dt, int device, void* stream,
                           fpe_cover* out);
fpe_status fpe_cover_finish(fpe_cover c, int32_t p_bits, int32_t drop_override, void* stream, fpe_poly* out);
void fpe_cover_destroy(fpe_cover c);

/*
 * fpe_precondition_host -- the same preconditioning, entirely on the host (no CUDA call):
 * writes the flat buffer that fpe_poly_device_buffer would hold into the host array buf.
 * With buf == NULL or cap too small, only *bytes (the required size) is set and
 * FPE_ERR_INVALID_ARG is returned.  Used to prepare / ship a handle without a GPU.
 */
fpe_status fpe_precondition_host(const void* coeffs_host, int64_t n_coeffs, fpe_dtype dt,
                                 int32_t p_bits, int32_t drop_override, void* buf, size_t cap,
                                 size_t* bytes);

fpe_status fpe_poly_get_info(fpe_poly h, fpe_poly_info* out);

/*
 * fpe_analyse -- the "-analyse" task: the intervals of lambda = log2|z| on which
 * the evaluation strategy (the reduced polynomial Q_lambda: its region i* and window [l, r],
 * PAPER.md:1249-1253) is constant, inside [lam_lo, lam_hi].  Host computation on the handle's cover
 * and G_p: breakpoints are the cover slopes -sigma_i (where i* changes) and, per region, the values
 * lambda = -J/I at which an index k enters or leaves the band (the exact predicates of the evaluator,
 * PAPER.md:1543-1559); each interval's (i*, l, r) is classified exactly at its midpoint and equal
 * neighbours are merged.  Breakpoints are reported rounded to double.  Intended for low degrees
 * (UNSUPPORTED when d_eff * |cover| > 2^26).
 *   out    host array of capacity cap (may be NULL with cap = 0 to query the count);
 *   *n     receives the number of intervals (INVALID_ARG if cap < *n and out != NULL).
 */
typedef struct {
    double lam_lo, lam_hi;   /* the interval [lam_lo, lam_hi] of log2|z|                              */
    int32_t region, l, r;    /* i* (k_lambda vertex index) and the window [l, r] (absolute indices)   */
    int32_t kept;            /* |G_p intersected with [l, r]|                                         */
} fpe_interval;
fpe_status fpe_analyse(fpe_poly h, double lam_lo, double lam_hi, fpe_interval* out, int64_t cap, int64_t* n);

/* Canonical cover vertices (hk[i], hh[i] = s(a_hk[i])) into host arrays of capacity cap;
 * *n receives the vertex count (INVALID_ARG if cap is too small). */
fpe_status fpe_poly_get_hull(fpe_poly h, int32_t* hk, int32_t* hh, int64_t cap, int64_t* n);

/* The handle's flat device buffer (immutable; e.g. for ncclBroadcast to other ranks). */
fpe_status fpe_poly_device_buffer(fpe_poly h, const void** dptr, size_t* bytes);

/* Copy the flat buffer (h's fpe_poly_info.bytes bytes) to dst, a host or device pointer
 * of capacity cap (synchronous on `stream`). */
fpe_status fpe_poly_export(fpe_poly h, void* dst, size_t cap, void* stream);

/* A new handle on `device` from a flat buffer produced by fpe_poly_device_buffer,
 * fpe_poly_export or fpe_precondition_host (possibly received from another rank); ptr may
 * be a host or a device pointer.  The buffer is validated (magic, version, size) and copied.
 * INVALID_ARG if it is not an fpe buffer. */
fpe_status fpe_poly_from_device_buffer(const void* ptr, size_t bytes, int device,
                                       void* stream, fpe_poly* out);

/* Bytes of device workspace fpe_evaluate / fpe_horner need for n_points points (the first 256 bytes
 * hold the call's counters, fpe_workspace_stats). */
fpe_status fpe_eval_workspace_size(fpe_poly h, int64_t n_points, size_t* bytes);

/*
 * fpe_evaluate -- lines 5-9 of Algorithm FPE_p for every point.
 *   points      n_points device values of dtype pt_dt.  pt_dt must have the coefficient
 *               dtype's precision (64 or 32 bit); a real polynomial at real points uses
 *               the real path, every other combination is evaluated in complex.
 *   values_out  device, n_points values: complex (interleaved) unless both the polynomial
 *               and the points are real; precision as pt_dt.
 *   exps_out    device int64[n_points] binary exponents, or NULL: then values are returned
 *               ldexp'd to plain floats (which may overflow to inf or underflow to 0).
 *   diag_out    device fpe_diag[n_points] or NULL.
 *   workspace   device scratch of at least fpe_eval_workspace_size bytes.
 * Per-point cases: z = 0 gives a_0 (0 if a_0 = 0) with region 0, l = r = k_min;
 *   a non-finite z gives NaN with region -1.  Asynchronous on `stream`.
 * Errors: INVALID_ARG (no work enqueued), CUDA.
 */
fpe_status fpe_evaluate(fpe_poly h, const void* points, fpe_dtype pt_dt, int64_t n_points,
                        void* values_out, int64_t* exps_out, fpe_diag* diag_out,
                        void* workspace, size_t ws_bytes, void* stream);

/*
 * fpe_evaluate_host -- the same as fpe_evaluate for HOST buffers (points in, values and
 * exponents out), staging through device memory owned by the handle; host<->device copies
 * are pipelined with the kernels in chunks.  Pinned host memory gives full copy bandwidth.
 * Synchronous: returns when the host outputs are written.  Not thread-safe per handle.
 * `stream` is unused: the call runs on the handle's own streams (one copy stream each way, one
 * kernel stream per staging slot) so that consecutive chunks overlap.
 */
fpe_status fpe_evaluate_host(fpe_poly h, const void* points_host, fpe_dtype pt_dt,
                             int64_t n_points, void* values_host, int64_t* exps_host,
                             void* stream);

/*
 * fpe_horner -- the full Horner scheme over all coefficients a_k_min..a_k_max with
 * in-loop exponent rescaling, the context baseline of the benchmark.
 * Arguments as fpe_evaluate (no diagnostics).
 */
fpe_status fpe_horner(fpe_poly h, const void* points, fpe_dtype pt_dt, int64_t n_points,
                      void* values_out, int64_t* exps_out, void* workspace, size_t ws_bytes,
                      void* stream);

/*
 * fpe_precondition_derivative -- preconditions P' ("the preconditioning of P and P'
 * can be done simultaneously"; this implementation takes the paper's alternative, a separate
 * preprocessing of P'): the coefficients b_j = (j+1) a_{j+1}, j = 0..d-1, are formed on the host in the
 * working format (one rounding each) and preconditioned as by fpe_precondition (same arguments; coeffs
 * are P's d+1 coefficients).  ZERO_POLY if P is constant.
 */
fpe_status fpe_precondition_derivative(const void* coeffs, int64_t n_coeffs, fpe_dtype dt, int32_t p_bits,
                                       int32_t drop_override, int device, void* stream, fpe_poly* out);

/* Bytes of device workspace fpe_newton_step needs for n_points points. */
fpe_status fpe_newton_workspace_size(fpe_poly P, fpe_poly dP, int64_t n_points, size_t* bytes);

/*
 * fpe_newton_step -- one Newton step N_P(z) = z - P(z)/P'(z) (eq:newton) for every
 * point: Q1 and Q2, the FPE values of P and P' (fpe_evaluate), stay in extended range (mantissa, int64
 * exponent), so the quotient m1/m2 2^(e1-e2) is formed without overflow or loss -- the paper's
 * "cancelation of valuation" m = min(l, l'): e.g. z^64 + 1 at z = 10 in FP32, where P and P'
 * overflow, gives the increment 0.15625.
 *   P, dP       handles of P and of P' (fpe_precondition_derivative), same device and precision.
 *   points      device, n_points points of dtype pt_dt (as fpe_evaluate).
 *   points_out  device, n_points values N_P(z) in the output type of fpe_evaluate (complex unless all real).
 *   incr_out    device, n_points increments P(z)/P'(z) in the same type, or NULL.
 *   workspace   device, at least fpe_newton_workspace_size bytes.
 * Per point: P'(z) = 0 gives inf/NaN; non-finite z gives NaN.  Errors: INVALID_ARG, CUDA.
 */
fpe_status fpe_newton_step(fpe_poly P, fpe_poly dP, const void* points, fpe_dtype pt_dt, int64_t n_points,
                           void* points_out, void* incr_out, void* workspace, size_t ws_bytes, void* stream);

/*
 * Per-stage timing (measurement support for bench.py).  With fpe_set_profiling(h, 1) every
 * later fpe_evaluate / fpe_horner on h records CUDA events on its stream around each kernel (the
 * events and stage names live in the handle: no concurrent calls on a profiling handle);
 * fpe_last_stage_ms (synchronising the stream of that call) returns the stage durations in
 * launch order (up to cap) and *n, and fpe_stage_name(h, i) names stage i.
 */
fpe_status fpe_set_profiling(fpe_poly h, int enable);
fpe_status fpe_last_stage_ms(fpe_poly h, float* ms, int cap, int* n);
const char* fpe_stage_name(fpe_poly h, int i);

/*
 * fpe_workspace_stats -- the counters the last fpe_evaluate with this workspace wrote into its first 256
 * bytes (the call zeroes them on its stream first).  Synchronises `stream` (the call's stream), then
 * copies min(cap, *n) counters into the host array stats; *n receives the number of counters (7):
 *   [0] lambdas within 2^-80 of an fp64 rounding boundary (Ziv test of the correctly rounded log2|z|;
 *       counted for the points whose lambda was computed: all with diagnostics, the undecided ones without)
 *   [1] (group, piece) tensor-core items planned (whole 16384-coefficient pieces, complex fp64)
 *   [2] ... of which did not fit the workspace's DMMA scratch and ran in-warp (same arithmetic)
 *   [3] parallel vector pieces of long windows
 *   [4] long-window groups evaluated serially (piece scratch full; same arithmetic)
 *   [5] (CTA, bucket) slices the classifier did not fill exactly as the histogram pass counted them --
 *       a self-check of the work bucketing (0 unless the two passes disagree on a point's bucket key)
 *   [6] points whose window [l, r] is not inside their group's planned union window -- a self-check of the
 *       per-bucket window bounds the plan uses (0 unless they fail to contain a point's window)
 * Errors: INVALID_ARG, CUDA.
 */
fpe_status fpe_workspace_stats(const void* workspace, void* stream, int64_t* stats, int cap, int* n);

/* Counters of the calling thread's last fpe_evaluate / fpe_evaluate_host / fpe_horner / fpe_newton_step
 * (thread-local record; the workspace that call used must still be allocated): stats4[0] = hard-to-round
 * lambdas, [1] = library kernel launches, [2] = tensor-core items, [3] = of which run in-warp.  Synchronises
 * that call's stream.  `h` is only checked for NULL. */
fpe_status fpe_last_stats(fpe_poly h, int64_t* stats4);

void fpe_destroy(fpe_poly h);
const char* fpe_status_string(fpe_status s);
const char* fpe_last_error_detail(void);

#ifdef __cplusplus
}
#endif
#endif /* FPE_H_ */
