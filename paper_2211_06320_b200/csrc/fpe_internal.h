// fpe_internal.h -- layout of the preconditioned polynomial and kernel parameters.
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>
#include <vector_types.h>
#include <cuda_runtime.h>
#include "../../include/fpe.h"

namespace fpe {

constexpr uint64_t kMagic = 0x4650453230304232ull;  // "FPE200B2"
constexpr uint32_t kVersion = 2;
constexpr int kCoefPad = 256;   // dense coefficient arrays are padded to whole evaluator chunks

// First 256 bytes of the flat device buffer (also kept on the host in the handle).
// Sections follow, each 256-byte aligned:
//   hull   int2[n_hull]                (k, s(a_k)) of the canonical cover vertices
//   coef   dense : CT[d_eff + 1]        a_k 2^-shift for k in [k_min, k_max], 0 where k not in G_p
//                                       (zero-padded to a multiple of kCoefPad)
//          sparse: CT[n_good]           a_k 2^-shift for the good indices
//   prefix int32[d_eff + 2]             dense & not all_good: #G_p below k (k - k_min)
//   sidx   int32[n_good]                sparse: the good indices, increasing
struct Header {
  uint64_t magic;
  uint32_t version;
  int32_t dtype;        // fpe_dtype of the stored coefficients
  int64_t n_coeffs, k_min, k_max, n_hull, n_good;
  int32_t p, drop, shift, sparse, all_good, wide;   // wide: scales beyond one common shift (raw a_k, shift 0)
  uint64_t off_hull, off_coef, off_prefix, off_sidx, bytes;
  uint8_t reserved[136];
};
static_assert(sizeof(Header) == 256, "header must be 256 bytes");

// Counters of one fpe_evaluate call, in the first kWsHeader bytes of its workspace (zeroed by the call on
// its stream; fpe_workspace_stats / fpe_last_stats read them).
constexpr size_t kWsHeader = 256;
enum : int {
  kStatHard = 0,          // lambdas within 2^-80 of an fp64 rounding boundary (Ziv test; counted when computed)
  kStatMmaItems = 1,      // (group, piece) tensor-core items planned
  kStatMmaInWarp = 2,     // ... of which the DMMA scratch could not hold: run in-warp by the vector evaluator
  kStatPieceItems = 3,    // parallel vector pieces of long windows
  kStatPieceSerial = 4,   // long-window groups evaluated serially (piece scratch full)
  kStatSliceMismatch = 5, // bucket slices a classify CTA did not fill exactly as k_bucket_hist counted (expected 0)
  kStatWindowEscape = 6,  // points whose window is not inside their group's planned union (expected 0)
  kStatCount = 7
};

// Kernel-side view of a handle.
struct PolyDev {
  const int2* hull;
  const void* coef;
  const int32_t* prefix;
  const int32_t* sidx;
  long long k_min, k_max, n_good;
  int nv, drop, shift, sparse, all_good, cdt;
  int wide;     // evaluate with per-step exponent tracking (k_eval_wide): shift = 0, raw coefficients
  int dbl_ok;   // band predicates exact in doubles: d_eff < 2^26 and (2 H + D) d_eff < 2^52
};

}  // namespace fpe

struct fpe_poly_s {
  fpe::Header hdr;
  int device = 0;
  void* dbuf = nullptr;                 // flat device buffer (owned)
  std::vector<int32_t> hk, hh;          // host copy of the cover
  // per-stage timing (fpe_set_profiling)
  bool profiling = false;
  void* prof_events[16] = {};
  const char* stage_names[16] = {};
  int n_stages = 0;
  void* prof_stream = nullptr;
  // staging for fpe_evaluate_host (grown on demand, owned)
  void* st_dev = nullptr; size_t st_bytes = 0;
  static constexpr int kHostSlots = 8;   // staging slots available to fpe_evaluate_host
  void* st_streams[3 + kHostSlots] = {};   // H2D copies, D2H copies, one kernel stream per staging slot, D2H #2
  void* st_events[4 * kHostSlots] = {};    // per staging slot: h2d done, eval done, d2h done, d2h #2 done
  fpe::PolyDev view() const;
};

namespace fpe {
void set_error(const char* fmt, ...);

// Per-stage CUDA-event marks on the launching stream (fpe_set_profiling).
struct Stage {
  fpe_poly h;
  void* stream;
  Stage(fpe_poly h_, void* s_);
  void mark(const char* name);
};
fpe_status precondition_host(const void* coeffs_host, int64_t n, fpe_dtype dt, int32_t p_bits,
                             int32_t drop_override, std::vector<uint8_t>& flat, Header& hdr,
                             std::vector<int32_t>& hk, std::vector<int32_t>& hh);
// Stage 1 of the device preconditioner (independent of p): scales and the canonical cover, kept on the
// device (precondition_gpu.cu); stage 2 finishes G_p and the flat buffer for a given p.
struct CoverDev {
  const void* coeffs = nullptr;   // device coefficients (borrowed or == owned)
  void* owned = nullptr;          // device copy owned by an fpe_cover
  void* scales = nullptr;         // int32[n]
  void* hull = nullptr;           // int2[nv]
  int64_t n = 0, k_min = 0, k_max = 0, nv = 0;
  fpe_dtype dt = FPE_R64;
  int device = 0;
  std::vector<int32_t> hk, hh;
  void release();
};
fpe_status cover_build(const void* coeffs, int64_t n, fpe_dtype dt, cudaStream_t s, CoverDev& cv);
fpe_status cover_finish(const CoverDev& cv, int32_t p_bits, int32_t drop_override, cudaStream_t s, void** dbuf,
                        Header& hdr, std::vector<int32_t>& hk, std::vector<int32_t>& hh);
// The same on the device (precondition_gpu.cu): coeffs is a device pointer; *dbuf receives the flat
// buffer (cudaMalloc'd, byte-identical to precondition_host's), hdr / hk / hh its host-side metadata.
fpe_status precondition_device(const void* coeffs, int64_t n, fpe_dtype dt, int32_t p_bits, int32_t drop_override,
                               cudaStream_t s, void** dbuf, Header& hdr, std::vector<int32_t>& hk,
                               std::vector<int32_t>& hh);
}  // namespace fpe

struct fpe_cover_s {
  fpe::CoverDev cv;
};
