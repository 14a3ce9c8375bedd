// internal.h -- plan object and shared host helpers of libspamm.so (not part of the ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/spamm.h"

namespace spamm {

constexpr int kTile = 32;   // LoNum; pinned by Table 1

// precisions whose A, B are float (FP32 norms, FP32 skip-map grouping)
inline bool f32_inputs(spamm_precision p) { return p == SPAMM_FP32 || p == SPAMM_FP32X3; }

// Scheduling macro-tile shapes (in C tiles).  FP32 SIMT: 128x128 (one warp per C tile);
// tensor path: 128x256 (one UMMA M=128 covers 4 tile rows, N up to 256 = 8 tile cols).
constexpr int kMacroI = 4;
constexpr int kMacroI_dual = 8;   // default tensor path: 256 x 256 macro-tiles (8 x 8 C tiles), multiply_dual.cu
constexpr int kMacroJ_simt = 4;
constexpr int kMacroJ_umma = 8;

struct Plan {
  int64_t M = 0, N = 0, K = 0;
  int32_t tile = kTile;
  double tau = 0.0;
  double alpha = 1.0, beta = 0.0;   // C = alpha * SpAMM(A, B) + beta * C (spamm_set_scalars)
  // chained SpAMM (spamm_multiply_chain): per-call outputs of the multiply epilogue
  double* nC = nullptr;             // [BM][BN] tile norms of the last chained C (allocated on first use)
  bool out_norms = false;
  void* out_low = nullptr;          // rounded copy of C in the input precision, or nullptr
  int64_t out_ldl = 0;
  bool nc_ready = false;
  spamm_precision prec = SPAMM_FP32;
  uint32_t flags = 0;
  int64_t BM = 0, BK = 0, BN = 0;
  int MI = kMacroI, MJ = kMacroJ_simt;
  int64_t GM = 0, GN = 0;
  int num_sms = 148;
  int device = 0;

  // device workspace
  double* nA = nullptr;      // [BM][BK]
  double* nBt = nullptr;     // [BN][BK]  (nB transposed)
  int64_t* V = nullptr;      // [BM*BN + 1] leaf counts, then (after scan) unused
  int64_t* U = nullptr;      // [GM*GN + 1] macro union counts
  int64_t* leaf_start = nullptr; // [BM*BN] start of each C tile's k list in leaf_k (macro-major)
  int64_t* L = nullptr;          // [GM*GN + 1] kept pairs per macro-tile
  int64_t* leaf_base = nullptr;  // [GM*GN + 1] exclusive scan of L
  int64_t* macro_ptr = nullptr;  // [GM*GN + 1]
  int64_t* row_work = nullptr;   // [BM + BK + 2]: row work, then the U histogram (one memset)
  unsigned int* ticket = nullptr; // CTA-completion ticket of the count kernel (self-resetting)
  unsigned int* sched = nullptr;  // dynamic tile counter of the multiply kernels (reset per launch)
  uint16_t* leaf_k = nullptr;    // [leaf_cap]
  uint2* macro_ent = nullptr;    // [macro_cap] (k, mask)
  uint4* macro_run = nullptr;    // [macro_cap] tensor path: k|nruns|cols, packed MMA runs
  int32_t* order = nullptr;      // [GM*GN] LPT schedule
  int64_t* hist = nullptr;       // = row_work + BM: [BK+2] histogram of macro union counts
  int64_t* totals = nullptr;     // = hist + BK + 2: [0] kept pairs, [1] macro entries
  int64_t* mstart = nullptr;     // [GM*GN] start of each macro-tile's entries (t*BK or macro_ptr)
  int umma_variant = 5;          // tensor-path kernel: 0-2, 4 multiply_umma.cu, 5 multiply_dual.cu
  unsigned int* split_cnt = nullptr;   // dual multiply k-split handshake counters (self-resetting)
  float* split_scr = nullptr;          // dual multiply k-split partials
  // workspace zeroing folded into the previous kernel of a spamm_run / AUTO call (saves a memset
  // node per stage): the norm kernel zeroes row_work/hist/totals for the skip map, the skip map's
  // last CTA zeroes the multiply's claim counters
  bool zero_ws_next = false, ws_zeroed = false, sched_zeroed = false;
  bool dual = false;             // the two-issuer 256 x 256 path (variant 5, multiply_dual.cu): MI = 8, two 4 x 8 run entries per k-step
  int64_t* Uw = nullptr;         // [GM*GN] tensor-path entries per macro-tile (pairs merged) or = U
  // stream-K workspace of the tensor multiply (allocated on first use)
  float* sk_scratch = nullptr;       // [2 * grid][128 * 256] FP32 partial tiles
  unsigned int* sk_ticket = nullptr; // [GM*GN] contributors arrived per LPT position (self-resetting)
  int64_t* sk_wpre = nullptr;        // [GM*GN + 1] exclusive prefix of Uw over the LPT order
  int64_t sk_cap_tiles = 0, sk_cap_slots = 0;
  // SPAMM_FP32X3: bfloat16 split planes a = a0 + a1 + a2, written by the norm stage:
  // A planes [3][M][ldpa], then B planes [3][K][ldpb] (unused when B is A)
  uint16_t* planes = nullptr;
  int64_t ldpa = 0, ldpb = 0;
  bool b_is_a = false;           // the last spamm_norms saw B == A (planes of A serve both)
  bool fixed_regions = false;    // lists stored in worst-case fixed regions (single-pass skip map)
  int64_t* bucket_pos = nullptr; // [BK+2] descending bucket starts (consumed by emit)
  void* cub_tmp = nullptr;
  size_t cub_tmp_bytes = 0;
  int64_t leaf_cap = 0, macro_cap = 0;
  int64_t* d_totals = nullptr;   // [2] kept, macro entries (device, written by scans)
  int64_t* h_totals = nullptr;   // pinned mirror

  // state
  bool norms_ready = false;
  bool skipmap_ready = false;
  bool leaf_ready = false;       // per-C-tile lists (V, leaf_start, leaf_k) materialised
  int64_t row_begin_macro = 0, row_end_macro = 0;   // macro-row range the skip map / multiply covers
  std::vector<int64_t> last_partition;
  cudaStream_t last_stream = nullptr;

  // timing
  cudaEvent_t ev[6] = {};
  bool ev_norms = false, ev_skip = false, ev_mul = false;
};

// error plumbing ------------------------------------------------------------
void set_error(const std::string& msg);
spamm_status fail(spamm_status s, const std::string& msg);
spamm_status cuda_fail(cudaError_t e, const char* where);

#define SPAMM_CUDA_TRY(expr)                                      \
  do {                                                            \
    cudaError_t _e = (expr);                                      \
    if (_e != cudaSuccess) return ::spamm::cuda_fail(_e, #expr);  \
  } while (0)

#define SPAMM_TRY(expr)                     \
  do {                                      \
    spamm_status _s = (expr);               \
    if (_s != SPAMM_OK) return _s;          \
  } while (0)

void count_launch(int n = 1);

// stage launchers (implemented in the .cu files) -----------------------------
// norms of A's tile rows [ar0, ar1) and B's tile columns [bj0, bj1) in one launch
spamm_status launch_norms2(const Plan& p, const void* A, int64_t lda, int64_t ar0, int64_t ar1, const void* B,
                           int64_t ldb, int64_t bj0, int64_t bj1, cudaStream_t s);
spamm_status launch_skipmap_count(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s);
spamm_status launch_skipmap_emit(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s);
spamm_status launch_skipmap_fused(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s);
spamm_status launch_multiply_simt(Plan& p, const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                                  int64_t ldc, cudaStream_t s);
spamm_status launch_leaf_expand(Plan& p, cudaStream_t s);   // per-C-tile lists from macro lists
int umma_variant_from_env();       // SPAMM_UMMA_VARIANT: 0 (default) 2 CTAs/SM 32-deep, 1 = 2 CTAs/SM 64-deep, 2 = 1 CTA/SM 64-deep split issuers, 4 = 1 CTA/SM 32-deep split issuers, 5 (default) = 256 x 256 tiles with two issuers (3, CTA pairs, was removed)
bool umma_variant_wide(int v);     // does the variant consume merged 64-deep k-steps?
spamm_status launch_multiply_dual(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C,
                                  int64_t ldc, cudaStream_t s);
spamm_status launch_multiply_x3(Plan& p, float* C, int64_t ldc, cudaStream_t s);   // SPAMM_FP32X3
spamm_status launch_multiply_umma(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C,
                                  int64_t ldc, cudaStream_t s);

size_t skipmap_cub_bytes(int64_t nleaf, int64_t nmac);
spamm_status launch_transpose_f64(const double* in, int64_t rows, int64_t cols, double* out, cudaStream_t s);

// 3-D map: dims {inner, mid, outer} with byte strides {mid_stride, outer_stride}.
spamm_status encode_tmap_3d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner,
                            uint64_t mid, uint64_t outer, uint64_t mid_stride_bytes, uint64_t outer_stride_bytes,
                            uint32_t box0, uint32_t box1, uint32_t box2, CUtensorMapSwizzle swz);

// TMA tensor-map encoder from the driver (resolved once via cudaGetDriverEntryPoint).
spamm_status encode_tmap_2d(CUtensorMap* map, CUtensorMapDataType dt, uint32_t esize, const void* base,
                            uint64_t inner, uint64_t outer, uint64_t ld_elems, uint32_t box_inner,
                            uint32_t box_outer, CUtensorMapSwizzle swz);

}  // namespace spamm
