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

// Scheduling macro-tile shapes (in C tiles).  FP32 SIMT: 128x128 (one warp per C tile);
// tensor path: 128x256 (one UMMA M=128 covers 4 tile rows, N up to 256 = 8 tile cols).
constexpr int kMacroI = 4;
constexpr int kMacroJ_simt = 4;
constexpr int kMacroJ_umma = 8;

struct Plan {
  int64_t M = 0, N = 0, K = 0;
  int32_t tile = kTile;
  double tau = 0.0;
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
  int64_t* leaf_ptr = nullptr;   // [BM*BN + 1]
  int64_t* macro_ptr = nullptr;  // [GM*GN + 1]
  int64_t* row_work = nullptr;   // [BM]
  uint16_t* leaf_k = nullptr;    // [leaf_cap]
  uint2* macro_ent = nullptr;    // [macro_cap] (k, mask)
  int32_t* order = nullptr;      // [GM*GN] LPT schedule
  int32_t* order_tmp = nullptr;  // [GM*GN]
  int64_t* keys_tmp = nullptr;   // [GM*GN]
  void* cub_tmp = nullptr;
  size_t cub_tmp_bytes = 0;
  int64_t leaf_cap = 0, macro_cap = 0;
  int64_t* d_totals = nullptr;   // [2] kept, macro entries (device, written by scans)
  int64_t* h_totals = nullptr;   // pinned mirror

  // state
  bool norms_ready = false;
  bool skipmap_ready = false;
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
spamm_status launch_norms(const Plan& p, const void* X, int64_t rows, int64_t cols, int64_t ld,
                          double* out, int64_t out_rs, int64_t out_cs, int64_t row_tile_begin,
                          int64_t row_tile_end, cudaStream_t s);
spamm_status launch_skipmap_count(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s);
spamm_status launch_skipmap_emit(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s);
spamm_status launch_multiply_simt(Plan& p, const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                                  int64_t ldc, cudaStream_t s);
spamm_status launch_multiply_umma(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C,
                                  int64_t ldc, cudaStream_t s);

size_t skipmap_cub_bytes(int64_t nleaf, int64_t nmac);

// TMA tensor-map encoder from the driver (resolved once via cudaGetDriverEntryPoint).
spamm_status encode_tmap_2d(CUtensorMap* map, CUtensorMapDataType dt, uint32_t esize, const void* base,
                            uint64_t inner, uint64_t outer, uint64_t ld_elems, uint32_t box_inner,
                            uint32_t box_outer, CUtensorMapSwizzle swz);

}  // namespace spamm
