// internal.h -- plan object and shared host helpers of libspamm.so (not part of the ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/spamm.h"

namespace spamm {

constexpr int kTile = 32;   // LoNum; pinned by Table 1

// precisions whose A, B are float (FP32 norms, FP32 skip-map grouping)
inline bool f32_inputs(spamm_precision p) { return p == SPAMM_FP32 || p == SPAMM_FP32X3; }

// Scheduling macro-tile shapes (in C tiles).  FP32 paths (SIMT, FP32X3): 128 x 128 (4 x 4 C
// tiles); BF16/FP16 tensor path: 256 x 256 (8 x 8 C tiles, multiply_dual.cu).
constexpr int kMacroF32 = 4;
constexpr int kMacroTC = 8;
constexpr int kChunk = 32;   // k-tiles per norm-pyramid chunk (one warp of the skip map)

// Device-side range block (Plan::d_range, int64[kRangeWords]): the macro rows the skip map and
// the multiply cover, written by the host for single-GPU calls or by the partition kernel of
// the multi-GPU path (so no host synchronisation is needed between partition and multiply).
//   [0] gi0, [1] gi1     macro rows [gi0, gi1) of this call's skip map and multiply
//   [2] ex0, [3] ex1     macro rows whose skip map is already built (skipped by the skip map)
//   [4] nranks, [5] rank, [6..] the partition cut (nranks + 1 macro-row boundaries)
constexpr int kMaxRanks = 64;
constexpr int kRangeWords = 6 + kMaxRanks + 1;

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
  bool out_low_only = false;        // SPAMM_MUL_LOW_ONLY: C_low is the only output (no FP32 C)
  bool nc_ready = false;
  spamm_precision prec = SPAMM_FP32;
  uint32_t flags = 0;
  int64_t BM = 0, BK = 0, BN = 0;
  int MI = kMacroF32, MJ = kMacroF32;
  int64_t GM = 0, GN = 0;
  int64_t NC = 0;            // k chunks of the norm pyramid: ceil(BK / kChunk)
  int num_sms = 148;
  int device = 0;

  // device workspace
  double* nA = nullptr;      // [BM][BK]
  double* nBt = nullptr;     // [BN][BK]  (nB transposed)
  // norm pyramid (Eq. 1's quadtree idea, one level above the leaves): per macro row
  // I and k chunk c, max / min of nA over the MI rows x kChunk k-tiles; per macro column J the
  // same over nB^T.  pyr = [paMax GM*NC][paMin GM*NC][pbMax GN*NC][pbMin GN*NC]
  double* pyr = nullptr;
  int64_t* V = nullptr;      // [BM*BN] per-C-tile list lengths (leaf view, on request)
  int64_t* U = nullptr;      // [GM*GN + 1] macro union counts (k-steps with a kept pair)
  int64_t* L = nullptr;      // [GM*GN + 1] kept pairs per macro-tile
  int64_t* leaf_start = nullptr;  // [BM*BN] start of each C tile's k list (leaf view, on request)
  int64_t* row_work = nullptr;    // [ws_words()]: row work, then the claim order's counters (one memset)
  // workspace counters, one zeroed region (the norm kernel zeroes it inside spamm_run):
  //   row_work[BM] | hist[BK+2] | totals[4] | hist_sb[NSB] | ws_cnt[4] (uint32, two int64 words) |
  //   bucket_cnt[NB], NB = max(BK + 2, NSB + 1) | sb_bits[ceil(R*C/64) NSB]
  int64_t* hist = nullptr;        // LPT bucket counts of the claim order (key BK - U)
  int64_t* totals = nullptr;      // [0] kept pairs, [1] macro entries, [2] macro-tiles without kept pairs
  int64_t* hist_sb = nullptr;     // super-block bucket counts of the claim order
  unsigned int* ws_cnt = nullptr; // [0] work-list length, [1] empty-list length, [2], [3] skip-map tile claims
  int64_t* bucket_cnt = nullptr;  // claim-order slots taken per bucket
  unsigned long long* sb_bits = nullptr;   // working macro-tiles per claim-order super-block (bit masks)
  int64_t NSB = 0;                // claim-order super-blocks of macro-tiles (SPAMM_ORD_R x SPAMM_ORD_C)
  int32_t* tile_lists = nullptr;  // [2 * GM*GN]: macro-tiles with kept pairs, then those without
  unsigned int* sched = nullptr;  // dynamic tile counters of the multiply kernels (reset per launch)
  uint16_t* leaf_k = nullptr;     // [BM*BN*BK] per-C-tile k lists (leaf view, on request)
  void* macro_ent = nullptr;      // [GM*GN*BK] (k, mask) entries, 8 B (4 x 4) or 16 B (8 x 8)
  uint4* macro_run = nullptr;     // tensor path: 2 x [GM*GN*BK] pre-decoded MMA runs (one per 128-row half)
  int32_t* order = nullptr;       // [GM*GN] LPT schedule
  int64_t* bucket_pos = nullptr;  // [BK+2] descending bucket starts
  int64_t* mstart = nullptr;      // [GM*GN] start of each macro-tile's entries (= t*BK)
  int64_t* d_range = nullptr;     // [kRangeWords] device-side range block (see above)
  unsigned long long* ts_cnt = nullptr;   // tau search: kept-count scratch
  double* ts_part = nullptr;              // tau search: column-sum scratch
  // SPAMM_FP32X3: bfloat16 split planes a = a0 + a1 + a2, written by the norm stage:
  // A planes [3][M][ldpa], then B planes [3][K][ldpb] (unused when B is A)
  uint16_t* planes = nullptr;
  int64_t ldpa = 0, ldpb = 0;
  void* im2col = nullptr;         // spamm_conv2d_im2col: the K x N im2col matrix (allocated on first use)
  bool b_is_a = false;            // the last spamm_norms saw B == A (planes of A serve both)
  bool x1 = false;                // BF16/FP16 on 128 x 128 macro-tiles (fewer 256 x 256 tiles than SMs)
  // spamm_run / AUTO on a small problem (128 x 128 macro-tiles -- FP32, FP32X3, small BF16/FP16 -- at
  // most one per SM): no skip-map
  // launch, the multiply's producer warps decide their tiles' lists (multiply_x3.cu XFuse)
  bool fused = false;
  bool leaf_alloc = false;

  // workspace zeroing folded into the previous kernel of a spamm_run / AUTO call: the norm kernel
  // zeroes row_work/hist/totals for the skip map, the skip map's last CTA zeroes the multiply's
  // claim counters
  bool zero_ws_next = false, ws_zeroed = false, sched_zeroed = false;

  // state
  bool norms_ready = false;
  bool pyr_ready = false;
  bool skipmap_ready = false;
  bool leaf_ready = false;        // per-C-tile lists (V, leaf_start, leaf_k) materialised
  bool range_on_device = false;   // the last skip map's range was decided on the device (multi-GPU)
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

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel instantiation and DEVICE (the
// attribute is per device; a process may drive several GPUs).  Concurrent first calls may both
// set it, which is harmless.
#define SPAMM_SET_SMEM(kern, bytes, dev)                                                              \
  do {                                                                                                \
    static std::atomic<unsigned long long> _done{0};                                                  \
    const unsigned long long _bit = 1ull << ((dev) & 63);                                             \
    if (!(_done.load(std::memory_order_relaxed) & _bit)) {                                            \
      SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (bytes))); \
      _done.fetch_or(_bit, std::memory_order_relaxed);                                                \
    }                                                                                                 \
  } while (0)

void count_launch(int n = 1);


inline int64_t ws_buckets(const Plan& p) { return p.BK + 2 > p.NSB + 1 ? p.BK + 2 : p.NSB + 1; }
// the many-tile claim order visits super-blocks of SPAMM_ORD_R x SPAMM_ORD_C macro-tiles row-major:
// by default bands of 6 macro rows walked column by column (skipmap.cu; measured at N = 65536,
// DESIGN.md "claim order")
#ifndef SPAMM_ORD_R
#define SPAMM_ORD_R 6
#endif
#ifndef SPAMM_ORD_C
#define SPAMM_ORD_C 1
#endif
inline int64_t ws_words(const Plan& p) {
  return p.BM + p.BK + 2 + 4 + p.NSB + 2 + ws_buckets(p) + (SPAMM_ORD_R * SPAMM_ORD_C + 63) / 64 * p.NSB;
}

// Launch with programmatic dependent launch (PDL, griddepcontrol): the kernel's CTAs may be
// scheduled while its stream predecessor drains.  Every kernel launched this way calls
// pdl_wait() (sm100.cuh) before it touches global memory its predecessors write, and
// pdl_trigger() once its own CTAs run, so a stage's launch latency and prologue (barrier init,
// TMEM allocation, descriptor prefetch) overlap the previous stage's tail.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// stage launchers (implemented in the .cu files) -----------------------------
// norms of A's tile rows [ar0, ar1) and B's tile columns [bj0, bj1) in one launch
spamm_status launch_norms2(Plan& p, const void* A, int64_t lda, int64_t ar0, int64_t ar1, const void* B,
                           int64_t ldb, int64_t bj0, int64_t bj1, cudaStream_t s);
// norm pyramid (max / min per macro row|column and k chunk) from the maps
spamm_status launch_pyramid(Plan& p, cudaStream_t s);
// skip map of macro rows [gi0, gi1) minus [ex0, ex1) (device range block when on_device);
// with order = true the last CTA builds the LPT order and totals over [gi0, gi1)
spamm_status launch_skipmap(Plan& p, int64_t gi0, int64_t gi1, bool on_device, bool order, bool row_work,
                            cudaStream_t s);
// multi-GPU: macro-row cut of the all-reduced row work on the device (spamm_partition_rows' rule)
spamm_status launch_partition(Plan& p, int rank, int nranks, cudaStream_t s);
spamm_status launch_leaf_expand(Plan& p, cudaStream_t s);   // per-C-tile lists from macro lists
spamm_status launch_multiply_simt(Plan& p, const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                                  int64_t ldc, bool fuse, cudaStream_t s);
spamm_status launch_multiply_dual(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C,
                                  int64_t ldc, cudaStream_t s);
// SPAMM_FP32X3; fuse = the multiply decides the skip map itself (Plan::fused, spamm_run)
spamm_status launch_multiply_x3(Plan& p, float* C, int64_t ldc, bool fuse, cudaStream_t s);
// BF16/FP16 plans with 128 x 128 macro-tiles (small problems, Plan::x1)
spamm_status launch_multiply_x1(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                                bool fuse, cudaStream_t s);
spamm_status launch_transpose_f64(const double* in, int64_t rows, int64_t cols, double* out, cudaStream_t s);

// 3-D map: dims {inner, mid, outer} with byte strides {mid_stride, outer_stride}.
spamm_status encode_tmap_3d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner,
                            uint64_t mid, uint64_t outer, uint64_t mid_stride_bytes, uint64_t outer_stride_bytes,
                            uint32_t box0, uint32_t box1, uint32_t box2, CUtensorMapSwizzle swz);

// 4-D map: dims {d0, d1, d2, d3} with byte strides of d1, d2, d3.
spamm_status encode_tmap_4d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, const uint64_t dims[4],
                            const uint64_t stride_bytes[3], const uint32_t box[4], CUtensorMapSwizzle swz);

// TMA tensor-map encoder from the driver (resolved once via cudaGetDriverEntryPoint).
spamm_status encode_tmap_2d(CUtensorMap* map, CUtensorMapDataType dt, uint32_t esize, const void* base,
                            uint64_t inner, uint64_t outer, uint64_t ld_elems, uint32_t box_inner,
                            uint32_t box_outer, CUtensorMapSwizzle swz);

// stage drivers shared by api.cu and mgpu.cu
spamm_status do_norms_range(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t ar0,
                            int64_t ar1, int64_t bj0, int64_t bj1, cudaStream_t s);
spamm_status do_multiply(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                         cudaStream_t s, bool fuse = false);
spamm_status check_matrix(const void* ptr, int64_t rows, int64_t cols, int64_t ld, size_t esize, const char* name);

}  // namespace spamm
