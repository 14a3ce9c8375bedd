// api.cu -- the C ABI of libspamm.so (include/spamm.h): plan lifetime, argument
// validation, stage orchestration, introspection and error reporting.
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

#include "internal.h"

namespace spamm {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
spamm_status fail(spamm_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
spamm_status cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return e == cudaErrorMemoryAllocation ? SPAMM_E_NOMEM : SPAMM_E_CUDA;
}
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ----------------------------------------------------------------- TMA maps
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static bool resolve_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

spamm_status encode_tmap_2d(CUtensorMap* map, CUtensorMapDataType dt, uint32_t esize, const void* base,
                            uint64_t inner, uint64_t outer, uint64_t ld_elems, uint32_t box_inner,
                            uint32_t box_outer, CUtensorMapSwizzle swz) {
  if (!resolve_encode()) return fail(SPAMM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * esize};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(map, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SPAMM_E_INVALID, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return SPAMM_OK;
}

spamm_status encode_tmap_3d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner,
                            uint64_t mid, uint64_t outer, uint64_t mid_stride_bytes, uint64_t outer_stride_bytes,
                            uint32_t box0, uint32_t box1, uint32_t box2, CUtensorMapSwizzle swz) {
  if (!resolve_encode()) return fail(SPAMM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {inner, mid, outer};
  cuuint64_t strides[2] = {mid_stride_bytes, outer_stride_bytes};
  cuuint32_t box[3] = {box0, box1, box2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(map, dt, 3, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SPAMM_E_INVALID, "cuTensorMapEncodeTiled(3d) failed (" + std::to_string(r) + ")");
  return SPAMM_OK;
}

spamm_status encode_tmap_4d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, const uint64_t dims[4],
                            const uint64_t stride_bytes[3], const uint32_t box[4], CUtensorMapSwizzle swz) {
  if (!resolve_encode()) return fail(SPAMM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t d[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t st[3] = {stride_bytes[0], stride_bytes[1], stride_bytes[2]};
  cuuint32_t b[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = g_encode(map, dt, 4, const_cast<void*>(base), d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SPAMM_E_INVALID, "cuTensorMapEncodeTiled(4d) failed (" + std::to_string(r) + ")");
  return SPAMM_OK;
}

// --------------------------------------------------------------- validation
static size_t esize_of(spamm_precision p) { return f32_inputs(p) ? 4 : 2; }

spamm_status check_matrix(const void* ptr, int64_t rows, int64_t cols, int64_t ld, size_t esize, const char* name) {
  if (ptr == nullptr) return fail(SPAMM_E_INVALID, std::string(name) + " is NULL");
  if (ld < cols) return fail(SPAMM_E_INVALID, std::string(name) + ": leading dimension < columns");
  if ((reinterpret_cast<uintptr_t>(ptr) & 15u) != 0)
    return fail(SPAMM_E_INVALID, std::string(name) + " is not 16-byte aligned");
  if ((static_cast<uint64_t>(ld) * esize) % 16 != 0)
    return fail(SPAMM_E_INVALID, std::string(name) + ": ld*sizeof(elem) must be a multiple of 16");
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(SPAMM_E_INVALID, std::string(name) + " is not a CUDA pointer");
  }
  if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
    return fail(SPAMM_E_INVALID, std::string(name) + " is not a device pointer");
  (void)rows;
  return SPAMM_OK;
}

static bool tau_ok(double tau) { return std::isfinite(tau) && tau >= 0.0; }

static spamm_status alloc(void** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(SPAMM_E_NOMEM, "cudaMalloc(" + std::to_string(bytes) + ") failed: " + cudaGetErrorString(e));
  }
  return SPAMM_OK;
}

__global__ void transpose_f64_kernel(const double* __restrict__ in, int64_t rows, int64_t cols,
                                     double* __restrict__ out) {
  __shared__ double t[32][33];
  const int64_t c = static_cast<int64_t>(blockIdx.x) * 32 + threadIdx.x;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = static_cast<int64_t>(blockIdx.y) * 32 + k;
    if (r < rows && c < cols) t[k][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  const int64_t r2 = static_cast<int64_t>(blockIdx.y) * 32 + threadIdx.x;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c2 = static_cast<int64_t>(blockIdx.x) * 32 + k;
    if (r2 < rows && c2 < cols) out[c2 * rows + r2] = t[threadIdx.x][k];
  }
}

spamm_status launch_transpose_f64(const double* in, int64_t rows, int64_t cols, double* out, cudaStream_t s) {
  const dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  transpose_f64_kernel<<<grid, dim3(32, 8), 0, s>>>(in, rows, cols, out);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

static void free_plan(Plan* p) {
  if (!p) return;
  void* ptrs[] = {p->nA, p->nBt, p->pyr, p->V, p->U, p->L, p->leaf_start, p->row_work, p->sched,
                  p->leaf_k, p->macro_ent, p->macro_run, p->order, p->bucket_pos, p->mstart, p->d_range, p->tile_lists,
                  p->ts_cnt, p->ts_part, p->planes, p->nC, p->im2col};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  for (auto& e : p->ev)
    if (e) cudaEventDestroy(e);
  delete p;
}

// per-C-tile k lists (2 B per C tile and k: 17 GB at N = 65536) are reserved at plan creation
// when under this budget, else on the first request for them
static constexpr size_t kLeafEagerBudget = size_t(2) << 30;

static spamm_status ensure_leaf_storage(Plan& p) {
  if (p.leaf_alloc) return SPAMM_OK;
  SPAMM_TRY(alloc(reinterpret_cast<void**>(&p.leaf_k),
                  sizeof(uint16_t) * static_cast<size_t>(p.BM * p.BN) * static_cast<size_t>(p.BK)));
  p.leaf_alloc = true;
  return SPAMM_OK;
}

// host view of the range decided on the device (multi-GPU partition)
spamm_status sync_range(Plan& p) {
  if (!p.range_on_device) return SPAMM_OK;
  int64_t h[kRangeWords];
  SPAMM_CUDA_TRY(cudaStreamSynchronize(p.last_stream));
  SPAMM_CUDA_TRY(cudaMemcpy(h, p.d_range, sizeof(h), cudaMemcpyDeviceToHost));
  p.row_begin_macro = h[0];
  p.row_end_macro = h[1];
  const int nr = static_cast<int>(h[4]);
  p.last_partition.assign(nr + 1, 0);
  for (int q = 0; q <= nr; ++q) p.last_partition[q] = std::min<int64_t>(h[6 + q] * p.MI, p.BM);
  p.range_on_device = false;
  return SPAMM_OK;
}

}  // namespace spamm

using namespace spamm;

extern "C" {

const char* spamm_status_string(spamm_status s) {
  switch (s) {
    case SPAMM_OK: return "SPAMM_OK";
    case SPAMM_E_INVALID: return "SPAMM_E_INVALID";
    case SPAMM_E_UNSUPPORTED: return "SPAMM_E_UNSUPPORTED";
    case SPAMM_E_CUDA: return "SPAMM_E_CUDA";
    case SPAMM_E_NOMEM: return "SPAMM_E_NOMEM";
    case SPAMM_E_NCCL: return "SPAMM_E_NCCL";
    case SPAMM_E_STATE: return "SPAMM_E_STATE";
  }
  return "SPAMM_E_UNKNOWN";
}

const char* spamm_last_error(void) { return g_last_error.c_str(); }

int64_t spamm_launch_count(void) { return g_launches.load(); }

spamm_status spamm_plan_ex(spamm_plan_t* out, int64_t M, int64_t N, int64_t K, int32_t tile, double tau,
                           spamm_precision prec, uint32_t flags) {
  if (!out) return fail(SPAMM_E_INVALID, "plan out-pointer is NULL");
  *out = nullptr;
  if (M <= 0 || N <= 0 || K <= 0) return fail(SPAMM_E_INVALID, "M, N, K must be positive");
  if (!tau_ok(tau)) return fail(SPAMM_E_INVALID, "tau must be finite and >= 0");
  if (prec != SPAMM_FP32 && prec != SPAMM_BF16 && prec != SPAMM_FP16 && prec != SPAMM_FP32X3)
    return fail(SPAMM_E_INVALID, "unknown precision");
  if (flags & ~(SPAMM_FLAG_TIMING | SPAMM_FLAG_LARGE_TILES | SPAMM_FLAG_STAGED))
    return fail(SPAMM_E_INVALID, "unknown plan flag");
  if (tile != kTile) {
    if (tile == 64 || tile == 128) return fail(SPAMM_E_UNSUPPORTED, "only tile (LoNum) = 32 is implemented");
    return fail(SPAMM_E_INVALID, "tile must be 32, 64 or 128");
  }
  const int64_t BM = (M + kTile - 1) / kTile, BK = (K + kTile - 1) / kTile, BN = (N + kTile - 1) / kTile;
  if (BK > 65535) return fail(SPAMM_E_UNSUPPORTED, "K/tile must be <= 65535 (uint16 k lists)");
  if (M > (int64_t(1) << 31) || N > (int64_t(1) << 31) || K > (int64_t(1) << 31))
    return fail(SPAMM_E_UNSUPPORTED, "dimensions must be < 2^31 (TMA coordinates)");
  int dev = 0;
  SPAMM_CUDA_TRY(cudaGetDevice(&dev));
  Plan* p = new Plan();
  p->M = M;
  p->N = N;
  p->K = K;
  p->tau = tau;
  p->prec = prec;
  p->flags = flags;
  p->BM = BM;
  p->BK = BK;
  p->BN = BN;
  cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, dev);
  const bool tc = !f32_inputs(prec);   // BF16/FP16: 256 x 256 two-issuer tensor path
  // ... unless the problem has fewer 256 x 256 macro-tiles than SMs and its 128 x 128 tiles still fit
  // one wave: then 128 x 128 tiles (up to 4x the CTAs; measured: N = 1024 multiply 17.5 -> 15.3 us,
  // but conv2_1's 200 tiles in two waves 17 -> 29 us, so that shape stays on 256 x 256)
  const int64_t tiles256 = ((BM + kMacroTC - 1) / kMacroTC) * ((BN + kMacroTC - 1) / kMacroTC);
  const int64_t tiles128 = ((BM + kMacroF32 - 1) / kMacroF32) * ((BN + kMacroF32 - 1) / kMacroF32);
  p->x1 = tc && !(flags & SPAMM_FLAG_LARGE_TILES) && tiles256 < p->num_sms && tiles128 <= p->num_sms;
  const bool dual = tc && !p->x1;
  p->MI = p->MJ = dual ? kMacroTC : kMacroF32;
  p->GM = (BM + p->MI - 1) / p->MI;
  p->GN = (BN + p->MJ - 1) / p->MJ;
  p->NC = (BK + kChunk - 1) / kChunk;
  // small problems: one 128 x 128 macro-tile per SM at most -> the skip map is decided inside the
  // multiply (one launch fewer on spamm_run; the per-tile list work is BK/32 warp steps)
  p->fused = !(flags & SPAMM_FLAG_STAGED) && (p->x1 || f32_inputs(prec)) && p->GM * p->GN <= p->num_sms;
  p->device = dev;
  p->row_begin_macro = 0;
  p->row_end_macro = p->GM;
  const int64_t nleaf = BM * BN, nmac = p->GM * p->GN;
  spamm_status st = SPAMM_OK;
#define ALLOC(field, type, count)                                                                   \
  if (st == SPAMM_OK)                                                                               \
    st = alloc(reinterpret_cast<void**>(&p->field), sizeof(type) * static_cast<size_t>(count));
  ALLOC(nA, double, BM * BK);
  ALLOC(nBt, double, BN * BK);
  ALLOC(pyr, double, 2 * (p->GM + p->GN) * p->NC);
  ALLOC(V, int64_t, nleaf);
  ALLOC(leaf_start, int64_t, nleaf);
  ALLOC(U, int64_t, nmac + 1);
  ALLOC(L, int64_t, nmac + 1);
  p->NSB = ((p->GM + SPAMM_ORD_R - 1) / SPAMM_ORD_R) * ((p->GN + SPAMM_ORD_C - 1) / SPAMM_ORD_C);
  ALLOC(row_work, int64_t, ws_words(*p));
  ALLOC(tile_lists, int32_t, 2 * nmac);
  ALLOC(sched, unsigned int, 4);   // [0] tile claims, [1] zero-fill unit claims
  ALLOC(order, int32_t, nmac);
  ALLOC(bucket_pos, int64_t, std::max<int64_t>(BK + 2, p->NSB + 1));
  ALLOC(mstart, int64_t, nmac);
  ALLOC(d_range, int64_t, kRangeWords);
  // macro lists at their worst case (macro-tile t owns entries [t*BK, t*BK + U[t])): the skip map
  // is one stream-ordered pass with no host synchronisation
  ALLOC(macro_ent, uint8_t, static_cast<size_t>(dual ? 16 : 8) * static_cast<size_t>(nmac * BK));
  if (dual) ALLOC(macro_run, uint4, 2 * nmac * BK);   // one 4 x 8 run entry per 128-row half and k-step
#undef ALLOC
  if (st == SPAMM_OK) {
    p->hist = p->row_work + BM;
    p->totals = p->hist + BK + 2;
    p->hist_sb = p->totals + 4;
    p->ws_cnt = reinterpret_cast<unsigned int*>(p->hist_sb + p->NSB);
    p->bucket_cnt = p->hist_sb + p->NSB + 2;
    p->sb_bits = reinterpret_cast<unsigned long long*>(p->bucket_cnt + ws_buckets(*p));
  }
  if (st == SPAMM_OK && (cudaMemset(p->U, 0, sizeof(int64_t) * (nmac + 1)) != cudaSuccess ||
                         cudaMemset(p->L, 0, sizeof(int64_t) * (nmac + 1)) != cudaSuccess ||
                         cudaMemset(p->sched, 0, 4 * sizeof(unsigned int)) != cudaSuccess ||
                         cudaMemset(p->row_work, 0, sizeof(int64_t) * ws_words(*p)) != cudaSuccess))
    st = fail(SPAMM_E_CUDA, "cudaMemset failed");
  if (st == SPAMM_OK) {
    std::vector<int64_t> h(static_cast<size_t>(nmac));
    for (int64_t t = 0; t < nmac; ++t) h[static_cast<size_t>(t)] = t * BK;
    if (cudaMemcpy(p->mstart, h.data(), sizeof(int64_t) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      st = fail(SPAMM_E_CUDA, "cudaMemcpy failed");
  }
  if (st == SPAMM_OK && sizeof(uint16_t) * static_cast<size_t>(nleaf) * static_cast<size_t>(BK) <= kLeafEagerBudget)
    st = ensure_leaf_storage(*p);
  // FP32X3: the three bfloat16 planes of A and of B (leading dimensions rounded to 8 elements
  // so every row is 16-byte aligned for TMA)
  if (st == SPAMM_OK && prec == SPAMM_FP32X3) {
    p->ldpa = (K + 7) / 8 * 8;
    p->ldpb = (N + 7) / 8 * 8;
    st = alloc(reinterpret_cast<void**>(&p->planes),
               sizeof(uint16_t) * 3 * (static_cast<size_t>(M * p->ldpa) + static_cast<size_t>(K * p->ldpb)));
  }
  if (st == SPAMM_OK) {
    for (auto& e : p->ev)
      if (cudaEventCreate(&e) != cudaSuccess) st = fail(SPAMM_E_CUDA, "cudaEventCreate failed");
  }
  if (st != SPAMM_OK) {
    free_plan(p);
    return st;
  }
  *out = reinterpret_cast<spamm_plan_t>(p);
  return SPAMM_OK;
}

spamm_status spamm_plan(spamm_plan_t* p, int64_t N, int32_t tile, double tau, spamm_precision prec) {
  return spamm_plan_ex(p, N, N, N, tile, tau, prec, SPAMM_FLAG_NONE);
}

spamm_status spamm_plan_destroy(spamm_plan_t h) {
  if (!h) return SPAMM_OK;
  Plan* p = reinterpret_cast<Plan*>(h);
  // the plan's work is ordered on the stream of its last call: wait for it, not for the device
  if (p->last_stream != nullptr || p->norms_ready) cudaStreamSynchronize(p->last_stream);
  free_plan(p);
  return SPAMM_OK;
}

spamm_status spamm_set_tau(spamm_plan_t h, double tau) {
  if (!h) return fail(SPAMM_E_INVALID, "plan is NULL");
  if (!tau_ok(tau)) return fail(SPAMM_E_INVALID, "tau must be finite and >= 0");
  Plan* p = reinterpret_cast<Plan*>(h);
  p->tau = tau;
  p->skipmap_ready = false;
  return SPAMM_OK;
}

spamm_status spamm_set_scalars(spamm_plan_t h, double alpha, double beta) {
  if (!h) return fail(SPAMM_E_INVALID, "plan is NULL");
  if (!std::isfinite(alpha) || !std::isfinite(beta)) return fail(SPAMM_E_INVALID, "alpha and beta must be finite");
  Plan* p = reinterpret_cast<Plan*>(h);
  p->alpha = alpha;
  p->beta = beta;
  return SPAMM_OK;
}

}  // extern "C"

namespace spamm {

// stage 1 over tile rows [ar0, ar1) of A and tile columns [bj0, bj1) of B; with zero_ws the norm
// kernel also zeroes the skip map's counters (saves a memset node in spamm_run)
static spamm_status norms_impl(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t ar0,
                               int64_t ar1, int64_t bj0, int64_t bj1, bool zero_ws, cudaStream_t s) {
  SPAMM_TRY(check_matrix(A, p.M, p.K, lda, esize_of(p.prec), "A"));
  SPAMM_TRY(check_matrix(B, p.K, p.N, ldb, esize_of(p.prec), "B"));
  const bool timing = p.flags & SPAMM_FLAG_TIMING;
  if (timing) SPAMM_CUDA_TRY(cudaEventRecord(p.ev[0], s));
  // A (M x K): tile row i, tile col k -> nA[i*BK + k];  B (K x N) column strip [bj0*T, bj1*T):
  // tile row k, tile col j -> nBt[j*BK + k]
  p.zero_ws_next = zero_ws;
  const spamm_status st = launch_norms2(p, A, lda, ar0, ar1, B, ldb, bj0, bj1, s);
  p.zero_ws_next = false;
  SPAMM_TRY(st);
  p.ws_zeroed = zero_ws;
  if (timing) SPAMM_CUDA_TRY(cudaEventRecord(p.ev[1], s));
  p.ev_norms = timing;
  p.norms_ready = true;
  p.pyr_ready = false;
  p.skipmap_ready = false;
  p.last_stream = s;
  return SPAMM_OK;
}

spamm_status do_norms_range(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t ar0,
                            int64_t ar1, int64_t bj0, int64_t bj1, cudaStream_t s) {
  return norms_impl(p, A, lda, B, ldb, ar0, ar1, bj0, bj1, false, s);
}

static spamm_status do_skipmap(Plan& p, cudaStream_t s) {
  if (!p.norms_ready) return fail(SPAMM_E_STATE, "spamm_build_skipmap before spamm_norms");
  const bool timing = p.flags & SPAMM_FLAG_TIMING;
  if (timing) SPAMM_CUDA_TRY(cudaEventRecord(p.ev[2], s));
  // the norm pyramid pays off once there are chunks to skip: K of more than two 32-tile chunks
  if (!p.pyr_ready && p.NC > 2) SPAMM_TRY(launch_pyramid(p, s));
  // row_work [BM], hist [BK+2] and totals [2] are contiguous in one allocation
  if (!p.ws_zeroed) SPAMM_CUDA_TRY(cudaMemsetAsync(p.row_work, 0, sizeof(int64_t) * ws_words(p), s));
  p.ws_zeroed = false;
  SPAMM_TRY(launch_skipmap(p, 0, p.GM, false, true, true, s));
  p.sched_zeroed = true;   // the last CTA zeroes the multiply's claim counters
  if (timing) SPAMM_CUDA_TRY(cudaEventRecord(p.ev[3], s));
  p.ev_skip = timing;
  p.leaf_ready = false;
  p.range_on_device = false;
  p.row_begin_macro = 0;
  p.row_end_macro = p.GM;
  p.skipmap_ready = true;
  p.last_stream = s;
  return SPAMM_OK;
}

spamm_status do_multiply(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                         cudaStream_t s, bool fuse) {
  if (!fuse && !p.skipmap_ready) return fail(SPAMM_E_STATE, "spamm_multiply before spamm_build_skipmap");
  SPAMM_TRY(check_matrix(A, p.M, p.K, lda, esize_of(p.prec), "A"));
  SPAMM_TRY(check_matrix(B, p.K, p.N, ldb, esize_of(p.prec), "B"));
  if (!p.out_low_only) SPAMM_TRY(check_matrix(C, p.M, p.N, ldc, 4, "C"));
  const bool timing = p.flags & SPAMM_FLAG_TIMING;
  if (timing) SPAMM_CUDA_TRY(cudaEventRecord(p.ev[4], s));
  if (p.prec == SPAMM_FP32X3) {
    SPAMM_TRY(launch_multiply_x3(p, C, ldc, fuse, s));
  } else if (p.prec == SPAMM_FP32) {
    SPAMM_TRY(launch_multiply_simt(p, static_cast<const float*>(A), lda, static_cast<const float*>(B), ldb, C, ldc,
                                   fuse, s));
  } else if (p.x1) {
    SPAMM_TRY(launch_multiply_x1(p, A, lda, B, ldb, C, ldc, fuse, s));
  } else {
    SPAMM_TRY(launch_multiply_dual(p, A, lda, B, ldb, C, ldc, s));
  }
  if (timing) SPAMM_CUDA_TRY(cudaEventRecord(p.ev[5], s));
  p.ev_mul = timing;
  p.last_stream = s;
  if (fuse) {   // the multiply wrote the complete skip map of the full range (multiply_x3.cu XFuse)
    if (timing) {   // stage 2 ran inside stage 3: zero-length skip-map interval
      SPAMM_CUDA_TRY(cudaEventRecord(p.ev[2], s));
      SPAMM_CUDA_TRY(cudaEventRecord(p.ev[3], s));
    }
    p.ev_skip = timing;
    p.ws_zeroed = false;
    p.leaf_ready = false;
    p.skipmap_ready = true;
  }
  return SPAMM_OK;
}

// spamm_run / AUTO: stages 1 and 2 (or stage 1 alone when the multiply decides the skip map)
static spamm_status do_auto(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, cudaStream_t s,
                            bool* fuse) {
  SPAMM_TRY(norms_impl(p, A, lda, B, ldb, 0, p.BM, 0, p.BN, true, s));
  *fuse = p.fused;
  if (!*fuse) return do_skipmap(p, s);
  p.skipmap_ready = false;
  p.range_on_device = false;
  p.row_begin_macro = 0;
  p.row_end_macro = p.GM;
  return SPAMM_OK;
}

}  // namespace spamm

extern "C" {

spamm_status spamm_norms(spamm_plan_t h, const void* A, int64_t lda, const void* B, int64_t ldb, void* stream) {
  if (!h) return fail(SPAMM_E_INVALID, "plan is NULL");
  Plan& p = *reinterpret_cast<Plan*>(h);
  return norms_impl(p, A, lda, B, ldb, 0, p.BM, 0, p.BN, false, static_cast<cudaStream_t>(stream));
}

spamm_status spamm_build_skipmap(spamm_plan_t h, void* stream) {
  if (!h) return fail(SPAMM_E_INVALID, "plan is NULL");
  Plan& p = *reinterpret_cast<Plan*>(h);
  return do_skipmap(p, static_cast<cudaStream_t>(stream));
}

spamm_status spamm_multiply(spamm_plan_t h, const void* A, int64_t lda, const void* B, int64_t ldb, float* C,
                            int64_t ldc, uint32_t flags, void* stream) {
  if (!h) return fail(SPAMM_E_INVALID, "plan is NULL");
  Plan& p = *reinterpret_cast<Plan*>(h);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (flags & ~SPAMM_MUL_AUTO) return fail(SPAMM_E_INVALID, "unknown spamm_multiply flag");
  bool fuse = false;
  if (flags & SPAMM_MUL_AUTO) SPAMM_TRY(do_auto(p, A, lda, B, ldb, s, &fuse));
  return do_multiply(p, A, lda, B, ldb, C, ldc, s, fuse);
}

spamm_status spamm_multiply_chain(spamm_plan_t h, const void* A, int64_t lda, const void* B, int64_t ldb, float* C,
                                  int64_t ldc, void* C_low, int64_t ldcl, uint32_t flags, void* stream) {
  if (!h) return fail(SPAMM_E_INVALID, "plan is NULL");
  Plan& p = *reinterpret_cast<Plan*>(h);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (flags & ~(SPAMM_MUL_AUTO | SPAMM_MUL_OUTPUT_NORMS | SPAMM_MUL_LOW_ONLY))
    return fail(SPAMM_E_INVALID, "unknown spamm_multiply_chain flag");
  const bool low_only = (flags & SPAMM_MUL_LOW_ONLY) != 0;
  if (C_low != nullptr) {
    if (f32_inputs(p.prec)) return fail(SPAMM_E_INVALID, "C_low is for BF16/FP16 plans (FP32 C is the next input)");
    SPAMM_TRY(check_matrix(C_low, p.M, p.N, ldcl, 2, "C_low"));
  }
  if (low_only) {
    if (C_low == nullptr) return fail(SPAMM_E_INVALID, "SPAMM_MUL_LOW_ONLY needs C_low");
    if (p.beta != 0.0) return fail(SPAMM_E_INVALID, "SPAMM_MUL_LOW_ONLY needs beta = 0 (no FP32 C to read)");
  }
  if (p.prec == SPAMM_FP32X3) return fail(SPAMM_E_UNSUPPORTED, "chained outputs: FP32, BF16, FP16 only");
  if ((flags & SPAMM_MUL_OUTPUT_NORMS) && !p.nC)
    SPAMM_TRY(alloc(reinterpret_cast<void**>(&p.nC), sizeof(double) * static_cast<size_t>(p.BM * p.BN)));
  bool fuse = false;
  if (flags & SPAMM_MUL_AUTO) SPAMM_TRY(do_auto(p, A, lda, B, ldb, s, &fuse));
  p.out_norms = (flags & SPAMM_MUL_OUTPUT_NORMS) != 0;
  p.out_low = C_low;
  p.out_ldl = ldcl;
  p.out_low_only = low_only;
  const spamm_status st = do_multiply(p, A, lda, B, ldb, low_only ? nullptr : C, ldc, s, fuse);
  p.nc_ready = st == SPAMM_OK && p.out_norms;
  p.out_norms = false;
  p.out_low = nullptr;
  p.out_low_only = false;
  return st;
}

spamm_status spamm_get_output_norms(spamm_plan_t h, const double** d_nC) {
  if (!h || !d_nC) return fail(SPAMM_E_INVALID, "plan or output is NULL");
  Plan& p = *reinterpret_cast<Plan*>(h);
  if (!p.nc_ready) return fail(SPAMM_E_STATE, "no spamm_multiply_chain with SPAMM_MUL_OUTPUT_NORMS on this plan");
  *d_nC = p.nC;
  return SPAMM_OK;
}

spamm_status spamm_set_norms(spamm_plan_t h, const double* nA, const double* nB, void* stream) {
  if (!h || !nA || !nB) return fail(SPAMM_E_INVALID, "plan or norm map is NULL");
  Plan& p = *reinterpret_cast<Plan*>(h);
  if (p.prec == SPAMM_FP32X3) return fail(SPAMM_E_UNSUPPORTED, "SPAMM_FP32X3 needs spamm_norms (it also splits A, B)");
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, nA) != cudaSuccess || at.type != cudaMemoryTypeDevice ||
      cudaPointerGetAttributes(&at, nB) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    return fail(SPAMM_E_INVALID, "norm maps must be device pointers");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SPAMM_CUDA_TRY(cudaMemcpyAsync(p.nA, nA, sizeof(double) * static_cast<size_t>(p.BM * p.BK), cudaMemcpyDeviceToDevice, s));
  SPAMM_TRY(launch_transpose_f64(nB, p.BK, p.BN, p.nBt, s));   // nB [BK][BN] -> nB^T [BN][BK]
  p.norms_ready = true;
  p.pyr_ready = false;
  p.skipmap_ready = false;
  p.b_is_a = false;
  p.last_stream = s;
  return SPAMM_OK;
}

spamm_status spamm_run(spamm_plan_t h, const void* A, int64_t lda, const void* B, int64_t ldb, float* C,
                       int64_t ldc, void* stream) {
  return spamm_multiply(h, A, lda, B, ldb, C, ldc, SPAMM_MUL_AUTO, stream);
}

spamm_status spamm_get_norms(spamm_plan_t h, const double** dA, const double** dBt, int64_t* BM, int64_t* BK,
                             int64_t* BN) {
  if (!h) return fail(SPAMM_E_INVALID, "plan is NULL");
  Plan& p = *reinterpret_cast<Plan*>(h);
  if (dA) *dA = p.nA;
  if (dBt) *dBt = p.nBt;
  if (BM) *BM = p.BM;
  if (BK) *BK = p.BK;
  if (BN) *BN = p.BN;
  return p.norms_ready ? SPAMM_OK : fail(SPAMM_E_STATE, "norms not computed");
}

// The skip map writes the macro-level lists only; the per-C-tile view is expanded from them on
// first request (same stream, then synchronised).
static spamm_status ensure_leaf_lists(spamm::Plan& p) {
  if (p.leaf_ready) return SPAMM_OK;
  SPAMM_TRY(sync_range(p));
  SPAMM_TRY(ensure_leaf_storage(p));
  SPAMM_TRY(launch_leaf_expand(p, p.last_stream));
  SPAMM_CUDA_TRY(cudaStreamSynchronize(p.last_stream));
  p.leaf_ready = true;
  return SPAMM_OK;
}

spamm_status spamm_get_skipmap(spamm_plan_t h, const int64_t** d_tile_start, const uint16_t** d_k_idx,
                               int64_t* kept) {
  if (!h) return fail(SPAMM_E_INVALID, "plan is NULL");
  Plan& p = *reinterpret_cast<Plan*>(h);
  if (!p.skipmap_ready) return fail(SPAMM_E_STATE, "skip map not built");
  SPAMM_TRY(ensure_leaf_lists(p));
  if (d_tile_start) *d_tile_start = p.leaf_start;
  if (d_k_idx) *d_k_idx = p.leaf_k;
  if (kept) {
    SPAMM_CUDA_TRY(cudaStreamSynchronize(p.last_stream));
    SPAMM_CUDA_TRY(cudaMemcpy(kept, p.totals, sizeof(int64_t), cudaMemcpyDeviceToHost));
  }
  return SPAMM_OK;
}

spamm_status spamm_get_counts(spamm_plan_t h, const int64_t** d_V, const int64_t** d_row_work) {
  if (!h) return fail(SPAMM_E_INVALID, "plan is NULL");
  Plan& p = *reinterpret_cast<Plan*>(h);
  if (!p.skipmap_ready) return fail(SPAMM_E_STATE, "skip map not built");
  if (d_V) SPAMM_TRY(ensure_leaf_lists(p));
  if (d_V) *d_V = p.V;
  if (d_row_work) *d_row_work = p.row_work;
  return SPAMM_OK;
}

spamm_status spamm_get_macro(spamm_plan_t h, const int64_t** d_start, const int64_t** d_count,
                             const uint32_t** d_entries, const int32_t** d_order, int64_t* GM, int64_t* GN) {
  if (!h) return fail(SPAMM_E_INVALID, "plan is NULL");
  Plan& p = *reinterpret_cast<Plan*>(h);
  if (!p.skipmap_ready) return fail(SPAMM_E_STATE, "skip map not built");
  SPAMM_TRY(sync_range(p));
  if (d_start) *d_start = p.mstart;
  if (d_count) *d_count = p.U;
  if (d_entries) *d_entries = reinterpret_cast<const uint32_t*>(p.macro_ent);
  if (d_order) *d_order = p.order;
  if (GM) *GM = p.GM;
  if (GN) *GN = p.GN;
  return SPAMM_OK;
}

spamm_status spamm_get_partition(spamm_plan_t h, int64_t* row_begin, int nranks) {
  if (!h || !row_begin) return fail(SPAMM_E_INVALID, "NULL argument");
  Plan& p = *reinterpret_cast<Plan*>(h);
  SPAMM_TRY(sync_range(p));
  if (static_cast<int>(p.last_partition.size()) != nranks + 1)
    return fail(SPAMM_E_STATE, "no partition for this rank count");
  std::memcpy(row_begin, p.last_partition.data(), sizeof(int64_t) * (nranks + 1));
  return SPAMM_OK;
}

spamm_status spamm_get_stats(spamm_plan_t h, spamm_stats* out) {
  if (!h || !out) return fail(SPAMM_E_INVALID, "NULL argument");
  Plan& p = *reinterpret_cast<Plan*>(h);
  SPAMM_TRY(sync_range(p));
  std::memset(out, 0, sizeof(*out));
  out->M = p.M;
  out->N = p.N;
  out->K = p.K;
  out->BM = p.BM;
  out->BK = p.BK;
  out->BN = p.BN;
  out->tile = p.tile;
  out->macro_i = p.MI;
  out->macro_j = p.MJ;
  out->tau = p.tau;
  out->precision = p.prec;
  out->row_begin = static_cast<int32_t>(p.row_begin_macro * p.MI);
  out->row_end = static_cast<int32_t>(std::min<int64_t>(p.row_end_macro * p.MI, p.BM));
  out->ms_norms = out->ms_skipmap = out->ms_multiply = -1.f;
  SPAMM_CUDA_TRY(cudaStreamSynchronize(p.last_stream));
  if (p.skipmap_ready) {
    int64_t tot[2];
    SPAMM_CUDA_TRY(cudaMemcpy(tot, p.totals, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost));
    out->kept = tot[0];
    out->macro_entries = tot[1];
    out->valid_ratio = static_cast<double>(tot[0]) / (static_cast<double>(p.BM) * p.BK * p.BN);
  }
  if (p.ev_norms) cudaEventElapsedTime(&out->ms_norms, p.ev[0], p.ev[1]);
  if (p.ev_skip) cudaEventElapsedTime(&out->ms_skipmap, p.ev[2], p.ev[3]);
  if (p.ev_mul) cudaEventElapsedTime(&out->ms_multiply, p.ev[4], p.ev[5]);
  return SPAMM_OK;
}

spamm_status spamm_partition_rows(const int64_t* row_work, int64_t BM, int nranks, int64_t* row_begin) {
  if (!row_work || !row_begin) return fail(SPAMM_E_INVALID, "NULL argument");
  if (BM <= 0 || nranks <= 0) return fail(SPAMM_E_INVALID, "BM and nranks must be positive");
  // cut r = first row i whose exclusive prefix `pre` reaches the r-th share by half of its own
  // work:  pre + w_i / 2 >= r * total / n  <=>  2 n pre + n w_i >= 2 r total  (integers: the
  // device partition of spamm_multiply_mgpu applies the identical rule to macro rows)
  int64_t total = 0;
  for (int64_t i = 0; i < BM; ++i) {
    if (row_work[i] < 0) return fail(SPAMM_E_INVALID, "negative row work");
    total += row_work[i];
  }
  const int64_t n = nranks;
  row_begin[0] = 0;
  int64_t pre = 0, i = 0;
  for (int r = 1; r < nranks; ++r) {
    while (i < BM && 2 * n * pre + n * row_work[i] < 2 * static_cast<int64_t>(r) * total) {
      pre += row_work[i];
      ++i;
    }
    row_begin[r] = std::max<int64_t>(i, row_begin[r - 1]);
  }
  row_begin[nranks] = BM;
  return SPAMM_OK;
}

}  // extern "C"
