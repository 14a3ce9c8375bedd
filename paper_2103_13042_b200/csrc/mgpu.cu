// mgpu.cu -- multi-GPU SpAMM over NCCL (Sec. 3.4, Alg. 4) with the
// load-balance idea of Sec. 3.5.1 applied to the row partition.
//
// The paper row-partitions C evenly and moves data with Unified-Memory page faults
// (PAPER.md:211).  Here: one process per GPU, three stream-ordered phases separated by NCCL
// collectives, and no host synchronisation anywhere in a step (unless C is gathered):
//   phase 1  each rank norms 1/n of A's tile rows and of B's tile columns  [all-gather the maps]
//            (FP32X3 norms everything: its split planes of every row are operands)
//   phase 2  norm pyramid; the skip map of the rank's provisional (even) macro-row share, which
//            also yields that share's row work                                [all-reduce row work]
//   phase 3  the partition kernel cuts macro rows at equal shares of the total work (the same
//            rule as spamm_partition_rows) into the plan's device range block; the skip map of
//            the final range's rows outside the provisional share (usually a thin margin) and the
//            LPT order of the final range; the multiply of the final range    [optional C gather]
// The collectives are behind a small transport interface: NCCL for spamm_multiply_mgpu, device
// copies between the plans of one GPU for spamm_multiply_mgpu_local (the same phases and kernels,
// used to verify multi-rank results on one device).
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.h"

namespace spamm {

spamm_status sync_range(Plan& p);

static spamm_status nccl_fail(ncclResult_t r, const char* where) {
  return fail(SPAMM_E_NCCL, std::string(where) + ": " + ncclGetErrorString(r));
}
#define SPAMM_NCCL_TRY(expr)                                     \
  do {                                                           \
    ncclResult_t _r = (expr);                                    \
    if (_r != ncclSuccess) return ::spamm::nccl_fail(_r, #expr); \
  } while (0)

static inline int64_t share(int64_t n, int r, int nr) { return n * r / nr; }

static bool full_norms(const Plan& p, int nranks) { return nranks == 1 || p.prec == SPAMM_FP32X3; }

static spamm_status phase_norms(Plan& p, int rank, int nranks, const void* A, int64_t lda, const void* B, int64_t ldb,
                                cudaStream_t s) {
  if (full_norms(p, nranks)) return do_norms_range(p, A, lda, B, ldb, 0, p.BM, 0, p.BN, s);
  return do_norms_range(p, A, lda, B, ldb, share(p.BM, rank, nranks), share(p.BM, rank + 1, nranks),
                        share(p.BN, rank, nranks), share(p.BN, rank + 1, nranks), s);
}

static spamm_status phase_provisional(Plan& p, int rank, int nranks, cudaStream_t s) {
  const bool timing = p.flags & SPAMM_FLAG_TIMING;
  if (timing) SPAMM_CUDA_TRY(cudaEventRecord(p.ev[2], s));
  SPAMM_CUDA_TRY(cudaMemsetAsync(p.row_work, 0, sizeof(int64_t) * ws_words(p), s));
  SPAMM_TRY(launch_pyramid(p, s));
  const int64_t g0 = share(p.GM, rank, nranks), g1 = share(p.GM, rank + 1, nranks);
  // one rank: this is the whole skip map, with its LPT order
  SPAMM_TRY(launch_skipmap(p, g0, g1, false, nranks == 1, true, s));
  p.ws_zeroed = false;
  return SPAMM_OK;
}

static spamm_status phase_final(Plan& p, int rank, int nranks, const void* A, int64_t lda, const void* B, int64_t ldb,
                                float* C, int64_t ldc, cudaStream_t s) {
  const bool timing = p.flags & SPAMM_FLAG_TIMING;
  if (nranks > 1) {
    SPAMM_TRY(launch_partition(p, rank, nranks, s));
    // rows of the final range outside the provisional share, then the order of the final range
    SPAMM_TRY(launch_skipmap(p, 0, 0, true, true, false, s));
    p.range_on_device = true;
  } else {
    p.range_on_device = false;
    p.row_begin_macro = 0;
    p.row_end_macro = p.GM;
    p.last_partition.assign({0, p.BM});
  }
  p.sched_zeroed = true;   // the skip map's last CTA zeroed the multiply's claim counters
  if (timing) SPAMM_CUDA_TRY(cudaEventRecord(p.ev[3], s));
  p.ev_skip = timing;
  p.skipmap_ready = true;
  p.leaf_ready = false;
  p.last_stream = s;
  return do_multiply(p, A, lda, B, ldb, C, ldc, s);
}

// C rows [r0, r1) of every rank (host view of the device cut; synchronises the stream)
static spamm_status rank_rows(Plan& p, int nranks, std::vector<int64_t>& rows) {
  SPAMM_TRY(sync_range(p));
  rows.assign(nranks + 1, 0);
  for (int q = 0; q <= nranks; ++q) rows[q] = std::min<int64_t>(p.last_partition[q] * kTile, p.M);
  return SPAMM_OK;
}

static spamm_status check_common(const Plan& p, int nranks) {
  if (nranks > kMaxRanks) return fail(SPAMM_E_UNSUPPORTED, "at most 64 ranks");
  if (p.out_norms || p.out_low) return fail(SPAMM_E_UNSUPPORTED, "chained outputs are single-GPU");
  return SPAMM_OK;
}

__global__ void add_i64_kernel(int64_t* __restrict__ dst, const int64_t* __restrict__ src, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) dst[i] += src[i];
}

}  // namespace spamm

using namespace spamm;

extern "C" {

spamm_status spamm_nccl_unique_id(uint8_t out_id[128]) {
  if (!out_id) return fail(SPAMM_E_INVALID, "NULL id buffer");
  ncclUniqueId id;
  SPAMM_NCCL_TRY(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out_id, &id, 128);
  return SPAMM_OK;
}

spamm_status spamm_nccl_comm_init(void** comm, int nranks, int rank, const uint8_t id[128]) {
  if (!comm || !id) return fail(SPAMM_E_INVALID, "NULL argument");
  if (nranks <= 0 || rank < 0 || rank >= nranks) return fail(SPAMM_E_INVALID, "bad rank / nranks");
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  ncclComm_t c;
  SPAMM_NCCL_TRY(ncclCommInitRank(&c, nranks, uid, rank));
  *comm = c;
  return SPAMM_OK;
}

spamm_status spamm_nccl_comm_destroy(void* comm) {
  if (!comm) return SPAMM_OK;
  SPAMM_NCCL_TRY(ncclCommDestroy(static_cast<ncclComm_t>(comm)));
  return SPAMM_OK;
}

spamm_status spamm_multiply_mgpu(spamm_plan_t h, void* nccl_comm, int rank, int nranks, const void* A, int64_t lda,
                                 const void* B, int64_t ldb, float* C, int64_t ldc, uint32_t flags, void* stream) {
  if (!h) return fail(SPAMM_E_INVALID, "plan is NULL");
  if (nranks <= 0 || rank < 0 || rank >= nranks) return fail(SPAMM_E_INVALID, "bad rank / nranks");
  if (nranks > 1 && !nccl_comm) return fail(SPAMM_E_INVALID, "NCCL communicator is NULL");
  if (flags & ~(SPAMM_MGPU_INPUTS_ON_ROOT | SPAMM_MGPU_GATHER_C)) return fail(SPAMM_E_INVALID, "unknown flag");
  Plan& p = *reinterpret_cast<Plan*>(h);
  SPAMM_TRY(check_common(p, nranks));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
  const size_t es = f32_inputs(p.prec) ? 4 : 2;

  // 0. inputs from the root (Alg. 4 lines 4 and 7: B to every GPU, A rows)
  if ((flags & SPAMM_MGPU_INPUTS_ON_ROOT) && nranks > 1) {
    SPAMM_NCCL_TRY(ncclGroupStart());
    SPAMM_NCCL_TRY(ncclBroadcast(A, const_cast<void*>(A), static_cast<size_t>((p.M - 1) * lda + p.K) * es,
                                 ncclUint8, 0, comm, s));
    SPAMM_NCCL_TRY(ncclBroadcast(B, const_cast<void*>(B), static_cast<size_t>((p.K - 1) * ldb + p.N) * es,
                                 ncclUint8, 0, comm, s));
    SPAMM_NCCL_TRY(ncclGroupEnd());
  }
  // 1. norms of this rank's share, all-gathered (grouped broadcasts of contiguous map slices)
  SPAMM_TRY(phase_norms(p, rank, nranks, A, lda, B, ldb, s));
  if (!full_norms(p, nranks)) {
    SPAMM_NCCL_TRY(ncclGroupStart());
    for (int q = 0; q < nranks; ++q) {
      const int64_t a0 = share(p.BM, q, nranks), a1 = share(p.BM, q + 1, nranks);
      const int64_t b0 = share(p.BN, q, nranks), b1 = share(p.BN, q + 1, nranks);
      if (a1 > a0)
        SPAMM_NCCL_TRY(ncclBroadcast(p.nA + a0 * p.BK, p.nA + a0 * p.BK, static_cast<size_t>((a1 - a0) * p.BK),
                                     ncclFloat64, q, comm, s));
      if (b1 > b0)
        SPAMM_NCCL_TRY(ncclBroadcast(p.nBt + b0 * p.BK, p.nBt + b0 * p.BK,
                                     static_cast<size_t>((b1 - b0) * p.BK), ncclFloat64, q, comm, s));
    }
    SPAMM_NCCL_TRY(ncclGroupEnd());
  }
  // 2. provisional skip map and its row work, all-reduced
  SPAMM_TRY(phase_provisional(p, rank, nranks, s));
  if (nranks > 1)
    SPAMM_NCCL_TRY(ncclAllReduce(p.row_work, p.row_work, static_cast<size_t>(p.BM), ncclInt64, ncclSum, comm, s));
  // 3. device partition, the final range's skip map and multiply
  SPAMM_TRY(phase_final(p, rank, nranks, A, lda, B, ldb, C, ldc, s));
  // 4. optional C all-gather (row blocks owned by each rank; sizes from the device cut)
  if ((flags & SPAMM_MGPU_GATHER_C) && nranks > 1) {
    std::vector<int64_t> rows;
    SPAMM_TRY(rank_rows(p, nranks, rows));
    SPAMM_NCCL_TRY(ncclGroupStart());
    for (int q = 0; q < nranks; ++q) {
      if (rows[q + 1] <= rows[q]) continue;
      float* base = C + rows[q] * ldc;
      const size_t cnt = static_cast<size_t>((rows[q + 1] - rows[q] - 1) * ldc + p.N);
      SPAMM_NCCL_TRY(ncclBroadcast(base, base, cnt, ncclFloat32, q, comm, s));
    }
    SPAMM_NCCL_TRY(ncclGroupEnd());
  }
  return SPAMM_OK;
}

spamm_status spamm_multiply_mgpu_local(spamm_plan_t* plans, int nranks, const void* A, int64_t lda, const void* B,
                                       int64_t ldb, float* const* C, int64_t ldc, uint32_t flags, void* stream) {
  if (!plans || !C) return fail(SPAMM_E_INVALID, "NULL argument");
  if (nranks <= 0) return fail(SPAMM_E_INVALID, "bad nranks");
  if (flags & ~(SPAMM_MGPU_INPUTS_ON_ROOT | SPAMM_MGPU_GATHER_C)) return fail(SPAMM_E_INVALID, "unknown flag");
  std::vector<Plan*> P(nranks);
  for (int q = 0; q < nranks; ++q) {
    if (!plans[q] || !C[q]) return fail(SPAMM_E_INVALID, "NULL plan or C");
    P[q] = reinterpret_cast<Plan*>(plans[q]);
    SPAMM_TRY(check_common(*P[q], nranks));
    if (P[q]->M != P[0]->M || P[q]->N != P[0]->N || P[q]->K != P[0]->K || P[q]->prec != P[0]->prec ||
        P[q]->device != P[0]->device || P[q]->tau != P[0]->tau)
      return fail(SPAMM_E_INVALID, "plans differ in shape, precision, tau or device");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Plan& p0 = *P[0];
  // 1. norms per rank; "all-gather": copy rank q's slices into every other plan
  for (int q = 0; q < nranks; ++q) SPAMM_TRY(phase_norms(*P[q], q, nranks, A, lda, B, ldb, s));
  if (!full_norms(p0, nranks)) {
    for (int q = 0; q < nranks; ++q) {
      const int64_t a0 = share(p0.BM, q, nranks), a1 = share(p0.BM, q + 1, nranks);
      const int64_t b0 = share(p0.BN, q, nranks), b1 = share(p0.BN, q + 1, nranks);
      for (int r = 0; r < nranks; ++r) {
        if (r == q) continue;
        if (a1 > a0)
          SPAMM_CUDA_TRY(cudaMemcpyAsync(P[r]->nA + a0 * p0.BK, P[q]->nA + a0 * p0.BK,
                                         sizeof(double) * static_cast<size_t>((a1 - a0) * p0.BK),
                                         cudaMemcpyDeviceToDevice, s));
        if (b1 > b0)
          SPAMM_CUDA_TRY(cudaMemcpyAsync(P[r]->nBt + b0 * p0.BK, P[q]->nBt + b0 * p0.BK,
                                         sizeof(double) * static_cast<size_t>((b1 - b0) * p0.BK),
                                         cudaMemcpyDeviceToDevice, s));
      }
    }
  }
  // 2. provisional skip maps; "all-reduce" of the row work through rank 0's buffer
  for (int q = 0; q < nranks; ++q) SPAMM_TRY(phase_provisional(*P[q], q, nranks, s));
  if (nranks > 1) {
    const unsigned blocks = static_cast<unsigned>((p0.BM + 255) / 256);
    for (int q = 1; q < nranks; ++q) add_i64_kernel<<<blocks, 256, 0, s>>>(p0.row_work, P[q]->row_work, p0.BM);
    count_launch(nranks - 1);
    SPAMM_CUDA_TRY(cudaGetLastError());
    for (int q = 1; q < nranks; ++q)
      SPAMM_CUDA_TRY(cudaMemcpyAsync(P[q]->row_work, p0.row_work, sizeof(int64_t) * static_cast<size_t>(p0.BM),
                                     cudaMemcpyDeviceToDevice, s));
  }
  // 3. partition, final skip maps, multiplies
  for (int q = 0; q < nranks; ++q) SPAMM_TRY(phase_final(*P[q], q, nranks, A, lda, B, ldb, C[q], ldc, s));
  // 4. "all-gather" of C rows
  if ((flags & SPAMM_MGPU_GATHER_C) && nranks > 1) {
    std::vector<int64_t> rows;
    SPAMM_TRY(rank_rows(p0, nranks, rows));
    for (int q = 0; q < nranks; ++q) {
      if (rows[q + 1] <= rows[q]) continue;
      for (int r = 0; r < nranks; ++r)
        if (r != q)
          SPAMM_CUDA_TRY(cudaMemcpy2DAsync(C[r] + rows[q] * ldc, ldc * 4, C[q] + rows[q] * ldc, ldc * 4, p0.N * 4,
                                           static_cast<size_t>(rows[q + 1] - rows[q]), cudaMemcpyDeviceToDevice, s));
    }
  }
  return SPAMM_OK;
}

}  // extern "C"
