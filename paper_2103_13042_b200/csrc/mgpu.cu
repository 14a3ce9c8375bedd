// mgpu.cu -- multi-GPU SpAMM over NCCL (Sec. 3.4, Alg. 4) with the
// load-balance idea of Sec. 3.5.1 applied to the row partition.
//
// The paper row-partitions C evenly and moves data with Unified-Memory page faults
// (PAPER.md:211).  Here: one process per GPU; inputs are broadcast over NVLink by NCCL
// when only the root holds them; each rank norms 1/n of A's tile rows and of B's tile
// columns and the maps are all-gathered (instead of every GPU recomputing B's map,
// Alg. 4 lines 4-6); kept-pair counts of provisional row blocks are all-reduced and
// C macro-rows (128 rows) are cut at equal shares of the work; each rank then emits
// the skip map of its rows and multiplies them.  C rows are all-gathered on request.
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.h"

namespace spamm {

spamm_status do_norms_range(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t ar0,
                            int64_t ar1, int64_t bj0, int64_t bj1, cudaStream_t s);
spamm_status do_skipmap(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s);
spamm_status do_multiply(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                         cudaStream_t s);

static spamm_status nccl_fail(ncclResult_t r, const char* where) {
  return fail(SPAMM_E_NCCL, std::string(where) + ": " + ncclGetErrorString(r));
}
#define SPAMM_NCCL_TRY(expr)                                     \
  do {                                                           \
    ncclResult_t _r = (expr);                                    \
    if (_r != ncclSuccess) return ::spamm::nccl_fail(_r, #expr); \
  } while (0)

static inline int64_t share(int64_t n, int r, int nr) { return n * r / nr; }

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
  Plan& p = *reinterpret_cast<Plan*>(h);
  if (p.prec == SPAMM_FP32X3 && nranks > 1)   // its split planes come from full-range norms
    return fail(SPAMM_E_UNSUPPORTED, "SPAMM_FP32X3 is single-GPU in this build");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
  const size_t es = f32_inputs(p.prec) ? 4 : 2;

  // 1. inputs from the root (Alg. 4 lines 4 and 7: B to every GPU, A rows)
  if ((flags & SPAMM_MGPU_INPUTS_ON_ROOT) && nranks > 1) {
    SPAMM_NCCL_TRY(ncclGroupStart());
    SPAMM_NCCL_TRY(ncclBroadcast(A, const_cast<void*>(A), static_cast<size_t>((p.M - 1) * lda + p.K) * es,
                                 ncclUint8, 0, comm, s));
    SPAMM_NCCL_TRY(ncclBroadcast(B, const_cast<void*>(B), static_cast<size_t>((p.K - 1) * ldb + p.N) * es,
                                 ncclUint8, 0, comm, s));
    SPAMM_NCCL_TRY(ncclGroupEnd());
  }

  // 2. norms of this rank's A tile rows and B tile columns, then all-gather (grouped broadcasts)
  const int64_t ar0 = share(p.BM, rank, nranks), ar1 = share(p.BM, rank + 1, nranks);
  const int64_t bj0 = share(p.BN, rank, nranks), bj1 = share(p.BN, rank + 1, nranks);
  SPAMM_TRY(do_norms_range(p, A, lda, B, ldb, ar0, ar1, bj0, bj1, s));
  if (nranks > 1) {
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

  // 3. work-balanced macro-row partition from all-reduced row work
  std::vector<int64_t> cut(nranks + 1);
  if (nranks > 1) {
    const int64_t g0 = share(p.GM, rank, nranks), g1 = share(p.GM, rank + 1, nranks);
    SPAMM_TRY(launch_skipmap_count(p, g0, g1, s));
    SPAMM_NCCL_TRY(ncclAllReduce(p.row_work, p.row_work, static_cast<size_t>(p.BM), ncclInt64, ncclSum, comm, s));
    std::vector<int64_t> rw(p.BM), mw(p.GM, 0);
    SPAMM_CUDA_TRY(cudaMemcpyAsync(rw.data(), p.row_work, sizeof(int64_t) * p.BM, cudaMemcpyDeviceToHost, s));
    SPAMM_CUDA_TRY(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < p.BM; ++i) mw[i / p.MI] += rw[i];
    SPAMM_TRY(spamm_partition_rows(mw.data(), p.GM, nranks, cut.data()));
  } else {
    cut[0] = 0;
    cut[1] = p.GM;
  }
  p.last_partition.assign(nranks + 1, 0);
  for (int q = 0; q <= nranks; ++q) p.last_partition[q] = std::min<int64_t>(cut[q] * p.MI, p.BM);

  // 4. this rank's skip map and multiply
  SPAMM_TRY(do_skipmap(p, cut[rank], cut[rank + 1], s));
  SPAMM_TRY(do_multiply(p, A, lda, B, ldb, C, ldc, s));

  // 5. optional C all-gather (row blocks owned by each rank)
  if ((flags & SPAMM_MGPU_GATHER_C) && nranks > 1) {
    SPAMM_NCCL_TRY(ncclGroupStart());
    for (int q = 0; q < nranks; ++q) {
      const int64_t r0 = std::min<int64_t>(cut[q] * p.MI * kTile, p.M);
      const int64_t r1 = std::min<int64_t>(cut[q + 1] * p.MI * kTile, p.M);
      if (r1 <= r0) continue;
      float* base = C + r0 * ldc;
      const size_t cnt = static_cast<size_t>((r1 - r0 - 1) * ldc + p.N);
      SPAMM_NCCL_TRY(ncclBroadcast(base, base, cnt, ncclFloat32, q, comm, s));
    }
    SPAMM_NCCL_TRY(ncclGroupEnd());
  }
  return SPAMM_OK;
}

}  // extern "C"
