/*
 * spamm.h -- C ABI of libspamm.so, the B200 (sm_100a) hot path of SpAMM / cuSpAMM.
 *
 * The method (arXiv 2103.13042, /root/reference/PAPER.md):
 *   C ~= A*B where a tile pair (i,k,j) is multiplied only if
 *   ||A[i,k]||_F * ||B[k,j]||_F >= tau                       (Alg. 1 l.7/10 PAPER.md:63,
 *                                                              Alg. 2 l.5 PAPER.md:155)
 *   with tiles of LoNum x LoNum elements, LoNum = 32          (Table 1 pins 32)
 *   and the flat two-kernel semantics of Sec. 3.1:
 *     stage 1  spamm_norms          tile Frobenius norms, Eq. 2
 *     stage 2  spamm_build_skipmap  per-C-tile surviving k-lists
 *     stage 3  spamm_multiply       C[i,j] = sum_{kept k} A[i,k]B[k,j], alpha=1, beta=0
 *                                   by default (spamm_set_scalars: C = alpha*SpAMM + beta*C)
 *   Multi-GPU row partitioning of C (Sec. 3.4, Alg. 4): spamm_multiply_mgpu.
 *
 * Conventions (every entry point):
 *   - Returns spamm_status. Nothing throws or aborts across the ABI. On error a
 *     thread-local message is available from spamm_last_error().
 *   - Matrix arguments are DEVICE pointers owned by the caller, row-major, with
 *     explicit leading dimensions in ELEMENTS.  Requirements: pointer 16-byte
 *     aligned and ld*sizeof(elem) a multiple of 16 (TMA), ld >= number of columns.
 *     A host pointer returns SPAMM_E_INVALID (checked with cudaPointerGetAttributes).
 *   - Element types: SPAMM_FP32 -> float A, B (CUDA-core FP32 multiply);
 *     SPAMM_FP32X3 -> float A, B (tensor cores on a 3 x bfloat16 split, FP32-accurate);
 *     SPAMM_BF16 / SPAMM_FP16 -> 16-bit A, B (tcgen05 tensor cores, FP32 accumulate).
 *     C is always float (ab_frag is FP32).
 *   - Ragged sizes are allowed: the result equals zero padding to a multiple of
 *     the tile, done by TMA out-of-bounds fill, never a physical pad.
 *   - Everything is stream-ordered on the caller's stream (a cudaStream_t passed
 *     as void*; NULL = legacy default stream).  Argument errors are reported
 *     synchronously; asynchronous CUDA faults surface as SPAMM_E_CUDA on a later call.
 *   - The plan OWNS its workspace (norm maps, skip map, schedules).  Pointers
 *     returned by getters stay valid until the next mutating call on the plan or
 *     spamm_plan_destroy().  A plan is not thread-safe; use one plan per stream.
 *   - There is no CPU fallback and no alternative backend: an unsupported
 *     combination returns SPAMM_E_UNSUPPORTED.
 */
#ifndef SPAMM_H_
#define SPAMM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SPAMM_OK = 0,
  SPAMM_E_INVALID = 1,      /* bad argument (size, pointer, alignment, NaN tau, ...) */
  SPAMM_E_UNSUPPORTED = 2,  /* valid but not implemented (e.g. tile != 32)            */
  SPAMM_E_CUDA = 3,         /* CUDA runtime / driver error                            */
  SPAMM_E_NOMEM = 4,        /* device allocation failed                               */
  SPAMM_E_NCCL = 5,         /* NCCL error in the multi-GPU path                       */
  SPAMM_E_STATE = 6         /* call order violated (e.g. multiply before norms)       */
} spamm_status;

typedef enum {
  SPAMM_FP32 = 0,  /* float inputs, CUDA-core FP32 FMA, two-level FP32 accumulation */
  SPAMM_BF16 = 1,  /* bfloat16 inputs, tcgen05.mma kind::f16, FP32 accumulation in TMEM */
  SPAMM_FP16 = 2,  /* float16 inputs, same tensor-core path as BF16 */
  SPAMM_FP32X3 = 3 /* float inputs on the tensor cores: spamm_norms also
                      splits A and B into three bfloat16 planes a = a0 + a1 + a2 (plan-owned,
                      6 bytes per element), the multiply sums the six products a0b0 + a0b1 +
                      a1b0 + a0b2 + a1b1 + a2b0 per kept pair with two-level FP32 accumulation
                      (TMEM partials of 4 k-steps added in registers).  FP32-level accuracy;
                      same norms, tau semantics and skip map as SPAMM_FP32. */
} spamm_precision;

/* plan flags */
#define SPAMM_FLAG_NONE           0u
#define SPAMM_FLAG_TIMING         1u  /* record per-stage CUDA events (spamm_get_stats) */
#define SPAMM_FLAG_LARGE_TILES    2u  /* BF16/FP16: always schedule 256 x 256 macro-tiles (8 x 8 C tiles,
                                         two MMA issuers per SM).  Without it, problems with fewer such
                                         tiles than SMs whose 128 x 128 tiles fit one wave use 128 x 128
                                         macro-tiles (4 x 4 C tiles) so that more SMs work; results agree
                                         up to FP32 rounding order. */
#define SPAMM_FLAG_STAGED         4u  /* never fuse the skip map into the multiply.  Without it, spamm_run /
                                         SPAMM_MUL_AUTO on a plan with 128 x 128 macro-tiles (BF16/FP16 of
                                         the small-problem rule above, SPAMM_FP32, SPAMM_FP32X3) of at most one per
                                         SM skip the stage-2 launch: each multiply CTA decides its own
                                         macro-tile's list with the same predicate and writes the same
                                         skip map (getters unchanged), then multiplies it.  Results are
                                         identical either way. */

/* spamm_multiply flags */
#define SPAMM_MUL_AUTO            1u  /* run spamm_norms + spamm_build_skipmap first (spamm_run) */

#define SPAMM_MUL_OUTPUT_NORMS    2u  /* spamm_multiply_chain: also write the tile norms of the result */
#define SPAMM_MUL_LOW_ONLY        4u  /* spamm_multiply_chain: C_low is the only output (no FP32 C is
                                         written or read; C may be NULL; needs beta = 0) */

/* spamm_multiply_mgpu flags (Sec. 3.4) */
#define SPAMM_MGPU_INPUTS_REPLICATED 0u  /* every rank already holds full A and B           */
#define SPAMM_MGPU_INPUTS_ON_ROOT    1u  /* rank 0 holds A and B; broadcast over NCCL first */
#define SPAMM_MGPU_GATHER_C          2u  /* all-gather C rows so every rank holds full C     */

typedef struct spamm_plan_s* spamm_plan_t;

typedef struct {
  int64_t M, N, K;            /* problem shape (C is M x N, inner dimension K)              */
  int64_t BM, BK, BN;         /* tiles per dimension: ceil(M/tile), ceil(K/tile), ceil(N/tile) */
  int32_t tile;               /* LoNum                                                      */
  int32_t macro_i, macro_j;   /* C tiles per scheduling macro-tile (rows, cols)             */
  int64_t kept;               /* kept (i,k,j) triples = sum V                */
  int64_t macro_entries;      /* (k, mask) entries over all macro-tiles = MMA k-steps       */
  double  valid_ratio;        /* kept / (BM*BK*BN)                          */
  double  tau;
  float   ms_norms, ms_skipmap, ms_multiply; /* last stage times if SPAMM_FLAG_TIMING, else -1 */
  int32_t precision;          /* spamm_precision                                            */
  int32_t row_begin, row_end; /* tile rows this plan multiplies (multi-GPU shard), [begin,end) */
} spamm_stats;

/* ---------------------------------------------------------------- plans --- */

/* Square N x N problem ("square matrices N x N", alpha=1, beta=0).
 * tile must be 32 (LoNum; other values -> SPAMM_E_UNSUPPORTED).
 * tau >= 0 and finite (NaN / negative / inf -> SPAMM_E_INVALID).
 * Allocates the plan's device workspace on the current device.
 * Ownership: *p is owned by the caller and released with spamm_plan_destroy. */
spamm_status spamm_plan(spamm_plan_t* p, int64_t N, int32_t tile, double tau, spamm_precision prec);

/* Rectangular C(M x N) = A(M x K) * B(K x N), e.g. the im2col shapes of PAPER.md:338.
 * flags: SPAMM_FLAG_*.  Same rules as spamm_plan. */
spamm_status spamm_plan_ex(spamm_plan_t* p, int64_t M, int64_t N, int64_t K, int32_t tile, double tau,
                           spamm_precision prec, uint32_t flags);

/* Releases all device memory of the plan (synchronises the device). NULL is a no-op. */
spamm_status spamm_plan_destroy(spamm_plan_t p);

/* Change tau without recomputing norms; invalidates the skip map (the
 * search re-evaluates the threshold on fixed norm maps). */
spamm_status spamm_set_tau(spamm_plan_t p, double tau);

/* -------------------------------------------------------------- stages --- */

/* Stage 1 (Sec. 3.2, Eq. 2): tile Frobenius norms of A (M x K)
 * and B (K x N) into plan-owned float64 maps nA[BM][BK] and nB^T[BN][BK]
 * (nB stored transposed so both maps are contiguous along k).  Each norm is the
 * float64 sum of squares of the tile in a fixed, tile-position-independent order,
 * then sqrt.  A and B are read exactly once (HBM-bound). */
spamm_status spamm_norms(spamm_plan_t p, const void* A, int64_t lda, const void* B, int64_t ldb,
                         void* stream);

/* Stage 2 (Alg. 2 lines 3-16; Sec. 3.5.1):
 * keep(i,k,j) <=> !(nA[i][k] * nB[k][j] < tau) in float64 (NaN kept).  Builds
 *   macro lists: per macro-tile of macro_i x macro_j C tiles, the union of kept k in
 *               ascending order with a keep bit per C tile (the complete skip map), the
 *               tensor path's pre-decoded MMA runs, and an LPT schedule;
 *   row_work[i] = sum_j V[i][j];  kept / macro-entry totals.
 * Output-sensitive: a norm pyramid (max and min of the norms over each macro row / column and
 * 32 k-tiles; one quadtree level of Eq. 1) decides whole chunks of k exactly
 * (all skipped / all kept) and only the remaining chunks test their products one by one.
 * The per-C-tile view (V, ascending k lists) is expanded from the macro lists on request
 * (spamm_get_skipmap / spamm_get_counts).  Requires spamm_norms on this plan (else
 * SPAMM_E_STATE).  Stream-ordered, no host synchronisation. */
spamm_status spamm_build_skipmap(spamm_plan_t p, void* stream);

/* Stage 3 (Sec. 3.3, Alg. 2/3): C[i,j] = sum over kept k, ascending,
 * of A[i,k] * B[k,j] for every C tile (tiles with no kept k are written as 0).
 * A, B must be the same arrays given to spamm_norms (not checked).  C (float, M x N,
 * ldc) is overwritten (beta = 0).  flags: SPAMM_MUL_AUTO runs stages 1 and 2 first.
 * Without AUTO, requires spamm_build_skipmap (else SPAMM_E_STATE). */
spamm_status spamm_multiply(spamm_plan_t p, const void* A, int64_t lda, const void* B, int64_t ldb,
                            float* C, int64_t ldc, uint32_t flags, void* stream);

/* All three stages, stream-ordered, no host synchronisation (== multiply with AUTO; small
 * problems fuse stages 2 and 3, SPAMM_FLAG_STAGED). */
spamm_status spamm_run(spamm_plan_t p, const void* A, int64_t lda, const void* B, int64_t ldb,
                       float* C, int64_t ldc, void* stream);

/* ------------------------------------------------------------ multi-GPU --- */

/* NCCL bootstrap helpers: rank 0 calls spamm_nccl_unique_id, the 128-byte id is
 * broadcast by the caller (e.g. torch.distributed), then every rank calls
 * spamm_nccl_comm_init on its own device.  The comm is owned by the caller. */
spamm_status spamm_nccl_unique_id(uint8_t out_id[128]);
spamm_status spamm_nccl_comm_init(void** comm, int nranks, int rank, const uint8_t id[128]);
spamm_status spamm_nccl_comm_destroy(void* comm);

/* Pure host function: contiguous split of BM tile rows into nranks ranges balanced by
 * row_work (prefix sums cut at multiples of total/nranks; Sec. 3.5.1 load balance,
 * PAPER.md:230-234, applied to the row partition of Sec. 3.4).
 * row_begin has nranks+1 entries, row_begin[0]=0, row_begin[nranks]=BM, non-decreasing. */
spamm_status spamm_partition_rows(const int64_t* row_work, int64_t BM, int nranks, int64_t* row_begin);

/* Row-partitioned SpAMM over nranks GPUs of one node (Sec. 3.4, Alg. 4):
 *   1. (INPUTS_ON_ROOT) ncclBroadcast of A and B from rank 0 into the caller's buffers;
 *   2. each rank norms its share of A's tile rows and B's tile columns (FP32X3: all of them,
 *      its split planes are operands); grouped ncclBroadcasts all-gather the maps;
 *   3. each rank builds the skip map of its provisional (even) macro-row share, which yields
 *      that share's row work; ncclAllReduce of the row work;
 *   4. a one-CTA kernel cuts macro rows at equal shares of the total work with the rule of
 *      spamm_partition_rows (identical on every rank, decided on the device: no host sync);
 *      each rank completes the skip map of its final rows and multiplies them into C rows;
 *   5. (GATHER_C) C rows are exchanged so every rank holds all of C (this step reads the cut
 *      back to the host: one stream synchronisation).
 * A, B, C are full-size device buffers on every rank (only this rank's rows of C are
 * written unless GATHER_C).  comm: ncclComm_t from spamm_nccl_comm_init.  At most 64 ranks;
 * chained outputs are single-GPU (SPAMM_E_UNSUPPORTED).  The partition is readable with
 * spamm_get_partition (synchronises). */
spamm_status spamm_multiply_mgpu(spamm_plan_t p, void* nccl_comm, int rank, int nranks,
                                 const void* A, int64_t lda, const void* B, int64_t ldb,
                                 float* C, int64_t ldc, uint32_t flags, void* stream);

/* The same nranks-rank computation emulated on ONE GPU for verification (the survey's P4
 * invariant: multi-rank C and skip maps equal single-GPU ones): plans[q] plays rank q (all
 * plans of the same shape, precision, tau and device), C[q] is rank q's full-size C buffer.
 * Phases and kernels are exactly those of spamm_multiply_mgpu; only the transport differs --
 * the collectives are device copies between the plans' buffers on `stream`, in rank order.
 * flags: SPAMM_MGPU_GATHER_C as above (INPUTS_ON_ROOT is a no-op: the ranks share A and B). */
spamm_status spamm_multiply_mgpu_local(spamm_plan_t* plans, int nranks, const void* A, int64_t lda,
                                       const void* B, int64_t ldb, float* const* C, int64_t ldc,
                                       uint32_t flags, void* stream);

/* General update C = alpha * SpAMM(A, B, tau) + beta * C (the problem statement's alpha and
 * beta) for every later spamm_multiply / spamm_run /
 * spamm_multiply_mgpu of this plan.  Defaults alpha = 1, beta = 0.  Applied in the multiply
 * epilogue in FP32: C = fmaf(alpha, P, beta * C_old); with beta == 0 the old C is never read
 * (BLAS convention: NaN there does not propagate).  Tiles without kept pairs get beta * C_old.
 * alpha, beta must be finite (else SPAMM_E_INVALID). */
spamm_status spamm_set_scalars(spamm_plan_t p, double alpha, double beta);

/* ---------------------------------------------------------- chained SpAMM --- */
/* chains such as matrix powers X <- X*X (ergo's density-matrix purification,
 * PAPER.md:320) without re-reading C to norm it.  spamm_multiply_chain is spamm_multiply
 * (flags SPAMM_MUL_AUTO as there) whose epilogue additionally
 *   - with C_low != NULL (BF16/FP16 plans only; device, row-major, leading dimension ldcl in
 *     elements): writes C rounded (RNE) to the plan's input type -- the next product's operand;
 *   - with SPAMM_MUL_OUTPUT_NORMS: writes the float64 tile norms of the written result into a
 *     plan-owned map nC[BM][BN] (Eq. 2 of the values stored: C, or C_low's rounded values when
 *     given -- reading R4), readable with spamm_get_output_norms;
 *   - with SPAMM_MUL_LOW_ONLY (BF16/FP16 plans, C_low required, beta = 0): C_low is the only
 *     output -- no FP32 C is stored (C may be NULL), halving the output traffic.
 * FP32X3 plans return SPAMM_E_UNSUPPORTED. */
spamm_status spamm_multiply_chain(spamm_plan_t p, const void* A, int64_t lda, const void* B, int64_t ldb,
                                  float* C, int64_t ldc, void* C_low, int64_t ldcl, uint32_t flags,
                                  void* stream);

/* Device pointer to nC[BM][BN] (row-major float64) of the last spamm_multiply_chain with
 * SPAMM_MUL_OUTPUT_NORMS (else SPAMM_E_STATE). */
spamm_status spamm_get_output_norms(spamm_plan_t p, const double** d_nC);

/* Stage 1 from given maps instead of the matrices: nA[BM][BK] and nB[BK][BN] (row-major float64
 * device arrays, e.g. another plan's output norms) are copied into the plan (nB transposed), which
 * then behaves as after spamm_norms.  Stream-ordered.  FP32X3 plans: SPAMM_E_UNSUPPORTED (their
 * norm stage also splits the inputs). */
spamm_status spamm_set_norms(spamm_plan_t p, const double* nA, const double* nB, void* stream);

/* ------------------------------------------------------- convolution drop-in --- */
/* a convolution layer as the SpAMM of its im2col
 * GEMM, Y = SpAMM(W, im2col(X), tau).  X: [batch][C_in][H][Wd] (NCHW, contiguous, the plan's input
 * type: float for FP32/FP32X3 plans, bf16/fp16 otherwise); W: [C_out][C_in*kh*kw] row-major
 * (leading dimension ldw), the plan's A; Y: [C_out][batch*Ho*Wo] float row-major (ldy), column
 * (n*Ho + y)*Wo + x, Ho = (H + 2 pad - kh)/stride + 1 (Wo likewise).  im2col row index
 * (ci*kh + ky)*kw + kx; out-of-image taps are 0.  The plan must have M = C_out, K = C_in*kh*kw,
 * N = batch*Ho*Wo (else SPAMM_E_INVALID).  A device kernel writes im2col(X) into plan-owned storage
 * (allocated on the first call), then the three stages run as spamm_run.  Stream-ordered. */
spamm_status spamm_conv2d_im2col(spamm_plan_t p, const void* W, int64_t ldw, const void* X, int64_t batch,
                                 int64_t C_in, int64_t H, int64_t Wd, int32_t kh, int32_t kw, int32_t stride,
                                 int32_t pad, float* Y, int64_t ldy, void* stream);

/* ------------------------------------------------------------ tau search --- */

/* Number of kept triples at tau, i.e. #{(i,k,j) : !(nA[i][k] * nB[k][j] < tau)} in float64
 * over all BM*BK*BN triples, from the plan's norm maps without building
 * a skip map.  Requires spamm_norms (else SPAMM_E_STATE); tau finite and >= 0 (else
 * SPAMM_E_INVALID).  Synchronises `stream` once; *kept is host memory. */
spamm_status spamm_count_kept(spamm_plan_t p, double tau, int64_t* kept, void* stream);

/* Sec. 3.5.2: search tau for a target valid ratio `target` (fraction in
 * [0,1]).  ave = mean of nA[i][k]*nB[k][j] over all BM*BK*BN triples (R17);
 * tau = ave, bracket [0, k*ave] with k = 1 and k incremented while vr(k*ave) > target;
 * bisection at the midpoint; stop when |vr - target| < tol (absolute, R16; the
 * paper uses 0.01) or after max_iter evaluations.  Every vr evaluation is one count kernel
 * (as spamm_count_kept) and one stream synchronisation.  Outputs (host memory): *tau, and
 * if non-NULL *valid_ratio = vr(*tau), *iters = evaluations of the main loop.  The plan's
 * tau is set to *tau and its skip map invalidated (call spamm_build_skipmap next).
 * Requires spamm_norms (else SPAMM_E_STATE); bad target/tol/max_iter -> SPAMM_E_INVALID. */
spamm_status spamm_tau_search(spamm_plan_t p, double target, double tol, int32_t max_iter,
                              double* tau, double* valid_ratio, int32_t* iters, void* stream);

/* -------------------------------------------------------- introspection --- */

/* Device pointers to the float64 norm maps: dA = nA[BM][BK], dBt = nB^T[BN][BK]. */
spamm_status spamm_get_norms(spamm_plan_t p, const double** dA, const double** dBt,
                             int64_t* BM, int64_t* BK, int64_t* BN);

/* Device pointers to the per-C-tile k lists: tile_start[BM*BN] (int64) and k_idx[kept]
 * (uint16); tile t's list is k_idx[tile_start[t] .. tile_start[t] + V[t]).
 * *kept is read back (synchronises). */
spamm_status spamm_get_skipmap(spamm_plan_t p, const int64_t** d_tile_start, const uint16_t** d_k_idx,
                               int64_t* kept);

/* Device pointers to V[BM*BN] (int64) and row_work[BM] (int64). */
spamm_status spamm_get_counts(spamm_plan_t p, const int64_t** d_V, const int64_t** d_row_work);

/* Device pointers to the macro lists: macro-tile t = I*GN+J owns the entries
 * [start[t], start[t] + count[t]) (start, count int64[GM*GN]); an entry is the pair
 * (uint32 k, uint32 mask), k ascending, bit (li*macro_j + lj) = keep of C tile
 * (I*macro_i+li, J*macro_j+lj); order[GM*GN] (int32) = LPT schedule (descending count;
 * order within equal counts unspecified). */
spamm_status spamm_get_macro(spamm_plan_t p, const int64_t** d_start, const int64_t** d_count,
                             const uint32_t** d_entries, const int32_t** d_order, int64_t* GM, int64_t* GN);

/* Tile-row range of the last multi-GPU partition (nranks+1 entries, host memory). */
spamm_status spamm_get_partition(spamm_plan_t p, int64_t* row_begin, int nranks);

/* Counters and last stage times (synchronises the plan's last stream). */
spamm_status spamm_get_stats(spamm_plan_t p, spamm_stats* out);

const char* spamm_status_string(spamm_status s);
const char* spamm_last_error(void);

/* Number of tcgen05 / SIMT / norm / skip-map kernel launches issued by this process
 * (for the bench's gpu_launches accounting). */
int64_t spamm_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SPAMM_H_ */
