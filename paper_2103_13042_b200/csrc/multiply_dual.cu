// multiply_dual.cu -- stage 3, BF16/FP16 tensor-core path on 256 x 256 macro-tiles with two MMA
// issuers:
//   C[i,j] = sum_{kept k, ascending} A[i,k] * B[k,j]   (Alg. 2/3),
// BF16/FP16 inputs, FP32 accumulation in TMEM (PAPER.md:187's FP32 accumulator fragment).
//
// Why 256 x 256 (round 1; the 128 x 256 kernel has since been removed): at the bench point it moved 1.50 GB of operand tiles
// L2 -> SMEM per call (24 KB per 32-deep k-step for 2 MMAs of N = 256); ncu shows the SM <-> L2
// request path busy 68 % of the kernel, i.e. the kernel is fed at ~12 TB/s (the chip's TMA
// throughput, B300_MICROARCH.md "TMA chip-throughput").  A 256 x 256 macro-tile (8 x 8 C tiles)
// reuses every B[32 x 256] box for 256 rows of A: 32 KB per k-step for 4 MMAs, 1.05 GB per call
// (-30 %), with the same tensor-pipe work (the skip semantics are per C tile, unchanged).
//
// One CTA per SM (384 threads), all 512 TMEM columns = two FP32 accumulators of 128 x 256:
//   warp 0 (lane 0): tile claims (atomic counter over the LPT order) and the A boxes
//            [128 x 32] of the halves that have runs (K-major SWIZZLE_64B, rows 128h..);
//   warp 3 (lane 0): the contiguous range of needed B[32 x 32] boxes (3-D stacked map);
//   warps 1, 2 (one elected lane): MMA issuer of half h = warp - 1 (C-tile rows 4h .. 4h+3): per run of
//            adjacent C-tile columns with the same row pattern, 2 x tcgen05.mma M=128 N=32*run
//            K=16 whose disable-output-lane mask switches off the skipped C-tile rows -- the
//            4 x 8 run encoding of skipmap.cu (encode_runs), one per half.  Two independent issuers
//            on one tensor pipe hide each other's per-k-step bookkeeping (scripts/probe_queue2);
//   warps 4-11: epilogue, warp w drains rows 128h + 32q .. +32 (h = (w-4)/4, q = w%4, its
//            TMEM lane quadrant) x 256 columns; they zero-fill the macro-tiles without kept
//            pairs (the LPT tail) with evict-first bulk stores of a 1 KB zero buffer -- after
//            their last tile, and while waiting for an accumulator when empty tiles dominate.
// Skip map: 8 x 8 macro-tiles; macro_run holds two uint4 per k-step (half 0, half 1), each the
// 4 x 8 encoding of skipmap.cu encode_runs, at 2 * (t * BK + e) + h.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.h"
#include "sm100.cuh"

namespace spamm {
namespace {

using namespace sm100;

constexpr int kDASlot = 256 * 32 * 2;                 // A[256 x 32] as two [128 x 32] SW64 boxes
constexpr int kDBSlot = 32 * 256 * 2;                 // B[32 x 256] as eight [32 x 32] boxes
constexpr int kDStepBytes = kDASlot + kDBSlot;        // one 32-deep k-step
constexpr int kDThreads = 384;   // w0 A/claims, w1-2 MMA, w3 B, w4-11 epilogue
constexpr int kDTQ = 4;                               // tile ring depth
// kPack = 2 k-steps of one macro-tile per ring stage (one wait / commit per stage for the issuers;
// measured 174 -> 165 us against one per stage, r01e); the ring holds 6 k-steps (192 KB)
constexpr int kPack = 2;
constexpr int kDStages = 6 / kPack;
constexpr int kDStageBytes = kPack * kDStepBytes;
// align slack, stages, zero atom, barriers + entry batches + tile ring
constexpr size_t kDSmem = 1024 + static_cast<size_t>(kDStages) * kDStageBytes + 1024 + 4096;

constexpr uint32_t kFullRun = 0u | (7u << 3) | (15u << 6);
constexpr uint32_t kFirst = 1u << 29, kLast = 1u << 30, kNoStep = 1u << 28, kEnd = 1u << 27;
// stage holds k-steps k, k+1 as 64-deep boxes: A [128 x 64] SW128 per half, B [64 x 32] per column
constexpr uint32_t kWideSt = 1u << 25;

struct DTile {
  int64_t t, e0, e1;   // macro-tile, k-step range [e0, e1) (in k-steps, entry pairs)
};

// warp-uniform copy of lane 0's value (lets the compiler keep MMA operands in uniform registers)
__device__ __forceinline__ uint4 bcast4(uint4 v) {
  v.x = __shfl_sync(0xffffffffu, v.x, 0);
  v.y = __shfl_sync(0xffffffffu, v.y, 0);
  v.z = __shfl_sync(0xffffffffu, v.z, 0);
  v.w = __shfl_sync(0xffffffffu, v.w, 0);
  return v;
}

struct DMaps {
  CUtensorMap a1;      // A [128 x 32] boxes, SW64
  CUtensorMap a2;      // A [128 x 64] boxes, SW128 (a stage of two consecutive k-steps)
  CUtensorMap b1[4];   // B stacked [32 k x 32 n] boxes, 8/4/2/1 boxes, SW64
  CUtensorMap b2[4];   // B stacked [64 k x 32 n] boxes (two consecutive k-steps), SW64
  CUtensorMap b2d1, b2d2;   // N % 32 != 0: plain 2-D B boxes [32 | 64 k x 32 n], SW64
};

struct DChain {
  double* nC;
  int64_t ldn;
  void* clow;
  int64_t ldl;
  int low_only;   // SPAMM_MUL_LOW_ONLY: C_low is the only output (no FP32 C stores)
};

template <uint32_t kFmt, bool kGen>
__global__ void __launch_bounds__(kDThreads, 1)
    spamm_mul_dual_kernel(const __grid_constant__ DMaps mp, const int64_t* __restrict__ mstart,
                          const int64_t* __restrict__ mcount, const uint4* __restrict__ ment,
                          const int32_t* __restrict__ order, int64_t n_tiles,
                          const int64_t* __restrict__ rng, const int64_t* __restrict__ n_empty_p, int64_t GN,
                          float* __restrict__ C, int64_t ldc, int64_t M, int64_t N, unsigned int* __restrict__ sched,
                          const Axpby ab, const DChain co, unsigned long long* __restrict__ prof, int use3d) {
  // claims follow the skip map's order (skipmap.cu order_pass: LPT for few tiles per CTA, ascending
  // first kept k for many); the tiles without kept pairs come last and are zero-filled by the
  // epilogue warps (plain epilogue), or go through the pipeline (n_empty_p == nullptr)
  constexpr int wide_ok = 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sZero = smem + kDStages * kDStageBytes;    // 1 KB zeros: MMA zero atom, bulk zero-fill source
  uint64_t* full = reinterpret_cast<uint64_t*>(sZero + 1024);
  uint64_t* empty = full + kDStages;
  uint64_t* tfull = empty + kDStages;                 // [2] per half
  uint64_t* tempty = tfull + 2;                       // [2]
  uint64_t* tq_full = tempty + 2;
  uint64_t* tq_empty = tq_full + kDTQ;
  uint4* srun = reinterpret_cast<uint4*>(tq_empty + kDTQ);   // [kDStages][kPack][2 halves]
  uint4* sent = srun + 2 * kPack * kDStages;                          // [64] producer A entry batch
  uint4* sentB = sent + 64;                                   // [64] producer B entry batch
  DTile* tq = reinterpret_cast<DTile*>(sentB + 64);           // [kDTQ]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq + kDTQ);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // profiling timeline (globaltimer ns): [0] CTA start [1] prologue done [2] issuer 0 done
  // [3] epilogue warp 4 last drain done [4] its zero-fill done [5] CTA end
  unsigned long long* tl = prof ? prof + 1024 * 16 + blockIdx.x * 8 : nullptr;
  auto stamp = [&](int i) {
    unsigned long long g_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));
    tl[i] = g_;
  };
  if (tl && threadIdx.x == 0) stamp(0);
  for (int i = threadIdx.x; i < 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sZero)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);         // both issuers release a stage
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&tfull[h], 1);
      mbar_init(&tempty[h], 4);        // the 4 epilogue warps of the half
    }
    for (int q = 0; q < kDTQ; ++q) {
      mbar_init(&tq_full[q], 1);
      mbar_init(&tq_empty[q], 1 + 8);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  if (tl && threadIdx.x == 0) stamp(1);
  pdl_wait();      // the skip map (order, lists, counts) and the claim counters are ready
  pdl_trigger();
  if (rng != nullptr) n_tiles = (rng[1] - rng[0]) * GN;   // multi-GPU: range decided on the device
  const int64_t n_empty = n_empty_p ? *n_empty_p : 0;
  const int64_t n_work = n_tiles - n_empty;

  // Zero-fill of the macro-tiles without kept pairs (the LPT tail of `order`): an epilogue warp
  // claims 32-row units (32 KB of C) from a global counter -- while its accumulator half is not
  // ready (interleaved, below) and after its CTA's last tile -- so the CTAs that finish their MMA
  // work early absorb it (the slowest one takes none).  Done greedily at the start instead, the
  // 141 MB of zero writes at N = 8192 compete with the operand loads' first DRAM touches
  // (multiply 165 vs 152 us without them).
  const int64_t n_units = n_empty * 8;
#ifndef SPAMM_ZF_INTERLEAVE
#define SPAMM_ZF_INTERLEAVE 1
#endif
  const uint64_t zf_pol = l2_policy_evict_first();   // zeros are never re-read: keep the operands in L2
  // Interleaved with the accumulator waits only when the empty tiles dominate (measured, ms of the
  // multiply, zero-fill last -> interleaved: N = 16384 lambda 0.99 tau 1e-6 0.343 -> 0.318 (3.5 empty
  // tiles per working tile), N = 8192 0.135 -> 0.141 (1.2), N = 65536 58.8 -> 59.0; scripts/gpu_r02zi.sh)
#ifndef SPAMM_ZF_RATIO
#define SPAMM_ZF_RATIO 2
#endif
#ifndef SPAMM_ZF_LSU
#define SPAMM_ZF_LSU 0
#endif
  const bool zf_inter = SPAMM_ZF_INTERLEAVE && n_empty >= SPAMM_ZF_RATIO * n_work;
  // interleaved units with 16-byte LSU stores instead of the bulk-copy engine (experiment
  // SPAMM_ZF_LSU=1, scripts/gpu_r02zr.sh: multiply at N = 16384 0.321 -> 0.338 ms, N = 8192 0.135 ->
  // 0.142 ms when always interleaved -- slower than the bulk stores, not used)
  auto zero_unit_lsu = [&]() -> bool {
    unsigned int u32 = 0;
    if (lane == 0) u32 = atomicAdd(sched + 1, 1u);
    const int64_t u = __shfl_sync(0xffffffffu, u32, 0);
    if (u >= n_units) return false;
    const int64_t t = order[n_work + u / 8];
    const int64_t r0 = (t / GN) * 256 + (u % 8) * 32, c0 = (t % GN) * 256;
    const int64_t ncol = N - c0 < 256 ? N - c0 : 256;
    for (int r = 0; r < 32; ++r) {
      const int64_t row = r0 + r;
      if (row >= M) break;
      float* crow = C + row * ldc + c0;
      for (int64_t cc = 4 * lane; cc < ncol; cc += 128) {
        if (cc + 4 <= ncol) st_zero16_hint(crow + cc, zf_pol);
        else
          for (int64_t x = cc; x < ncol; ++x) crow[x] = 0.f;
      }
    }
    return true;
  };
  auto zero_unit = [&]() -> bool {
    unsigned int u32 = 0;
    if (lane == 0) u32 = atomicAdd(sched + 1, 1u);
    const int64_t u = __shfl_sync(0xffffffffu, u32, 0);
    if (u >= n_units) return false;
    const int64_t t = order[n_work + u / 8];
    const int64_t row = (t / GN) * 256 + (u % 8) * 32 + lane, c0 = (t % GN) * 256;
    const int64_t ncol = N - c0 < 256 ? N - c0 : 256;
    const uint32_t bytes = static_cast<uint32_t>(ncol * 4) & ~15u;
    if (row < M) {   // one row per lane: 32 bulk (TMA-engine) stores of the 1 KB zero buffer
      if (bytes) bulk_store_1d_hint(C + row * ldc + c0, sZero, bytes, zf_pol);
      for (int64_t cc = bytes / 4; cc < ncol; ++cc) C[row * ldc + c0 + cc] = 0.f;
    }
    bulk_commit_group();
    return true;
  };
  if (warp == 0) {
    // ------------------------------------------------- producer A: tile claims, srun, A boxes
    if (lane == 0) {
      tma_prefetch_desc(&mp.a1);
      tma_prefetch_desc(&mp.a2);
    }
    int s = 0;
    uint32_t ph = 0;
    int tq_s = 0;
    uint32_t tq_ph = 0;
    auto claim = [&]() -> DTile {
      DTile d{-1, 0, 0};
      unsigned int idx = 0;
      if (lane == 0) idx = atomicAdd(sched, 1u);
      idx = __shfl_sync(0xffffffffu, idx, 0);
      if (static_cast<int64_t>(idx) < n_work) {
        d.t = order[idx];
        d.e0 = mstart[d.t];
        d.e1 = d.e0 + mcount[d.t];
      }
      return d;
    };
    // A tile is claimed when the previous one's loads have all been issued, not when it starts:
    // claiming ahead assigns the LPT tail by start time instead of by finish time (the ring's
    // three stages of issued loads hide the claim's latency).
    DTile cur = claim();
    for (;;) {
      if (lane == 0) {
        mbar_wait(&tq_empty[tq_s], tq_ph ^ 1);
        tq[tq_s] = cur;
        mbar_arrive(&tq_full[tq_s]);
      }
      if (++tq_s == kDTQ) {
        tq_s = 0;
        tq_ph ^= 1;
      }
      if (cur.t < 0 || cur.e1 == cur.e0) {   // end of stream, or a tile without k-steps (C = 0)
        if (lane == 0) {
          mbar_wait(&empty[s], ph ^ 1);
          const uint32_t fl = cur.t < 0 ? kEnd : (kFirst | kLast | kNoStep);
          for (int j = 0; j < 2 * kPack; ++j) srun[2 * kPack * s + j] = make_uint4(0, 0, 0, fl);
          mbar_arrive(&full[s]);
        }
        if (++s == kDStages) {
          s = 0;
          ph ^= 1;
        }
        if (cur.t < 0) break;
        cur = claim();
        continue;
      }
      const int32_t I = static_cast<int32_t>(cur.t / GN);
      for (int64_t eb = cur.e0; eb < cur.e1; eb += 32) {
        const int cnt = static_cast<int>(cur.e1 - eb < 32 ? cur.e1 - eb : 32);
        if (lane < cnt) {
          sent[2 * lane] = ment[2 * (eb + lane)];
          sent[2 * lane + 1] = ment[2 * (eb + lane) + 1];
        }
        __syncwarp();
        {   // whole warp, warp-uniform values (see the issuers); one elected lane issues
          auto X = [&](int e) -> uint32_t { return __shfl_sync(0xffffffffu, sent[e].x, 0); };
          for (int q = 0; q < cnt; q += kPack) {
            // (batches hold 32 k-steps, a multiple of kPack: a stage never spans two batches,
            // and only a tile's last stage can be partly empty)
            const int np = cnt - q < kPack ? cnt - q : kPack;
            // two consecutive k-tiles: one 64-deep box per A half and per B column range
            const bool wide = wide_ok && kPack == 2 && np == 2 &&
                              (X(2 * q + 2) & 0xFFFFu) == (X(2 * q) & 0xFFFFu) + 1u;
            uint32_t tx = 0;
            if (wide) {
              const uint32_t x00 = X(2 * q), x01 = X(2 * q + 1), x10 = X(2 * q + 2), x11 = X(2 * q + 3);
              const uint32_t cols = (x00 | x01 | x10 | x11) >> 24;
              const int c0 = __ffs(cols) - 1, len = (32 - __clz(cols)) - c0;
              const bool h0 = ((x00 | x10) >> 16) & 15u, h1 = ((x01 | x11) >> 16) & 15u;
              tx = 16384u * ((h0 ? 1u : 0u) + (h1 ? 1u : 0u)) + 4096u * len;
            } else {
              for (int j = 0; j < np; ++j) {
                const uint32_t x0 = X(2 * (q + j)), x1 = X(2 * (q + j) + 1);
                const uint32_t cols = (x0 >> 24) | (x1 >> 24);
                const int c0 = __ffs(cols) - 1, len = (32 - __clz(cols)) - c0;
                tx += 8192u * ((((x0 >> 16) & 15u) != 0u ? 1u : 0u) + (((x1 >> 16) & 15u) != 0u ? 1u : 0u)) + 2048u * len;
              }
            }
            const uint32_t fl = (eb + q == cur.e0 ? kFirst : 0u) | (eb + q + np == cur.e1 ? kLast : 0u) |
                                (wide ? kWideSt : 0u);
            mbar_wait(&empty[s], ph ^ 1);
            const bool leader = elect_one();
            for (int j = 0; j < kPack && leader; ++j) {
              uint4 e0 = make_uint4(0, 0, 0, 0), e1 = make_uint4(0, 0, 0, 0);
              if (j < np) {
                e0 = sent[2 * (q + j)];
                e1 = sent[2 * (q + j) + 1];
              }
              if (j == 0) {   // the stage's flags live in its first k-step's entries
                e0.w |= fl;
                e1.w |= fl;
              }
              srun[2 * (kPack * s + j)] = e0;
              srun[2 * (kPack * s + j) + 1] = e1;
            }
            if (elect_one()) mbar_arrive_expect_tx(&full[s], tx);
            if (wide) {
              const uint32_t x00 = X(2 * q), x01 = X(2 * q + 1), x10 = X(2 * q + 2), x11 = X(2 * q + 3);
              const int32_t k0 = static_cast<int32_t>(x00 & 0xFFFFu) * 32;
              uint8_t* adst = smem + s * kDStageBytes;
              if (elect_one()) {
                if (((x00 | x10) >> 16) & 15u) tma_load_2d(adst, &mp.a2, &full[s], k0, I * 256);
                if (((x01 | x11) >> 16) & 15u) tma_load_2d(adst + 16384, &mp.a2, &full[s], k0, I * 256 + 128);
              }
            } else {
              for (int j = 0; j < np; ++j) {
                const uint32_t x0 = X(2 * (q + j)), x1 = X(2 * (q + j) + 1);
                const int32_t k0 = static_cast<int32_t>(x0 & 0xFFFFu) * 32;
                uint8_t* adst = smem + s * kDStageBytes + j * kDStepBytes;
                if (elect_one()) {
                  if ((x0 >> 16) & 15u) tma_load_2d(adst, &mp.a1, &full[s], k0, I * 256);
                  if ((x1 >> 16) & 15u) tma_load_2d(adst + 8192, &mp.a1, &full[s], k0, I * 256 + 128);
                }
              }
            }
            if (++s == kDStages) {
              s = 0;
              ph ^= 1;
            }
          }
        }
        __syncwarp();
      }
      cur = claim();
    }
  } else if (warp == 3) {
    // ---------------------------------------------------------------- producer B
    if (lane == 0)
      for (int q = 0; q < 4 && use3d; ++q) {
        tma_prefetch_desc(&mp.b1[q]);
        tma_prefetch_desc(&mp.b2[q]);
      }
    if (lane == 0 && !use3d) {
      tma_prefetch_desc(&mp.b2d1);
      tma_prefetch_desc(&mp.b2d2);
    }
    int s = 0;
    uint32_t ph = 0;
    int tq_s = 0;
    uint32_t tq_ph = 0;
    for (;;) {
      mbar_wait(&tq_full[tq_s], tq_ph);
      const DTile cur = tq[tq_s];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tq_empty[tq_s]);
      if (++tq_s == kDTQ) {
        tq_s = 0;
        tq_ph ^= 1;
      }
      if (cur.t < 0) break;
      if (cur.e1 == cur.e0) {
        if (++s == kDStages) {
          s = 0;
          ph ^= 1;
        }
        continue;
      }
      const int32_t jb = static_cast<int32_t>(cur.t % GN) * 8;
      for (int64_t eb = cur.e0; eb < cur.e1; eb += 32) {
        const int cnt = static_cast<int>(cur.e1 - eb < 32 ? cur.e1 - eb : 32);
        if (lane < cnt) {
          sentB[2 * lane] = ment[2 * (eb + lane)];
          sentB[2 * lane + 1] = ment[2 * (eb + lane) + 1];
        }
        __syncwarp();
        {   // whole warp, warp-uniform values; one elected lane issues
          auto X = [&](int e) -> uint32_t { return __shfl_sync(0xffffffffu, sentB[e].x, 0); };
          for (int q = 0; q < cnt; q += kPack) {
            const int np = cnt - q < kPack ? cnt - q : kPack;
            const bool wide = wide_ok && kPack == 2 && np == 2 && (X(2 * q + 2) & 0xFFFFu) == (X(2 * q) & 0xFFFFu) + 1u;
            mbar_wait(&empty[s], ph ^ 1);
            if (wide) {
              const uint32_t cols = (X(2 * q) | X(2 * q + 1) | X(2 * q + 2) | X(2 * q + 3)) >> 24;
              const int32_t k0 = static_cast<int32_t>(X(2 * q) & 0xFFFFu) * 32;
              uint8_t* bdst = smem + s * kDStageBytes + 2 * kDASlot;
              const int c0 = __ffs(cols) - 1, len = (32 - __clz(cols)) - c0;
              if (elect_one()) {
                if (!use3d) {   // N % 32 != 0: one 2-D box per column tile (zero fill past N)
                  for (int c = c0; c < c0 + len; ++c)
                    tma_load_2d(bdst + c * 4096, &mp.b2d2, &full[s], (jb + c) * 32, k0);
                } else if (len == 8) {
                  tma_load_3d(bdst, &mp.b2[0], &full[s], 0, k0, jb);
                } else {
                  int off = c0;
                  if (len & 4) { tma_load_3d(bdst + off * 4096, &mp.b2[1], &full[s], 0, k0, jb + off); off += 4; }
                  if (len & 2) { tma_load_3d(bdst + off * 4096, &mp.b2[2], &full[s], 0, k0, jb + off); off += 2; }
                  if (len & 1) { tma_load_3d(bdst + off * 4096, &mp.b2[3], &full[s], 0, k0, jb + off); }
                }
              }
            }
            for (int j = 0; j < (wide ? 0 : np); ++j) {
              const uint32_t x0 = X(2 * (q + j)), x1 = X(2 * (q + j) + 1);
              const uint32_t cols = (x0 >> 24) | (x1 >> 24);
              const int32_t k0 = static_cast<int32_t>(x0 & 0xFFFFu) * 32;
              uint8_t* bdst = smem + s * kDStageBytes + j * kDStepBytes + kDASlot;
              const int c0 = __ffs(cols) - 1, len = (32 - __clz(cols)) - c0;
              if (elect_one()) {
                if (!use3d) {
                  for (int c = c0; c < c0 + len; ++c)
                    tma_load_2d(bdst + c * 2048, &mp.b2d1, &full[s], (jb + c) * 32, k0);
                } else if (len == 8) {
                  tma_load_3d(bdst, &mp.b1[0], &full[s], 0, k0, jb);
                } else {
                  int off = c0;
                  if (len & 4) { tma_load_3d(bdst + off * 2048, &mp.b1[1], &full[s], 0, k0, jb + off); off += 4; }
                  if (len & 2) { tma_load_3d(bdst + off * 2048, &mp.b1[2], &full[s], 0, k0, jb + off); off += 2; }
                  if (len & 1) { tma_load_3d(bdst + off * 2048, &mp.b1[3], &full[s], 0, k0, jb + off); }
                }
              }
            }
            if (++s == kDStages) {
              s = 0;
              ph ^= 1;
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1 || warp == 2) {
    // ------------------------------------------------------------ MMA issuer of half h
    const int h = warp - 1;
    // The whole warp runs the loop on broadcast (warp-uniform) values and one elected lane issues
    // each tcgen05 op: with uniform operands the compiler moves them to uniform registers with a
    // plain R2UR, where a lane-0-only loop gets an ELECT/R2UR.BROADCAST/BRA.U.ANY waterfall per MMA.
    {
      constexpr uint32_t idesc_base = idesc_f16(kFmt, 128, 0, 0, 1);
      constexpr uint32_t idesc_full = idesc_base | (8u << 19);   // N = 256
      const uint32_t base_addr = smem_u32(smem);
      const uint32_t srun_addr = smem_u32(srun) + 16u * static_cast<uint32_t>(h);
      const uint64_t zdesc = smem_desc(smem_u32(sZero), 0, 0, kLayoutSW64);   // all strides 0: the zero atom
      const uint32_t dcol = tbase + 256u * static_cast<uint32_t>(h);
      uint32_t ph = 0;
      uint32_t tile_par = 0;
      bool fin = false;
      unsigned long long c_full = 0, c_te = 0, c_mma = 0, c_cm = 0, n_st = 0, c_head = 0, n_tiles_done = 0;
      int st_in_tile = 0;
      const unsigned long long c_start = clock64();
      while (!fin) {
#pragma unroll 1
        for (int st = 0; st < kDStages; ++st) {
          const unsigned long long ta = prof ? clock64() : 0;
          mbar_wait(&full[st], ph);
          if (prof) {
            const unsigned long long dw = clock64() - ta;
            c_full += dw;
            if (st_in_tile < 3) c_head += dw;
            ++st_in_tile;
          }
          tc_fence_after();
          uint4 rs;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(rs.x), "=r"(rs.y), "=r"(rs.z), "=r"(rs.w)
                       : "r"(srun_addr + st * (32 * kPack)));
          rs = bcast4(rs);
          const uint32_t fl = rs.w;
          if (fl & kEnd) {
            fin = true;
            break;
          }
          if (fl & kFirst) {
            const unsigned long long tb = prof ? clock64() : 0;
            mbar_wait(&tempty[h], tile_par);   // phase 0 = the epilogue's initial arrival
            if (prof) c_te += clock64() - tb;
            tc_fence_after();
            if (elect_one()) umma_f16(dcol, zdesc, zdesc, idesc_full, 0u, 0u, 0u, 0u, 0u);   // D = 0
          }
          const unsigned long long tc = prof ? clock64() : 0;
#pragma unroll
          for (int j = 0; j < kPack; ++j) {
            if (j > 0) {
              asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(rs.x), "=r"(rs.y), "=r"(rs.z), "=r"(rs.w)
                           : "r"(srun_addr + st * (32 * kPack) + 32 * j));
              rs = bcast4(rs);
            }
            const uint32_t nr = (rs.x >> 16) & 15u;
            if ((fl & kNoStep) || nr == 0u) continue;
            // 32-deep slots: A K-major SW64 rows of 32 (SBO 512), +32 B per K=16, half h at +8 KB;
            //   B MN-major SW64 boxes of 32 columns x 32 k (LBO = 2048), +1024 B per K=16.
            // wide stage (k-steps k, k+1): A SW128 rows of 64 (SBO 1024), half h at +16 KB, k-step j
            //   at +64 B; B boxes of 32 columns x 64 k (LBO = 4096) after 32 KB of A, k-step j at +2 KB.
            const bool wst = (fl & kWideSt) != 0u;
            const uint32_t st_addr = base_addr + st * kDStageBytes;
            const uint64_t ad = wst ? smem_desc(st_addr + 16384u * static_cast<uint32_t>(h), 16, 1024, kLayoutSW128) + 4u * j
                                    : smem_desc(st_addr + j * kDStepBytes + 8192u * static_cast<uint32_t>(h), 16, 512, kLayoutSW64);
            const uint64_t bd = wst ? smem_desc(st_addr + 2 * kDASlot, 4096, 512, kLayoutSW64) + 128u * j
                                    : smem_desc(st_addr + j * kDStepBytes + kDASlot, 2048, 512, kLayoutSW64);
            const uint32_t bbox = wst ? 256u : 128u;   // descriptor units (16 B) per column box
            if (nr == 1u && rs.y == kFullRun) {
              if (elect_one()) {
                umma_f16(dcol, ad, bd, idesc_full, 1u, 0u, 0u, 0u, 0u);
                umma_f16(dcol, ad + 2, bd + 64, idesc_full, 1u, 0u, 0u, 0u, 0u);
              }
            } else {
              uint32_t cw = rs.y;
              for (uint32_t rr = 0; rr < nr; ++rr) {
                if (rr == 3) cw = rs.z;
                if (rr == 6) cw = rs.w;
                const uint32_t w = cw & 0x3FFu;
                cw >>= 10;
                const uint32_t j0 = w & 7u, len = ((w >> 3) & 7u) + 1u, pat = w >> 6;
                const uint32_t idesc = idesc_base | (len << 19);
                const uint32_t m0 = (pat & 1u) - 1u, m1 = ((pat >> 1) & 1u) - 1u;   // 0 keep, ~0 disable
                const uint32_t m2 = ((pat >> 2) & 1u) - 1u, m3 = ((pat >> 3) & 1u) - 1u;
                const uint64_t bj = bd + static_cast<uint64_t>(j0 * bbox);
                const uint32_t d = dcol + j0 * 32u;
                if (elect_one()) {
                  umma_f16(d, ad, bj, idesc, 1u, m0, m1, m2, m3);
                  umma_f16(d, ad + 2, bj + 64, idesc, 1u, m0, m1, m2, m3);
                }
              }
            }
          }
          const unsigned long long td = prof ? clock64() : 0;
          if (elect_one()) umma_commit(&empty[st]);
          if (fl & kLast) {
            if (elect_one()) umma_commit(&tfull[h]);
            tile_par ^= 1;
            st_in_tile = 0;
            ++n_tiles_done;
          }
          if (prof) {
            const unsigned long long te = clock64();
            c_mma += td - tc;
            c_cm += te - td;
            ++n_st;
          }
        }
        ph ^= 1;
      }
      if (prof && lane == 0) {
        unsigned long long* pr = prof + blockIdx.x * 16 + h * 6;
        pr[0] = clock64() - c_start;
        if (h == 0) stamp(2);
        pr[1] = c_full;
        pr[2] = c_te;
        pr[3] = c_mma;
        pr[4] = c_cm;
        pr[5] = n_st;
        if (h == 0) {
          prof[blockIdx.x * 16 + 13] = c_head;
          prof[blockIdx.x * 16 + 14] = n_tiles_done;
          unsigned int smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          prof[blockIdx.x * 16 + 15] = smid;
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // --------------------------------------------------------------------- epilogue
    const int q = warp & 3;              // TMEM lane quadrant
    const int h = (warp - 4) >> 2;       // accumulator half (C rows 128h ..)
    if (lane == 0) mbar_arrive(&tempty[h]);   // the accumulator starts empty
    const int t0 = lane & 3, t1 = lane >> 2;
    int tq_s = 0;
    uint32_t tq_ph = 0;
    uint32_t par = 0;
    for (;;) {
      mbar_wait(&tq_full[tq_s], tq_ph);
      const DTile cur = tq[tq_s];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tq_empty[tq_s]);
      if (++tq_s == kDTQ) {
        tq_s = 0;
        tq_ph ^= 1;
      }
      if (cur.t < 0) break;
      const int64_t I = cur.t / GN, J = cur.t % GN;
      const unsigned long long tw = prof ? clock64() : 0;
      if (zf_inter && !kGen) {
        // while this half's accumulator is not ready, zero-fill units of the macro-tiles without
        // kept pairs (evict-first bulk stores); the phase is monotone, so any lane seeing it
        // complete means complete for the warp (zero_unit is warp-collective)
        while (!__any_sync(0xffffffffu, mbar_try_wait(&tfull[h], par))) {
          if (!(SPAMM_ZF_LSU ? zero_unit_lsu() : zero_unit())) break;
        }
      }
      mbar_wait(&tfull[h], par);
      par ^= 1;
      if (prof && warp == 4 && lane == 0) prof[blockIdx.x * 16 + 12] += clock64() - tw;
      tc_fence_after();
      const uint32_t tq_addr = tbase + 256u * static_cast<uint32_t>(h);
      if constexpr (kGen) {
        double tsum[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};   // C tiles (I*8 + 4h + q, J*8 + c)
#pragma unroll 1
        for (int hh = 0; hh < 8; ++hh) {
          const int lh = hh & 1;
          const int c0 = (hh >> 1) * 64;
          uint32_t v[32];
          tmem_ld_16x256b_x8(tq_addr + ((static_cast<uint32_t>(q * 32 + 16 * lh)) << 16) + c0, v);
          tmem_wait_ld();
          const int64_t ra = I * 256 + h * 128 + q * 32 + 16 * lh + t1;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int64_t col = J * 256 + c0 + 8 * i + 2 * t0;
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
              const int64_t row = ra + 8 * rr;
              if (row >= M || col >= N) continue;
              float* cp = C + row * ldc + col;
              float2 x = make_float2(__uint_as_float(v[4 * i + 2 * rr]), __uint_as_float(v[4 * i + 2 * rr + 1]));
              const bool two = col + 1 < N;
              if (co.low_only) {   // alpha only (beta = 0 is required): no FP32 C exists
                x = make_float2(ab.alpha * x.x, two ? ab.alpha * x.y : 0.f);
              } else if (two) {
                x = axpby2(ab, x, cp);
                __stcs(reinterpret_cast<float2*>(cp), x);
              } else {
                x.x = axpby1(ab, x.x, cp);
                x.y = 0.f;
                *cp = x.x;
              }
              if (co.clow != nullptr) {   // round to the input type; norms of what is stored (R4)
                if (kFmt == 1) {
                  __nv_bfloat16* lp = static_cast<__nv_bfloat16*>(co.clow) + row * co.ldl + col;
                  const __nv_bfloat16 l0 = __float2bfloat16_rn(x.x), l1 = __float2bfloat16_rn(x.y);
                  lp[0] = l0;
                  if (two) lp[1] = l1;
                  x = make_float2(__bfloat162float(l0), __bfloat162float(l1));
                } else {
                  __half* lp = static_cast<__half*>(co.clow) + row * co.ldl + col;
                  const __half l0 = __float2half_rn(x.x), l1 = __float2half_rn(x.y);
                  lp[0] = l0;
                  if (two) lp[1] = l1;
                  x = make_float2(__half2float(l0), __half2float(l1));
                }
              }
              const double d0 = x.x, d1 = two ? static_cast<double>(x.y) : 0.0;
              tsum[(hh >> 1) * 2 + (i >> 2)] += d0 * d0 + d1 * d1;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[h]);
        if (co.nC != nullptr) {
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            double x = tsum[t];
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            const int64_t ti = I * 8 + h * 4 + q, tj = J * 8 + t;
            if (lane == 0 && ti * 32 < M && tj * 32 < N) co.nC[ti * co.ldn + tj] = sqrt(x);
          }
        }
      } else {
#pragma unroll 1
      for (int hh = 0; hh < 8; ++hh) {
        const int lh = hh & 1;                // lanes [16*lh, 16*lh + 16) of the quadrant
        const int c0 = (hh >> 1) * 64;        // 64-column block
        uint32_t v[32];
        tmem_ld_16x256b_x8(tq_addr + ((static_cast<uint32_t>(q * 32 + 16 * lh)) << 16) + c0, v);
        tmem_wait_ld();
        if (hh == 7) {   // the whole accumulator slice is in registers: release it early
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[h]);
        }
        const int64_t ra = I * 256 + h * 128 + q * 32 + 16 * lh + t1, rb = ra + 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int64_t col = J * 256 + c0 + 8 * i + 2 * t0;
          float* ca = C + ra * ldc + col;
          float* cb = C + rb * ldc + col;
          float2 pa = make_float2(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]));
          float2 pb = make_float2(__uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
          if (col + 1 < N) {
            if (ra < M) __stcs(reinterpret_cast<float2*>(ca), pa);
            if (rb < M) __stcs(reinterpret_cast<float2*>(cb), pb);
          } else if (col < N) {
            if (ra < M) *ca = pa.x;
            if (rb < M) *cb = pb.x;
          }
        }
      }
      }
    }
    if (tl && warp == 4 && lane == 0) stamp(3);
    while (zero_unit()) {
    }
    bulk_wait_group<0>();   // zero-fill stores complete before the CTA retires
    if (tl && warp == 4 && lane == 0) stamp(4);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tbase);
  if (tl && threadIdx.x == 0) stamp(5);
}

#ifdef SPAMM_PROFILE
// per-CTA issuer counters and a globaltimer timeline (compile with -DSPAMM_PROFILE)
static void print_profile(const unsigned long long* hp, int grid) {
  double a[16] = {0};
  double mx = 0, mn = 1e30;
  for (int c = 0; c < grid; ++c) {
    for (int k = 0; k < 16; ++k) a[k] += static_cast<double>(hp[c * 16 + k]) / grid;
    mx = std::max(mx, static_cast<double>(hp[c * 16]));
    mn = std::min(mn, static_cast<double>(hp[c * 16]));
  }
  for (int h = 0; h < 2; ++h)
    fprintf(stderr, "[dual prof] issuer %d cycles/CTA %.0f (min %.0f max %.0f): full-wait %.0f tmem-empty %.0f "
            "mma %.0f commit %.0f stages %.0f\n", h, a[6 * h], mn, mx, a[6 * h + 1], a[6 * h + 2], a[6 * h + 3],
            a[6 * h + 4], a[6 * h + 5]);
  fprintf(stderr, "[dual prof] epilogue warp 4 tmem-full wait %.0f; issuer 0 full-wait in a tile's first 3 stages %.0f\n",
          a[12], a[13]);
  const unsigned long long* t = hp + 1024 * 16;
  unsigned long long g0 = ~0ull;
  for (int c = 0; c < grid; ++c) g0 = std::min(g0, t[c * 8]);
  double m[6] = {0}, mxs[6] = {0};
  for (int c = 0; c < grid; ++c)
    for (int k = 0; k < 6; ++k) {
      const double v = (static_cast<double>(t[c * 8 + k]) - static_cast<double>(g0)) * 1e-3;
      m[k] += v / grid;
      mxs[k] = std::max(mxs[k], v);
    }
  fprintf(stderr, "[dual tl] us from first CTA start (mean / max): start %.1f/%.1f prologue %.1f/%.1f issuer-done %.1f/%.1f "
          "last-drain %.1f/%.1f zero-fill-done %.1f/%.1f cta-end %.1f/%.1f\n", m[0], mxs[0], m[1], mxs[1], m[2], mxs[2],
          m[3], mxs[3], m[4], mxs[4], m[5], mxs[5]);
}
#endif

template <uint32_t kFmt, bool kGen>
spamm_status launch_dual_t(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                           cudaStream_t s, CUtensorMapDataType dt) {
  DMaps mp;
  std::memset(&mp, 0, sizeof(mp));
  SPAMM_TRY(encode_tmap_2d(&mp.a1, dt, 2, A, p.K, p.M, lda, 32, 128, CU_TENSOR_MAP_SWIZZLE_64B));
  SPAMM_TRY(encode_tmap_2d(&mp.a2, dt, 2, A, p.K, p.M, lda, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B));
  const uint32_t nbs[4] = {8, 4, 2, 1};
  if (p.N % 32 == 0) {   // stacked 3-D maps need whole 32-column boxes
    for (int q = 0; q < 4; ++q) {
      SPAMM_TRY(encode_tmap_3d(&mp.b1[q], dt, B, 32, p.K, p.N / 32, static_cast<uint64_t>(ldb) * 2, 64, 32, 32, nbs[q],
                               CU_TENSOR_MAP_SWIZZLE_64B));
      SPAMM_TRY(encode_tmap_3d(&mp.b2[q], dt, B, 32, p.K, p.N / 32, static_cast<uint64_t>(ldb) * 2, 64, 32, 64, nbs[q],
                               CU_TENSOR_MAP_SWIZZLE_64B));
    }
  } else {
    SPAMM_TRY(encode_tmap_2d(&mp.b2d1, dt, 2, B, p.N, p.K, ldb, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B));
    SPAMM_TRY(encode_tmap_2d(&mp.b2d2, dt, 2, B, p.N, p.K, ldb, 32, 64, CU_TENSOR_MAP_SWIZZLE_64B));
  }
  auto kern = spamm_mul_dual_kernel<kFmt, kGen>;
  SPAMM_SET_SMEM(kern, static_cast<int>(kDSmem), p.device);
  // range: host-known for single-GPU calls, decided on the device for the multi-GPU partition
  const int64_t n_tiles = p.range_on_device ? 0 : (p.row_end_macro - p.row_begin_macro) * p.GN;
  if (!p.range_on_device && n_tiles <= 0) return SPAMM_OK;
  // the LPT order ends with the macro-tiles without kept pairs (hist[0] of them); with the
  // plain epilogue the epilogue warps zero-fill those, otherwise they go through the pipeline
  // (beta * C_old, chained norms)
  const int grid = static_cast<int>(!p.range_on_device && n_tiles < p.num_sms ? n_tiles : p.num_sms);
  if (!p.sched_zeroed) SPAMM_CUDA_TRY(cudaMemsetAsync(p.sched, 0, 2 * sizeof(unsigned int), s));
  p.sched_zeroed = false;
  unsigned long long* prof = nullptr;
#ifdef SPAMM_PROFILE
  static unsigned long long* prof_buf = nullptr;
  if (!prof_buf) cudaMalloc(&prof_buf, 1024 * 24 * 8);
  prof = prof_buf;
  cudaMemsetAsync(prof, 0, 1024 * 24 * 8, s);
#endif
  SPAMM_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(kDThreads), kDSmem, s, mp, static_cast<const int64_t*>(p.mstart),
                            static_cast<const int64_t*>(p.U), static_cast<const uint4*>(p.macro_run),
                            static_cast<const int32_t*>(p.order), n_tiles,
                            static_cast<const int64_t*>(p.range_on_device ? p.d_range : nullptr),
                            static_cast<const int64_t*>(kGen ? nullptr : p.totals + 2), p.GN, C, ldc, p.M, p.N, p.sched,
                            Axpby{static_cast<float>(p.alpha), static_cast<float>(p.beta)},
                            DChain{p.out_norms ? p.nC : nullptr, p.BN, p.out_low, p.out_ldl, p.out_low_only ? 1 : 0},
                            prof, p.N % 32 == 0 ? 1 : 0));
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
#ifdef SPAMM_PROFILE
  static unsigned long long hp[1024 * 24];
  cudaMemcpyAsync(hp, prof, sizeof(hp), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  print_profile(hp, grid);
#endif
  return SPAMM_OK;
}

}  // namespace

spamm_status launch_multiply_dual(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C,
                                  int64_t ldc, cudaStream_t s) {
  const bool gen = p.alpha != 1.0 || p.beta != 0.0 || p.out_norms || p.out_low != nullptr;
  const CUtensorMapDataType dt = p.prec == SPAMM_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  if (p.prec == SPAMM_BF16)
    return gen ? launch_dual_t<1, true>(p, A, lda, B, ldb, C, ldc, s, dt) : launch_dual_t<1, false>(p, A, lda, B, ldb, C, ldc, s, dt);
  return gen ? launch_dual_t<0, true>(p, A, lda, B, ldb, C, ldc, s, dt) : launch_dual_t<0, false>(p, A, lda, B, ldb, C, ldc, s, dt);
}

}  // namespace spamm
