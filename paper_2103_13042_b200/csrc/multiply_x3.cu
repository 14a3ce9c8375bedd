// multiply_x3.cu -- stage 3 for SPAMM_FP32X3: FP32 inputs on the tensor cores (SURVEY.md
// §8(f) f2), same skip semantics as every path: C[i,j] = sum_{kept k, ascending} A[i,k]B[k,j]
// (PAPER.md:127), C in FP32.
//
// Each FP32 input is split by the norm stage into three bfloat16 planes, a = a0 + a1 + a2
// (a0 = rn(a), a1 = rn(a - a0), a2 = rn(a - a0 - a1); exact to ~2^-24 |a|).  A kept tile
// pair contributes the six products whose order is at most 2^-16 relative to a0 b0:
//   a0b0 + a0b1 + a1b0 + a0b2 + a1b1 + a2b0      (dropped: a1b2, a2b1 ~2^-24, a2b2 ~2^-32)
// so every product is FP32-accurate.  Accumulation is two-level: the tensor core's FP32
// accumulator in TMEM only ever sums 4 k-steps (6 x 2 MMAs each); the epilogue adds the
// chunk partials into a per-thread FP32 running sum with IEEE adds, alternating between two
// TMEM buffers so the next chunk's MMAs overlap the add.  (A single TMEM accumulation over
// thousands of MMAs drifts by ~2^-24 per MMA: measured 4e-5 at K = 16384 on the BF16 path.)
//
// Layout: one CTA per SM (384 threads: w0 TMA producer, w1 MMA issuer, w2 TMEM allocator,
// w4-11 epilogue), 128 x 128 macro-tiles (4 x 4 C tiles: the FP32 path's skip map, entries
// (k, 16-bit mask)), a 4-deep ring of 48 KB stages holding A[3 planes][128 x 32] (K-major
// SWIZZLE_64B, one 3-D TMA) and, per needed 32-column tile, B[3 planes][32 x 32] (MN-major
// SWIZZLE_64B, one 3-D TMA each).  Per k-step the MMA thread decodes the 4 x 4 keep bits into
// runs of adjacent C-tile columns with equal row patterns and issues, per run, 6 products x 2
// tcgen05.mma (M = 128, N = 32*run, K = 16) with the disable-output-lane mask of the skipped
// C-tile rows -- exact leaf-level skipping, as on the BF16 path.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.h"
#include "skipdecide.cuh"
#include "sm100.cuh"

namespace spamm {
namespace {

using namespace sm100;

constexpr int kAPlane = 128 * 32 * 2;              // 8 KB
constexpr int kBBox = 32 * 32 * 2;                 // 2 KB
// P bfloat16/half planes per operand: P = 3 for SPAMM_FP32X3; P = 1 is the BF16/FP16 path of small
// problems (fewer 256 x 256 macro-tiles than SMs: 128 x 128 tiles keep more SMs busy)
template <int P>
struct XCfg {
  // P = 1: a stage carries up to two k-steps (two 16 KB slots): the per-stage round trip (full /
  // empty barriers, descriptor, commit) was ~700 cycles for 132 cycles of MMA per k-step
  static constexpr int kPack = P == 3 ? 1 : 2;
#ifndef SPAMM_X1_STAGES
#define SPAMM_X1_STAGES 4
#endif
  // P = 1: SPAMM_X1_STAGES stages of two k-steps; 6 leaves no room for the 64 KB C staging (the
  // epilogue then stores from registers)
  static constexpr int kStages = P == 3 ? 4 : SPAMM_X1_STAGES;
  static constexpr int kBCol = P * kBBox;                     // one 32-column tile, P planes
  static constexpr int kStageA = P * kAPlane;
  static constexpr int kSlotBytes = kStageA + 4 * kBCol;      // one k-step: 48 KB (P = 3) / 16 KB (P = 1)
  static constexpr int kStageBytes = kPack * kSlotBytes;
  // P = 1: a 64 KB staging tile for the TMA-store epilogue (4 boxes of [128 rows x 32] FP32, SWIZZLE_128B)
  static constexpr int kStageC = (P == 1 && kStages <= 4) ? 65536 : 0;
  static constexpr size_t kSmem = 1024 + static_cast<size_t>(kStages) * kStageBytes + 2048 + kStageC;
};
constexpr int kThreads = 384;
constexpr int kEpiWarps = 8;
constexpr int kTQ = 4;
// k-steps per TMEM partial: 4 for FP32X3 (FP32 accuracy, above); the one-plane BF16/FP16 path
// accumulates a whole tile in TMEM like the 256 x 256 kernel (one epilogue read per tile)
template <int P>
constexpr uint32_t kChunkOf = P == 3 ? 4u : 0x40000000u;
constexpr uint32_t kTmemCols = 256;                // 2 buffers x 128 columns
constexpr uint32_t kFirst = 1u << 29, kLast = 1u << 30, kNoStep = 1u << 28, kEnd = 1u << 27;
// P = 1 stage of two consecutive k-steps (k, k+1) loaded as 64-deep boxes: A [128 x 64] SWIZZLE_128B
// (16 KB), then B boxes [64 k x 32 n] SWIZZLE_64B of 4 KB per column tile -- half the TMA
// instructions of two 32-deep slots (the producer's ~160 cycles per TMA bound the small-problem
// stage rate), the layout of multiply_dual.cu's wide stages
constexpr uint32_t kWide = 1u << 26;

// Runs of a 4 x 4 keep mask (bit 4 li + lj: C-tile row li, column lj): maximal groups of adjacent
// kept columns with equal row patterns, one MMA group each (N = 32 len, disable-output-lane masks
// from the pattern).  8 bits per run (j0: 2, len - 1: 2, row pattern: 4); .x runs 0-3, .y = count |
// needed-columns << 4.  Encoded by the producer warp, one entry per lane, so the MMA thread only
// unpacks (decoding the mask there cost ~700 cycles per k-step of a single warp's dependent chain,
// measured with -DSPAMM_PROFILE on configs[0]).
__device__ __forceinline__ uint2 encode_runs4(uint32_t mask) {
  if (mask == 0xFFFFu) return make_uint2((3u << 2) | (15u << 4), 1u | (15u << 4));
  const uint32_t d = (mask ^ (mask >> 1)) & 0x7777u;   // col lj differs from lj+1 in some row
  const uint32_t bnd = (d | (d >> 4) | (d >> 8) | (d >> 12)) & 0x7u;
  const uint32_t nz = (mask | (mask >> 4) | (mask >> 8) | (mask >> 12)) & 0xFu;
  uint32_t w = 0u, nr = 0u, j = 0u;
  while (j < 4u) {
    const uint32_t b = bnd >> j;
    const uint32_t j1 = b ? j + static_cast<uint32_t>(__ffs(b)) : 4u;
    if ((nz >> j) & 1u) {
      const uint32_t pat = ((mask >> j) & 1u) | (((mask >> (4 + j)) & 1u) << 1) | (((mask >> (8 + j)) & 1u) << 2) |
                           (((mask >> (12 + j)) & 1u) << 3);
      w |= (j | ((j1 - j - 1u) << 2) | (pat << 4)) << (8u * nr);
      ++nr;
    }
    j = j1;
  }
  return make_uint2(w, nr | (nz << 4));
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
  return v;
}

struct TileQ {
  int64_t t, e0, e1;
};

struct X3Maps {
  CUtensorMap a, b;   // 3-D: {cols, rows, plane}
  // N % 32 == 0: B viewed as stacked column tiles {32 n, K, plane, N/32}, boxes of 4 / 2 / 1 whole
  // column tiles with all planes -- the needed column range of a k-step in 1-2 TMAs instead of one
  // per column tile (the producer's TMA issues bound the small-problem k-step rate)
  CUtensorMap bs[3];
  int stacked;
  CUtensorMap c;      // P = 1, plain epilogue: C (FP32) boxes [128 rows x 32], SWIZZLE_128B, for TMA stores
  int tstore;
  // P = 1 wide stages: A boxes {64 k, 128 rows, 1} SW128; B {32 n, 64 k, 1} per column tile and,
  // when stacked, {32, 64, 1, 4/2/1 column tiles}
  CUtensorMap a2, b2, bs2[3];
  int wide;
};

struct XChain {       // chained outputs (P = 1): tile norms of the stored C, a rounded copy, C_low only
  double* nC;
  int64_t ldn;
  void* clow;
  int64_t ldl;
  int low_only;
};

#ifdef SPAMM_PROFILE
// per-CTA timeline (globaltimer ns) [0] start [1] after griddepcontrol.wait [2] first TMA issued
// [3] first stage landed (MMA) [4] MMA done [5] epilogue last TMEM read [6] epilogue done;
// counters (clock64 cycles) [8] MMA full-wait [9] MMA tmem-empty wait [10] epilogue tmem-full wait
// [11] producer empty-wait [12] k-steps (compile with -DSPAMM_PROFILE)
__device__ unsigned long long* g_x3_prof;
#define X3_STAMP(k) do { unsigned long long g_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_)); \
  g_x3_prof[blockIdx.x * 24 + (k)] = g_; } while (0)
#define X3_CLK() clock64()
#define X3_ADD(k, v) (pc[(k) - 8] += (v))   // register counters, stored once at the end
#else
#define X3_STAMP(k) do { } while (0)
#define X3_CLK() 0ll
#define X3_ADD(k, v) do { (void)(v); } while (0)
#endif
#ifdef SPAMM_PROFILE
#define X3_FLUSH() do { for (int k_ = 0; k_ < 12; ++k_) if (pc[k_]) atomicAdd(g_x3_prof + blockIdx.x * 24 + 8 + k_, \
  static_cast<unsigned long long>(pc[k_])); } while (0)
#else
#define X3_FLUSH() do { } while (0)
#endif

template <int P, uint32_t kFmt, bool kGen, bool kFuse>
__global__ void __launch_bounds__(kThreads, 1)
    spamm_mul_x3_kernel(const __grid_constant__ X3Maps mp, const int64_t* __restrict__ mstart,
                        const int64_t* __restrict__ mcount, const uint2* ment,
                        const int32_t* __restrict__ order, int64_t n_tiles, int64_t GN, float* __restrict__ C,
                        int64_t ldc, int64_t M, int64_t N, unsigned int* __restrict__ sched, const Axpby ab,
                        const int64_t* __restrict__ rng, const int64_t* __restrict__ n_empty_p, const XChain co,
                        const XFuse fz) {
  constexpr int kStages = XCfg<P>::kStages, kStageBytes = XCfg<P>::kStageBytes;
  constexpr int kStageA = XCfg<P>::kStageA, kBCol = XCfg<P>::kBCol;
  constexpr int kPack = XCfg<P>::kPack, kSlotBytes = XCfg<P>::kSlotBytes;
  // claims follow the skip map's order (skipmap.cu order_pass); every tile, with or without
  // k-steps, goes through the pipeline (the tiles without kept pairs are last)
  (void)n_empty_p;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sZero = smem + kStages * kStageBytes;                  // 512-B zero atom (D = 0 MMA)
  uint64_t* full = reinterpret_cast<uint64_t*>(sZero + 512);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* tq_full = tempty + 2;
  uint64_t* tq_empty = tq_full + kTQ;
  uint4* srun = reinterpret_cast<uint4*>(tq_empty + kTQ);        // [kStages] k-step descriptors
  TileQ* tq = reinterpret_cast<TileQ*>(srun + kStages);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq + kTQ);
  uint8_t* sC = smem + kStages * kStageBytes + 2048;                // P = 1: C staging (1024-aligned)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) X3_STAMP(0);
#ifdef SPAMM_PROFILE
  long long pc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  bool st2 = false, st3 = false;
#endif
  for (int i = threadIdx.x; i < 512 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sZero)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    for (int q = 0; q < kTQ; ++q) {
      mbar_init(&tq_full[q], 1);
      mbar_init(&tq_empty[q], kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  pdl_wait();      // the skip map (order, lists) and the claim counter are ready
  pdl_trigger();
  if (threadIdx.x == 0) X3_STAMP(1);
  if (rng != nullptr) n_tiles = (rng[1] - rng[0]) * GN;   // multi-GPU: range decided on the device

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&mp.a);
      tma_prefetch_desc(&mp.b);
      if (mp.stacked)
        for (int q = 0; q < 3; ++q) tma_prefetch_desc(&mp.bs[q]);
      if (mp.wide) {
        tma_prefetch_desc(&mp.a2);
        tma_prefetch_desc(&mp.b2);
        if (mp.stacked)
          for (int q = 0; q < 3; ++q) tma_prefetch_desc(&mp.bs2[q]);
      }
    }
    int s = 0, tq_s = 0;
    uint32_t ph = 0, tq_ph = 0;
    int64_t fz_next = blockIdx.x;   // kFuse: static tile assignment
    uint2 fz_reg = make_uint2(0u, 0u);
    uint32_t fz_any = 0u;
    auto claim = [&]() -> TileQ {
      TileQ ti{-1, 0, 0};
      if constexpr (kFuse) {
        if (fz_next < n_tiles) {
          ti.t = fz_next;
          ti.e0 = ti.t * fz.BK;
          ti.e1 = ti.e0 + fuse_tile_list(fz, ti.t, GN, lane, &fz_reg, &fz_any);
        }
        fz_next += gridDim.x;
      } else {
        unsigned int idx = 0;
        if (lane == 0) idx = atomicAdd(sched, 1u);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (static_cast<int64_t>(idx) < n_tiles) {
          ti.t = order[idx];
          ti.e0 = mstart[ti.t];
          ti.e1 = ti.e0 + mcount[ti.t];
        }
      }
      return ti;
    };
    // the next tile is claimed once the current one's loads are issued (LPT tail by finish time;
    // claiming at tile start measured 163.5 vs 143.6 us on the 256 x 256 kernel, multiply_dual.cu)
    TileQ cur = claim();
    if (lane == 0) X3_STAMP(7);   // first tile claimed (kFuse: its list decided)
    for (;;) {
      if (lane == 0) {   // publish the tile (or the end marker) to the epilogue
        mbar_wait(&tq_empty[tq_s], tq_ph ^ 1);
        tq[tq_s] = cur;
        mbar_arrive(&tq_full[tq_s]);
      }
      if (++tq_s == kTQ) {
        tq_s = 0;
        tq_ph ^= 1;
      }
      if (cur.t < 0 || cur.e1 == cur.e0) {   // end of stream / a tile without k-steps (C = 0)
        if (lane == 0) {
          mbar_wait(&empty[s], ph ^ 1);
          srun[s] = make_uint4(0, 0, 0, cur.t < 0 ? kEnd : (kFirst | kLast | kNoStep));
          mbar_arrive(&full[s]);
        }
        if (++s == kStages) {
          s = 0;
          ph ^= 1;
        }
        if (cur.t < 0) break;
        cur = claim();
        continue;
      }
      const int32_t I = static_cast<int32_t>(cur.t / GN), J = static_cast<int32_t>(cur.t % GN);
      // 32 entries per warp load; the whole warp walks them on shuffled (warp-uniform) values and
      // one elected lane issues the stage's operations (no per-entry dependent global load, no
      // R2UR waterfall around the TMA instructions)
      for (int64_t eb = cur.e0; eb < cur.e1; eb += 32) {
        const int cnt = static_cast<int>(cur.e1 - eb < 32 ? cur.e1 - eb : 32);
        uint2 en_l = make_uint2(0u, 0u);
        if (kFuse && fz.BK <= 32) {   // one chunk: entry q from the q-th lane with a kept pair
          const int src = lane < cnt ? static_cast<int>(__fns(fz_any, 0u, lane + 1)) : 0;
          en_l.x = __shfl_sync(0xffffffffu, fz_reg.x, src);
          en_l.y = __shfl_sync(0xffffffffu, fz_reg.y, src);
          if (lane >= cnt) en_l = make_uint2(0u, 0u);
        } else if (lane < cnt) {
          // kFuse: entries this warp just wrote (coherent load, not the read-only path)
          en_l = kFuse ? __ldcg(ment + eb + lane) : __ldg(ment + eb + lane);
        }
        const uint2 run_l = encode_runs4(en_l.y & 0xFFFFu);
        for (int q = 0; q < cnt; q += kPack) {
          const int np = cnt - q < kPack ? cnt - q : kPack;   // k-steps in this stage
          const int64_t e = eb + q;
          const long long tw0 = X3_CLK();
          mbar_wait(&empty[s], ph ^ 1);
          if (lane == 0) X3_ADD(11, X3_CLK() - tw0);
          uint8_t* st = smem + s * kStageBytes;
#ifdef SPAMM_PROFILE
          if (lane == 0 && !st2) {
            X3_STAMP(2);
            st2 = true;
          }
#endif
          const long long ti0 = X3_CLK();
          uint32_t rws[kPack], rns[kPack], exs[kPack];
#pragma unroll
          for (int j = 0; j < kPack; ++j) {   // warp-uniform: lane q + j's entry and runs
            const int src = q + j < cnt ? q + j : q;
            exs[j] = __shfl_sync(0xffffffffu, en_l.x, src);
            rws[j] = __shfl_sync(0xffffffffu, run_l.x, src);
            rns[j] = __shfl_sync(0xffffffffu, run_l.y, src);
          }
          const bool wide = kPack == 2 && mp.wide && np == 2 && exs[kPack - 1] == exs[0] + 1u;
          if (elect_one()) {
            // srun: x = runs of slot 0, y = runs of slot 1, z = run counts (8 bits per slot) | slots << 16
            srun[s] = make_uint4(rws[0], kPack > 1 ? rws[kPack - 1] : 0u,
                                 (rns[0] & 0xFu) | (kPack > 1 ? (rns[kPack - 1] & 0xFu) << 8 : 0u) |
                                     (static_cast<uint32_t>(np) << 16),
                                 (e == cur.e0 ? kFirst : 0u) | (e + np == cur.e1 ? kLast : 0u) | (wide ? kWide : 0u));
          }
          if (wide) {   // one A box and the union column range of B for both k-steps
            if (elect_one()) {
              const uint32_t cols = (rns[0] | rns[kPack - 1]) >> 4;
              const int c0 = __ffs(cols) - 1, len = (32 - __clz(cols)) - c0;
              const int32_t k0 = static_cast<int32_t>(exs[0]) * 32;
              mbar_arrive_expect_tx(&full[s], 2 * kStageA + 2 * kBCol * (mp.stacked ? len : __popc(cols)));
              tma_load_3d(st, &mp.a2, &full[s], k0, I * 128, 0);
              uint8_t* sb = st + 2 * kStageA;
              if (mp.stacked) {
                int off = c0;
                if (len == 4) {
                  tma_load_4d(sb, &mp.bs2[0], &full[s], 0, k0, 0, J * 4);
                } else {
                  if (len & 2) {
                    tma_load_4d(sb + off * 2 * kBCol, &mp.bs2[1], &full[s], 0, k0, 0, J * 4 + off);
                    off += 2;
                  }
                  if (len & 1) tma_load_4d(sb + off * 2 * kBCol, &mp.bs2[2], &full[s], 0, k0, 0, J * 4 + off);
                }
              } else {
#pragma unroll
                for (int lj = 0; lj < 4; ++lj)
                  if ((cols >> lj) & 1u) tma_load_3d(sb + lj * 2 * kBCol, &mp.b2, &full[s], J * 128 + lj * 32, k0, 0);
              }
            }
          } else if (elect_one()) {
            uint32_t bytes = 0;
#pragma unroll
            for (int j = 0; j < kPack; ++j) {
              if (j >= np) break;
              const uint32_t cols = rns[j] >> 4;   // needed C-tile columns
              bytes += kStageA + kBCol * (mp.stacked ? (32 - __clz(cols)) - (__ffs(cols) - 1) : __popc(cols));
            }
            mbar_arrive_expect_tx(&full[s], bytes);
#pragma unroll
            for (int j = 0; j < kPack; ++j) {
              if (j >= np) break;
              uint8_t* sl = st + j * kSlotBytes;
              const uint32_t cols = rns[j] >> 4;
              const int32_t k0 = static_cast<int32_t>(exs[j]) * 32;
              tma_load_3d(sl, &mp.a, &full[s], k0, I * 128, 0);
              if (mp.stacked) {   // the column range [c0, c0 + len) covering the needed tiles
                const int c0 = __ffs(cols) - 1, len = (32 - __clz(cols)) - c0;
                int off = c0;
                if (len == 4) {
                  tma_load_4d(sl + kStageA, &mp.bs[0], &full[s], 0, k0, 0, J * 4);
                } else {
                  if (len & 2) {
                    tma_load_4d(sl + kStageA + off * kBCol, &mp.bs[1], &full[s], 0, k0, 0, J * 4 + off);
                    off += 2;
                  }
                  if (len & 1) tma_load_4d(sl + kStageA + off * kBCol, &mp.bs[2], &full[s], 0, k0, 0, J * 4 + off);
                }
              } else {
#pragma unroll
                for (int lj = 0; lj < 4; ++lj)
                  if ((cols >> lj) & 1u) tma_load_3d(sl + kStageA + lj * kBCol, &mp.b, &full[s], J * 128 + lj * 32, k0, 0);
              }
            }
          }
          __syncwarp();
          if (lane == 0) {
            X3_ADD(18, X3_CLK() - ti0);   // TMA issue (elected lane's block)
            X3_ADD(19, X3_CLK() - tw0);   // whole producer stage
          }
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      __syncwarp();
      cur = claim();
    }
  } else if (warp == 1) {
    // -------------------------------------------------------------- MMA issuer
    // the whole warp runs the loop on warp-uniform values; one elected lane issues each tcgen05
    // op (uniform operands go to uniform registers without a per-MMA R2UR waterfall)
    {
      const uint32_t base_addr = smem_u32(smem);
      const uint64_t zdesc = smem_desc(smem_u32(sZero), 0, 0, kLayoutSW64);
      const uint32_t idesc_zero = idesc_f16(kFmt, 128, 128, 0, 1);
      constexpr int kProd = P == 3 ? 6 : 1;   // products per kept pair (plane pairs)
      const uint32_t pa[6] = {0, 0, 1, 0, 1, 2}, pb[6] = {0, 1, 0, 2, 1, 0};
      uint32_t ph = 0, ub = 0;   // bit b: phase parity of TMEM buffer b (no local-memory array)
      int buf = 0;
      uint32_t kin = 0;   // k-steps of the current tile issued so far
      bool fin = false;
      while (!fin) {
#pragma unroll 1
        for (int st = 0; st < kStages; ++st) {
          const long long tw0 = X3_CLK();
          mbar_wait(&full[st], ph);
          if (lane == 0) X3_ADD(8, X3_CLK() - tw0);
#ifdef SPAMM_PROFILE
          if (lane == 0 && !st3) {
            X3_STAMP(3);
            st3 = true;
          }
#endif
          tc_fence_after();
          const uint4 rs = lds128(smem_u32(srun + st));   // (runs, run count, -, flags): same for all lanes
          const uint32_t fl = rs.w;
          if (fl & kEnd) {
            fin = true;
            break;
          }
          if (fl & kFirst) kin = 0;
          const uint32_t dcol = tbase + static_cast<uint32_t>(buf) * 128u;
          if ((kin % kChunkOf<P>) == 0) {   // chunk start: a drained buffer, zeroed
            const long long tw1 = X3_CLK();
            mbar_wait(&tempty[buf], (ub >> buf) & 1u);
            if (lane == 0) X3_ADD(9, X3_CLK() - tw1);
            tc_fence_after();
            if (elect_one()) umma_f16(dcol, zdesc, zdesc, idesc_zero, 0u, 0u, 0u, 0u, 0u);
          }
          if (!(fl & kNoStep)) {
            const uint32_t nsl = rs.z >> 16;
#pragma unroll
            for (int sl = 0; sl < kPack; ++sl) {
              if (static_cast<uint32_t>(sl) >= nsl) break;
              const uint32_t runs = sl == 0 ? rs.x : rs.y;
              const uint32_t nrun = (rs.z >> (8 * sl)) & 0xFFu;
              // 32-deep slot: A K-major SW64 rows of 32 (SBO 512), B MN-major SW64 boxes of 32 n x 32 k
              // (LBO = kBCol); wide stage: A SW128 rows of 64 (SBO 1024), k-step sl at +64 B; B boxes of
              // 32 n x 64 k (LBO = 2 kBCol) after both A halves, k-step sl at +2 KB (32 k-rows)
              const bool wst = (fl & kWide) != 0u;
              const uint32_t st_addr = base_addr + st * kStageBytes;
              const uint64_t ad = wst ? smem_desc(st_addr, 16, 1024, kLayoutSW128) + 4u * sl
                                      : smem_desc(st_addr + sl * kSlotBytes, 16, 512, kLayoutSW64);
              const uint64_t bd = wst ? smem_desc(st_addr + 2 * kStageA, 2 * kBCol, 512, kLayoutSW64) + 128u * sl
                                      : smem_desc(st_addr + sl * kSlotBytes + kStageA, kBCol, 512, kLayoutSW64);
              const uint32_t bcol = wst ? (2 * kBCol) >> 4 : kBCol >> 4;   // descriptor units per column tile
#pragma unroll
              for (uint32_t r = 0; r < 4; ++r) {
                if (r >= nrun) break;
                const uint32_t run = (runs >> (8u * r)) & 0xFFu;
                const uint32_t j = run & 3u, len = ((run >> 2) & 3u) + 1u, pat = run >> 4;
                const uint32_t idesc = idesc_f16(kFmt, 128, 0, 0, 1) | ((len * 4u) << 17);   // N = 32 len
                const uint32_t m0 = (pat & 1u) - 1u, m1 = ((pat >> 1) & 1u) - 1u;
                const uint32_t m2 = ((pat >> 2) & 1u) - 1u, m3 = ((pat >> 3) & 1u) - 1u;
                const uint32_t d = dcol + j * 32u;
                const long long ti0 = X3_CLK();
                if (elect_one()) {
#pragma unroll
                  for (int p = 0; p < kProd; ++p) {
                    const uint64_t a = ad + ((pa[p] * kAPlane) >> 4);
                    const uint64_t b = bd + j * bcol + ((pb[p] * kBBox) >> 4);
                    umma_f16(d, a, b, idesc, 1u, m0, m1, m2, m3);
                    umma_f16(d, a + 2, b + 64, idesc, 1u, m0, m1, m2, m3);
                  }
                }
                __syncwarp();
                if (lane == 0) X3_ADD(14, X3_CLK() - ti0);
              }
            }
          }
          const long long tc0 = X3_CLK();
          if (elect_one()) umma_commit(&empty[st]);
          __syncwarp();
          if (lane == 0) X3_ADD(15, X3_CLK() - tc0);
          if (lane == 0 && !(fl & kNoStep)) X3_ADD(12, 1);
          if (lane == 0) X3_ADD(13, X3_CLK() - tw0);
          ++kin;
          if ((fl & kLast) || (kin % kChunkOf<P>) == 0) {   // chunk complete: hand the buffer over
            if (elect_one()) umma_commit(&tfull[buf]);
            ub ^= 1u << buf;
            buf ^= 1;
          }
        }
        ph ^= 1;
      }
    }
    if (lane == 0) X3_STAMP(4);
    __syncwarp();
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;             // TMEM lane quadrant
    const int half = (warp - 4) >> 2;   // columns [64*half, 64*half + 64)
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&tempty[0]);
      mbar_arrive(&tempty[1]);
    }
    const int t0 = lane & 3, t1 = lane >> 2;
    uint32_t eu = 0;   // bit b: phase parity of TMEM buffer b
    int buf = 0, tq_s = 0;
    uint32_t tq_ph = 0;
    for (;;) {
      const long long tq0 = X3_CLK();
      mbar_wait(&tq_full[tq_s], tq_ph);
      if (warp == 4 && lane == 0) X3_ADD(17, X3_CLK() - tq0);
      const TileQ cur = tq[tq_s];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tq_empty[tq_s]);
      if (++tq_s == kTQ) {
        tq_s = 0;
        tq_ph ^= 1;
      }
      if (cur.t < 0) break;
      const int64_t U = cur.e1 - cur.e0;
      const int64_t nch = U > 0 ? (U + kChunkOf<P> - 1) / kChunkOf<P> : 1;
      float acc[64];
      for (int64_t c = 0; c < nch; ++c) {
        const long long tw0 = X3_CLK();
        mbar_wait(&tfull[buf], (eu >> buf) & 1u);
        if (warp == 4 && lane == 0) X3_ADD(10, X3_CLK() - tw0);
        tc_fence_after();
#pragma unroll
        for (int lh = 0; lh < 2; ++lh) {
          uint32_t v[32];
          tmem_ld_16x256b_x8(tbase + ((static_cast<uint32_t>(q * 32 + 16 * lh)) << 16) + buf * 128 + half * 64, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[32 * lh + i] = c == 0 ? __uint_as_float(v[i]) : acc[32 * lh + i] + __uint_as_float(v[i]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        eu ^= 1u << buf;
        buf ^= 1;
      }
      if (warp == 4 && lane == 0) X3_STAMP(5);
      const long long tst0 = X3_CLK();
      const int64_t I = cur.t / GN, J = cur.t % GN;
      if constexpr (P == 1 && !kGen) {
        if (mp.tstore) {   // stage the tile in shared memory, 4 TMA stores (clipped at M, N)
          if (warp == 4 && lane == 0) bulk_wait_group_read<0>();   // the previous tile's stores have read sC
          named_bar_sync(1, kEpiWarps * 32);
#pragma unroll
          for (int lh = 0; lh < 2; ++lh) {
            const uint32_t ra = static_cast<uint32_t>(q * 32 + 16 * lh + t1);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const uint32_t b = static_cast<uint32_t>(half * 2 + (i >> 2));
              const uint32_t ch = ((2u * (i & 3) + (t0 >> 1)) ^ (ra & 7u)) << 4;   // rb = ra + 8: same row phase
              uint8_t* pa = sC + b * 16384u + ra * 128u + ch + ((t0 & 1) << 3);
              *reinterpret_cast<float2*>(pa) = make_float2(acc[32 * lh + 4 * i], acc[32 * lh + 4 * i + 1]);
              *reinterpret_cast<float2*>(pa + 8 * 128) = make_float2(acc[32 * lh + 4 * i + 2], acc[32 * lh + 4 * i + 3]);
            }
          }
          fence_proxy_async_smem();
          named_bar_sync(1, kEpiWarps * 32);
          if (warp == 4 && lane == 0) {
#pragma unroll
            for (int b = 0; b < 4; ++b)
              tma_store_2d(&mp.c, sC + b * 16384, static_cast<int32_t>(J * 128 + b * 32), static_cast<int32_t>(I * 128));
            bulk_commit_group();
          }
          if (warp == 4 && lane == 0) X3_ADD(16, X3_CLK() - tst0);
          continue;
        }
      }
      double tsum[2] = {0.0, 0.0};   // kGen: sums of squares of the two C tiles of this warp's slice
#pragma unroll
      for (int lh = 0; lh < 2; ++lh) {
        const int64_t ra = I * 128 + q * 32 + 16 * lh + t1, rb = ra + 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int64_t col = J * 128 + half * 64 + 8 * i + 2 * t0;
          const float v0 = acc[32 * lh + 4 * i], v1 = acc[32 * lh + 4 * i + 1];
          const float v2 = acc[32 * lh + 4 * i + 2], v3 = acc[32 * lh + 4 * i + 3];
          float* ca = C + ra * ldc + col;
          float* cb = C + rb * ldc + col;
          if constexpr (!kGen) {
            if (col + 1 < N) {
              if (ra < M) __stcs(reinterpret_cast<float2*>(ca), axpby2(ab, make_float2(v0, v1), ca));
              if (rb < M) __stcs(reinterpret_cast<float2*>(cb), axpby2(ab, make_float2(v2, v3), cb));
            } else if (col < N) {
              if (ra < M) *ca = axpby1(ab, v0, ca);
              if (rb < M) *cb = axpby1(ab, v2, cb);
            }
          } else {
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
              const int64_t row = rr ? rb : ra;
              if (row >= M || col >= N) continue;
              const bool two = col + 1 < N;
              float* cp = rr ? cb : ca;
              float2 x = rr ? make_float2(v2, v3) : make_float2(v0, v1);
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
              tsum[i >> 2] += d0 * d0 + d1 * d1;
            }
          }
        }
      }
      if (warp == 4 && lane == 0) X3_ADD(16, X3_CLK() - tst0);
      if constexpr (kGen) {
        if (co.nC != nullptr) {
#pragma unroll
          for (int tt = 0; tt < 2; ++tt) {
            double x = tsum[tt];
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            const int64_t ti = I * 4 + q, tj = J * 4 + half * 2 + tt;
            if (lane == 0 && ti * 32 < M && tj * 32 < N) co.nC[ti * co.ldn + tj] = sqrt(x);
          }
        }
      }
    }
  }
  if constexpr (P == 1 && !kGen) {
    if (mp.tstore && warp == 4 && lane == 0) bulk_wait_group<0>();   // C written before the CTA retires
  }
  if (warp == 4 && lane == 0) X3_STAMP(6);
  if (lane == 0) X3_FLUSH();
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<kTmemCols>(tbase);
}

}  // namespace

namespace {

#ifdef SPAMM_PROFILE
static void print_x3_profile(const unsigned long long* hp, int grid, int P) {
  unsigned long long g0 = ~0ull;
  for (int c = 0; c < grid; ++c) g0 = std::min(g0, hp[c * 24]);
  double m[8] = {0}, mx[8] = {0}, cn[12] = {0};
  for (int c = 0; c < grid; ++c) {
    for (int k = 0; k < 8; ++k) {
      const double v = hp[c * 24 + k] ? (static_cast<double>(hp[c * 24 + k]) - static_cast<double>(g0)) * 1e-3 : 0.0;
      m[k] += v / grid;
      mx[k] = std::max(mx[k], v);
    }
    for (int k = 0; k < 12; ++k) cn[k] += static_cast<double>(hp[c * 24 + 8 + k]) / grid;
  }
  fprintf(stderr, "[x3 tl P=%d grid %d] us from first CTA start (mean/max): start %.2f/%.2f pdl %.2f/%.2f claim0 %.2f/%.2f "
          "tma0 %.2f/%.2f land0 %.2f/%.2f mma-done %.2f/%.2f epi-read %.2f/%.2f epi-done %.2f/%.2f\n", P, grid, m[0], mx[0],
          m[1], mx[1], m[7], mx[7], m[2], mx[2], m[3], mx[3], m[4], mx[4], m[5], mx[5], m[6], mx[6]);
  fprintf(stderr, "[x3 prof] cycles/CTA: mma full-wait %.0f tmem-empty %.0f | epi tmem-full %.0f | producer empty %.0f | "
          "k-steps %.1f | mma loop incl. waits %.0f (mma issue %.0f, commit %.0f) | epi stores %.0f tile-queue %.0f | "
          "producer k-steps %.0f (tma issue %.0f)\n", cn[0], cn[1], cn[2], cn[3], cn[4], cn[5], cn[6], cn[7], cn[8], cn[9],
          cn[11], cn[10]);
}
#endif

template <int P, uint32_t kFmt, bool kGen, bool kFuse = false>
spamm_status launch_x(Plan& p, const X3Maps& mp, float* C, int64_t ldc, cudaStream_t s) {
  auto kern = spamm_mul_x3_kernel<P, kFmt, kGen, kFuse>;
  constexpr size_t kSmem = XCfg<P>::kSmem;
  SPAMM_SET_SMEM(kern, static_cast<int>(kSmem), p.device);
  const int64_t n_tiles = p.range_on_device ? 0 : (p.row_end_macro - p.row_begin_macro) * p.GN;
  if (!p.range_on_device && n_tiles <= 0) return SPAMM_OK;
  const int grid = static_cast<int>(!p.range_on_device && n_tiles < p.num_sms ? n_tiles : p.num_sms);
  if (!kFuse) {
    if (!p.sched_zeroed) SPAMM_CUDA_TRY(cudaMemsetAsync(p.sched, 0, sizeof(unsigned int), s));
    p.sched_zeroed = false;
  }
#ifdef SPAMM_PROFILE
  static unsigned long long* prof_buf = nullptr;
  if (!prof_buf) {
    cudaMalloc(&prof_buf, 1024 * 24 * 8);
    cudaMemcpyToSymbol(g_x3_prof, &prof_buf, sizeof(prof_buf));
  }
  cudaMemsetAsync(prof_buf, 0, 1024 * 24 * 8, s);
#endif
  SPAMM_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(kThreads), kSmem, s, mp, static_cast<const int64_t*>(p.mstart),
                            static_cast<const int64_t*>(p.U), static_cast<const uint2*>(p.macro_ent),
                            static_cast<const int32_t*>(p.order), n_tiles, p.GN, C, ldc, p.M, p.N, p.sched,
                            Axpby{static_cast<float>(p.alpha), static_cast<float>(p.beta)},
                            static_cast<const int64_t*>(p.range_on_device ? p.d_range : nullptr),
                            static_cast<const int64_t*>(p.totals + 2),
                            XChain{p.out_norms ? p.nC : nullptr, p.BN, p.out_low, p.out_ldl, p.out_low_only ? 1 : 0},
                            XFuse{p.nA, p.nBt, p.BM, p.BK, p.BN, p.tau, p.U, p.L, static_cast<uint2*>(p.macro_ent),
                                  p.order, reinterpret_cast<unsigned long long*>(p.row_work),
                                  reinterpret_cast<unsigned long long*>(p.totals)}));
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
#ifdef SPAMM_PROFILE
  static unsigned long long hp[1024 * 24];
  cudaMemcpyAsync(hp, prof_buf, sizeof(hp), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  print_x3_profile(hp, grid, P);
#endif
  return SPAMM_OK;
}

}  // namespace

// B (K x N, ld elements, `planes` planes K*ld apart) as stacked 32-column tiles {32, K, planes, N/32}
// with boxes of 4, 2 and 1 whole tiles (all planes): smem [tile][plane][32 k][32 n], the per-column
// layout of a stage.  Only when N % 32 == 0 (a partial last tile cannot be a stacked box).
static spamm_status encode_stacked(X3Maps& mp, CUtensorMapDataType dt, const void* B, int64_t N, int64_t K, int64_t ld,
                                   int planes) {
  mp.stacked = N % 32 == 0 ? 1 : 0;
  if (!mp.stacked) return SPAMM_OK;
  const uint64_t dims[4] = {32, static_cast<uint64_t>(K), static_cast<uint64_t>(planes), static_cast<uint64_t>(N / 32)};
  const uint64_t st[3] = {static_cast<uint64_t>(ld) * 2, static_cast<uint64_t>(K * ld) * 2, 64};
  const uint32_t nb[3] = {4, 2, 1};
  for (int q = 0; q < 3; ++q) {
    const uint32_t box[4] = {32, 32, static_cast<uint32_t>(planes), nb[q]};
    SPAMM_TRY(encode_tmap_4d(&mp.bs[q], dt, B, dims, st, box, CU_TENSOR_MAP_SWIZZLE_64B));
  }
  return SPAMM_OK;
}

spamm_status launch_multiply_x3(Plan& p, float* C, int64_t ldc, bool fuse, cudaStream_t s) {
  if (!p.planes) return fail(SPAMM_E_STATE, "FP32X3 split planes missing (spamm_norms not run on this plan)");
  if (p.out_norms || p.out_low) return fail(SPAMM_E_UNSUPPORTED, "chained outputs are not implemented for SPAMM_FP32X3");
  const uint16_t* pA = p.planes;
  const uint16_t* pB = p.b_is_a ? p.planes : p.planes + 3 * p.M * p.ldpa;
  const int64_t ldb = p.b_is_a ? p.ldpa : p.ldpb;
  X3Maps mp;
  std::memset(&mp, 0, sizeof(mp));
  SPAMM_TRY(encode_tmap_3d(&mp.a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, pA, p.K, p.M, 3,
                           static_cast<uint64_t>(p.ldpa) * 2, static_cast<uint64_t>(p.M * p.ldpa) * 2, 32, 128, 3,
                           CU_TENSOR_MAP_SWIZZLE_64B));
  SPAMM_TRY(encode_tmap_3d(&mp.b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, pB, p.N, p.K, 3, static_cast<uint64_t>(ldb) * 2,
                           static_cast<uint64_t>(p.K * ldb) * 2, 32, 32, 3, CU_TENSOR_MAP_SWIZZLE_64B));
  SPAMM_TRY(encode_stacked(mp, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, pB, p.N, p.K, ldb, 3));
  return fuse ? launch_x<3, 1, false, true>(p, mp, C, ldc, s) : launch_x<3, 1, false>(p, mp, C, ldc, s);
}

// BF16/FP16 plans with fewer 256 x 256 macro-tiles than SMs: the same kernel on the inputs
// themselves (one plane, one product per kept pair) over 128 x 128 macro-tiles
spamm_status launch_multiply_x1(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                                bool fuse, cudaStream_t s) {
  const CUtensorMapDataType dt = p.prec == SPAMM_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  X3Maps mp;
  std::memset(&mp, 0, sizeof(mp));
  SPAMM_TRY(encode_tmap_3d(&mp.a, dt, A, p.K, p.M, 1, static_cast<uint64_t>(lda) * 2,
                           static_cast<uint64_t>(p.M * lda) * 2, 32, 128, 1, CU_TENSOR_MAP_SWIZZLE_64B));
  SPAMM_TRY(encode_tmap_3d(&mp.b, dt, B, p.N, p.K, 1, static_cast<uint64_t>(ldb) * 2,
                           static_cast<uint64_t>(p.K * ldb) * 2, 32, 32, 1, CU_TENSOR_MAP_SWIZZLE_64B));
  SPAMM_TRY(encode_stacked(mp, dt, B, p.N, p.K, ldb, 1));
  // wide stages (two consecutive k-steps): A {64, 128} SW128, B {32, 64} per column tile / stacked
  mp.wide = 1;
  SPAMM_TRY(encode_tmap_3d(&mp.a2, dt, A, p.K, p.M, 1, static_cast<uint64_t>(lda) * 2,
                           static_cast<uint64_t>(p.M * lda) * 2, 64, 128, 1, CU_TENSOR_MAP_SWIZZLE_128B));
  SPAMM_TRY(encode_tmap_3d(&mp.b2, dt, B, p.N, p.K, 1, static_cast<uint64_t>(ldb) * 2,
                           static_cast<uint64_t>(p.K * ldb) * 2, 32, 64, 1, CU_TENSOR_MAP_SWIZZLE_64B));
  if (mp.stacked) {
    const uint64_t dims[4] = {32, static_cast<uint64_t>(p.K), 1, static_cast<uint64_t>(p.N / 32)};
    const uint64_t st[3] = {static_cast<uint64_t>(ldb) * 2, static_cast<uint64_t>(p.K * ldb) * 2, 64};
    const uint32_t nb[3] = {4, 2, 1};
    for (int q = 0; q < 3; ++q) {
      const uint32_t box[4] = {32, 64, 1, nb[q]};
      SPAMM_TRY(encode_tmap_4d(&mp.bs2[q], dt, B, dims, st, box, CU_TENSOR_MAP_SWIZZLE_64B));
    }
  }
  const bool gen = p.alpha != 1.0 || p.beta != 0.0 || p.out_norms || p.out_low != nullptr;
  mp.tstore = !gen && C != nullptr && XCfg<1>::kStageC > 0;
  if (mp.tstore)
    SPAMM_TRY(encode_tmap_2d(&mp.c, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, C, p.N, p.M, ldc, 32, 128,
                             CU_TENSOR_MAP_SWIZZLE_128B));
  if (fuse) {
    if (p.prec == SPAMM_BF16)
      return gen ? launch_x<1, 1, true, true>(p, mp, C, ldc, s) : launch_x<1, 1, false, true>(p, mp, C, ldc, s);
    return gen ? launch_x<1, 0, true, true>(p, mp, C, ldc, s) : launch_x<1, 0, false, true>(p, mp, C, ldc, s);
  }
  if (p.prec == SPAMM_BF16)
    return gen ? launch_x<1, 1, true>(p, mp, C, ldc, s) : launch_x<1, 1, false>(p, mp, C, ldc, s);
  return gen ? launch_x<1, 0, true>(p, mp, C, ldc, s) : launch_x<1, 0, false>(p, mp, C, ldc, s);
}

}  // namespace spamm
