// multiply_umma.cu -- stage 3, tensor-core path (tensor-core multiplication kernel,
// Sec. 3.3, Alg. 3), BF16/FP16 inputs, FP32 accumulation.
//
// C[i,j] = sum_{kept k, ascending} A[i,k] * B[k,j]; the paper's FP32
// accumulator fragment becomes an FP32 accumulator in TMEM.
//
// B200 design (tcgen05, not the paper's wmma):
//   * persistent CTAs (one per SM) claim 128x256 macro-tiles (4 x 8 C tiles of 32x32)
//     dynamically from an atomic counter in LPT order (descending union length);
//   * the skip map pre-decodes every k-step: its 4 x 8 keep bits become runs of
//     adjacent C-tile columns with the same 4-bit row pattern, and two consecutive
//     k-tiles (2p, 2p+1) with the same mask are merged into one 64-deep k-step, which
//     halves the per-step control work of the two single-thread roles below;
//   * warp 0 (one lane): TMA producer -- A[128 x 32] (K-major SWIZZLE_64B) or
//     A[128 x 64] (SWIZZLE_128B) and the contiguous range of needed B[32|64 x 32] boxes
//     (MN-major SWIZZLE_64B), one 3-D TMA per power-of-two piece, into a 4-deep ring of
//     48 KB stages (mbarriers with transaction counts);
//   * warp 1 (one lane): tcgen05.mma kind::f16 M=128, K=16 (2 or 4 per run) into a TMEM
//     accumulator; each run is ONE MMA of N = 32*run whose disable-output-lane mask
//     switches off the 32-lane groups (C-tile rows) whose pair is skipped -- exact
//     leaf-level skip semantics (Alg. 2 l.3-8) on 128-row instructions.
//     Each accumulator is reset by one accumulate=0 MMA on a 512-byte zero atom;
//   * warps 4-11: epilogue -- TMEM (16x256b loads: a thread quad holds 8 consecutive
//     columns of a row) -> coalesced 8-byte stores of C, every 32-byte sector written
//     whole; two TMEM accumulators (2 x 256 columns) overlap the epilogue (C is 4 bytes
//     per output, the dominant store traffic) with the next macro-tile's MMAs.
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

// Two configurations (SPAMM_UMMA_VARIANT, chosen per plan):
//   kCtas = 2: two CTAs per SM, each with ONE 128x256 TMEM accumulator and its own MMA
//              issuer.  A single issuing thread cannot queue tcgen05.mma ahead of the pipe
//              (each issue waits for the previous MMA; scripts/probe_queue*.cu), so the
//              bookkeeping between k-steps is only hidden when a second issuer feeds the
//              same tensor pipe meanwhile; the other CTA's epilogue overlaps as well.
//   kCtas = 1: one CTA per SM with two accumulators (epilogue overlap, one issuer).
//   kWide:     stages hold 64-deep k-steps (merged k pairs), else 32-deep.
template <int kCtas, bool kWide>
struct Cfg {
  static constexpr int kASlot = kWide ? 128 * 64 * 2 : 128 * 32 * 2;    // A[128 x 64|32]
  static constexpr int kBSlot = kWide ? 64 * 256 * 2 : 32 * 256 * 2;    // B[64|32 x 256]
  static constexpr int kStageBytes = kASlot + kBSlot;
  // kCtas == 1: one CTA per SM whose two MMA warps each own one 128-column half of the
  // macro-tile (both consume every stage), two TMEM tiles (512 columns) and an 8-deep ring
  static constexpr int kStages = kCtas == 2 ? (kWide ? 2 : 4) : (kWide ? 4 : 8);
  static constexpr int kBufs = kCtas == 2 ? 1 : 2;                       // TMEM accumulators
  static constexpr uint32_t kTmemCols = 256u * kBufs;
  static constexpr size_t kSmemBytes = 1024 + static_cast<size_t>(kStages) * kStageBytes + 1024 + 1536;
};
constexpr int kThreads = 384;                   // w0 TMA, w1 MMA, w2 TMEM alloc, w4-11 epilogue
constexpr int kEpiWarps = 8;                    // 2 per TMEM lane quadrant, 4 column chunks each
constexpr int kTQ = 4;                          // tile ring depth (dynamic LPT scheduling)

// run word of a k-step whose 4 x 8 keep bits are all set: j0 = 0, len = 8, pattern 1111
constexpr uint32_t kFullRun = 0u | (7u << 3) | (15u << 6);
// stream flags in srun[s].w (bits 0-19 hold runs 6-7, bit 31 marks a 64-deep k-step)
constexpr uint32_t kFirst = 1u << 29, kLast = 1u << 30, kNoStep = 1u << 28, kEnd = 1u << 27;

// A chunk of the k-step stream: macro-tile t (LPT position i), entries [e0, e1) of its list;
// part != 0 when the chunk is not the whole list (stream-K split, combined via scratch).
struct TileInfo {
  int64_t t, e0, e1, i;
  int32_t part, pad;
};
__device__ __forceinline__ TileInfo tile_info(const int32_t* order, const int64_t* mstart, const int64_t* mcount,
                                              int64_t idx, int64_t n_tiles) {
  TileInfo ti{-1, 0, 0, idx, 0, 0};
  if (idx < n_tiles) {
    ti.t = order[idx];
    ti.e0 = mstart[ti.t];
    ti.e1 = ti.e0 + mcount[ti.t];
  }
  return ti;
}

// Stream-K partition: CTA c of G owns k-steps [B(c), B(c+1)) of the LPT-ordered stream of
// W steps, B(c) = c*W/G; owner(x) is the CTA whose range holds step x.
__device__ __forceinline__ int64_t sk_bound(int64_t c, int64_t W, int64_t G) { return (c * W) / G; }
__device__ __forceinline__ int64_t sk_owner(int64_t x, int64_t W, int64_t G) {
  int64_t c = (x * G) / W;
  while (c + 1 < G && sk_bound(c + 1, W, G) <= x) ++c;
  while (c > 0 && sk_bound(c, W, G) > x) --c;
  return c;
}
// scratch slot of contributor c2 to the partial tile at LPT position i: a CTA's first chunk
// uses slot 2c, its last chunk slot 2c+1 (a single-chunk range uses 2c).
__device__ __forceinline__ int64_t sk_slot(int64_t c2, int64_t c_lo, int64_t wi, int64_t W, int64_t G) {
  return 2 * c2 + ((c2 == c_lo && sk_bound(c_lo, W, G) < wi) ? 1 : 0);
}
// Cost weight of one k-step entry for the stream-K split, in units of ~one MMA pair: the
// issuing thread's per-step overhead (~3) plus one per MMA run (x2 for a 64-deep step).
// Measured on B200: MMA-thread cycles per CTA track MMA count (corr 0.97), not step count.
constexpr int64_t kMaxEntryW = 3 + 2 * 8;
__device__ __forceinline__ int64_t entry_w(const uint4& en) {
  const uint32_t nr = (en.x >> 16) & 15u;
  return 3 + static_cast<int64_t>(nr) * ((en.w >> 31) ? 2 : 1);
}
// Smallest e in [0, n) whose start weight w_start + sum_{e' < e} w(e') is >= target (n if none);
// whole warp, returns the same value in every lane.  *w_at = start weight of that entry.
__device__ __forceinline__ int64_t find_entry(const uint4* __restrict__ ent, int64_t n, int64_t w_start, int64_t target,
                                              int64_t* w_at) {
  const int lane = threadIdx.x & 31;
  int64_t base = 0, w = w_start;
  while (base < n && w < target) {
    const int64_t e = base + lane;
    const int64_t we = e < n ? entry_w(ent[e]) : 0;
    int64_t incl = we;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int64_t start = w + incl - we;                  // start weight of entry e
    const uint32_t hit = __ballot_sync(0xffffffffu, e < n && start >= target);
    if (hit) {
      const int l = __ffs(hit) - 1;
      *w_at = __shfl_sync(0xffffffffu, start, l);
      return base + l;
    }
    w += __shfl_sync(0xffffffffu, incl, 31);
    base += 32;
  }
  *w_at = w;
  return base < n ? base : n;
}

// Chained SpAMM outputs: the tile norms of the written C, and optionally a
// copy of C rounded to the plan's input precision (the next product's operand); the norms are
// then those of the rounded values (reading R4).
struct ChainOut {
  double* nC;       // [BM][ldn] or nullptr
  int64_t ldn;
  void* clow;       // bf16/fp16 copy of C or nullptr
  int64_t ldl;
};

struct Maps {   // A (32- and 64-deep boxes); B as stacked 32-column boxes, 1..8 boxes, 32- or 64-deep
  CUtensorMap a1, a2, b1[4], b2[4], b2d, b64, b64w;
};

// kGen: general epilogue (alpha/beta, chained outputs).  The plain instantiation (alpha = 1,
// beta = 0, no chain outputs) keeps the register budget of 2 CTAs/SM free of spills.
template <uint32_t kFmt, int kCtas, bool kWide, bool kGen>
__global__ void __launch_bounds__(kThreads, kCtas)
    spamm_mul_umma_kernel(const __grid_constant__ Maps mp, int use3d, const int64_t* __restrict__ mstart,
                          const int64_t* __restrict__ mcount, const uint4* __restrict__ ment,
                          const int32_t* __restrict__ order, int64_t n_tiles, int64_t GN, float* __restrict__ C,
                          int64_t ldc, int64_t M, int64_t N, unsigned int* __restrict__ sched,
                          const int64_t* __restrict__ n_empty_p, const int64_t* __restrict__ wpre,
                          float* __restrict__ sk_scratch, unsigned int* __restrict__ sk_ticket,
                          const Axpby ab, const ChainOut co, unsigned long long* __restrict__ prof, int dbg) {
  using C_ = Cfg<kCtas, kWide>;
  // The LPT order lists macro-tiles by descending union length, so the tiles without any
  // kept pair (C = 0 there; often most of a banded product) are its tail.  Default
  // (n_empty_p == nullptr): they are claimed like any tile and written through the pipeline
  // (one D = 0 MMA and an epilogue pass), which lets early-finishing CTAs absorb them at the
  // end -- measured fastest.  With n_empty_p (required by stream-K) only the first n_work
  // tiles go through the pipeline and the epilogue warps zero-fill the rest in 8-row units
  // (bulk stores of a zero buffer, dealt round-robin).
  const int64_t n_empty = n_empty_p ? *n_empty_p : 0;
  const int64_t n_work = n_tiles - n_empty;
  // Stream-K (wpre != nullptr): the n_work non-empty tiles' k-steps, in LPT order, are one
  // stream of W = wpre[n_work] steps split evenly over the grid; a tile cut by a range
  // boundary is accumulated in parts whose FP32 partials meet in sk_scratch, and the last
  // contributor (per-tile ticket) adds them in CTA order and stores C.  Otherwise CTAs
  // claim whole tiles dynamically (sched[0]).
  const bool streamk = wpre != nullptr;
  // W is in entry-weight units (entry_w); an entry belongs to the worker whose range holds
  // its start weight.  G = min(grid, W / kMaxEntryW) workers (CTAs >= G only zero-fill), so
  // the contributors to a split tile are exactly owner(w0) .. owner(start of its last entry).
  const int64_t skW = streamk ? wpre[n_work] : 0, skC = blockIdx.x;
  // (workers' ranges are >= kMaxEntryW wide, so each holds at least one entry start)
  const int64_t skGmax = skW / kMaxEntryW;
  const int64_t skG = skGmax < static_cast<int64_t>(gridDim.x) ? (skGmax > 0 ? skGmax : 1) : static_cast<int64_t>(gridDim.x);
  constexpr int kStages = C_::kStages, kStageBytes = C_::kStageBytes, kASlot = C_::kASlot, kBufs = C_::kBufs;
  constexpr uint32_t kTmemCols = C_::kTmemCols;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sZero = smem + kStages * kStageBytes;                // 1 KB of zeros: MMA zero atom, bulk zero-fill source
  uint64_t* full = reinterpret_cast<uint64_t*>(sZero + 1024);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* tq_full = tempty + 2;
  uint64_t* tq_empty = tq_full + kTQ;
  uint4* srun = reinterpret_cast<uint4*>(tq_empty + kTQ);       // [kStages] the stage's k-step
  uint4* sentA = srun + kStages;                                 // [32] producer A entry batch
  uint4* sentB = sentA + 32;                                     // [32] producer B entry batch
  TileInfo* tq = reinterpret_cast<TileInfo*>(sentB + 32);       // [kTQ]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq + kTQ);
  volatile uint32_t* sk_flag = tmem_slot + 1;                    // stream-K: "this CTA combines" 

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (prof && threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    prof[blockIdx.x * 16 + 8] = g;
  }
  for (int i = threadIdx.x; i < 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sZero)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();   // the zero atom is read by tcgen05.mma (async proxy)
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCtas == 1 ? 2 : 1);   // split issuers: both halves release a stage
    }
    for (int b = 0; b < kBufs; ++b) {
      mbar_init(&tfull[b], kCtas == 1 ? 2 : 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    for (int q = 0; q < kTQ; ++q) {
      mbar_init(&tq_full[q], 1);
      mbar_init(&tq_empty[q], 1 + kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  if (prof && threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    prof[blockIdx.x * 16 + 10] = g;
  }

  // The k-steps of all tiles form one stream through the stage ring; srun[s].w carries
  // the tile boundaries so the MMA issuer needs no tile queue and its ring position is a
  // compile-time constant (stage loop unrolled): the issuing thread's per-k-step
  // instruction count is what bounds this kernel (a single thread cannot queue MMAs).
  if (warp == 0) {
    // ------------------------------------------- producer A: tile claims, srun, A boxes
    if (lane == 0) {
      tma_prefetch_desc(&mp.a1);
      tma_prefetch_desc(&mp.a2);
    }
    int s = 0;
    uint32_t ph = 0;
    int tq_s = 0;
    uint32_t tq_ph = 0;
    unsigned long long p_wait = 0, p_claim = 0;
    const unsigned long long p_t0 = clock64();
    // dynamic mode: tiles are claimed one ahead so the claim's latency hides behind the
    // current tile; stream-K mode: walk the tiles overlapping [b0, b1)
    const bool worker = streamk && skC < skG;
    const int64_t b0 = worker ? sk_bound(skC, skW, skG) : 0, b1 = worker ? sk_bound(skC + 1, skW, skG) : 0;
    int64_t sk_i = 0;
    if (streamk && b0 < b1) {   // largest i < n_work with wpre[i] <= b0
      int64_t lo = 0, hi = n_work - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (wpre[mid] <= b0) lo = mid; else hi = mid - 1;
      }
      sk_i = lo;
    }
    auto sk_next = [&]() -> TileInfo {
      TileInfo ti{-1, 0, 0, -1, 0, 0};
      while (b0 < b1 && sk_i < n_work && wpre[sk_i] < b1) {
        const int64_t w0 = wpre[sk_i], w1 = wpre[sk_i + 1];
        const int64_t t = order[sk_i];
        const int64_t ms = mstart[t], cnt = mcount[t];
        int64_t wa = w0;
        const int64_t ea = w0 >= b0 ? 0 : find_entry(ment + ms, cnt, w0, b0, &wa);
        int64_t wb = w1;
        const int64_t eb = w1 <= b1 ? cnt : ea + find_entry(ment + ms + ea, cnt - ea, wa, b1, &wb);
        ++sk_i;
        if (ea < eb) {
          ti.t = t;
          ti.i = sk_i - 1;
          ti.e0 = ms + ea;
          ti.e1 = ms + eb;
          ti.part = (ea > 0 || eb < cnt) ? 1 : 0;
          break;
        }
      }
      return ti;
    };
    TileInfo nxt;
    if (streamk) {
      nxt = sk_next();
    } else {
      unsigned int idx = 0;
      if (lane == 0) idx = atomicAdd(sched, 1u);
      nxt = tile_info(order, mstart, mcount, __shfl_sync(0xffffffffu, idx, 0), n_work);
    }
    auto next_stage = [&]() {
      if (++s == kStages) {
        s = 0;
        ph ^= 1;
      }
    };
    for (;;) {
      const TileInfo cur = nxt;
      const unsigned long long tc0 = prof ? clock64() : 0;
      if (cur.t >= 0) {
        if (streamk) {
          nxt = sk_next();
        } else {
          unsigned int idx = 0;
          if (lane == 0) idx = atomicAdd(sched, 1u);
          nxt = tile_info(order, mstart, mcount, __shfl_sync(0xffffffffu, idx, 0), n_work);
        }
      }
      if (prof) p_claim += clock64() - tc0;
      if (lane == 0) {
        mbar_wait(&tq_empty[tq_s], tq_ph ^ 1);
        tq[tq_s] = cur;
        mbar_arrive(&tq_full[tq_s]);
      }
      if (++tq_s == kTQ) {
        tq_s = 0;
        tq_ph ^= 1;
      }
      if (cur.t < 0 || cur.e1 == cur.e0) {   // end of stream, or a tile without k-steps (C = 0)
        if (lane == 0) {
          mbar_wait(&empty[s], ph ^ 1);
          srun[s] = make_uint4(0, 0, 0, cur.t < 0 ? kEnd : (kFirst | kLast | kNoStep));
          mbar_arrive(&full[s]);
        }
        next_stage();
        if (cur.t < 0) break;
        continue;
      }
      const int32_t I = static_cast<int32_t>(cur.t / GN);
      for (int64_t eb = cur.e0; eb < cur.e1; eb += 32) {
        const int cnt = static_cast<int>(cur.e1 - eb < 32 ? cur.e1 - eb : 32);
        if (lane < cnt) sentA[lane] = ment[eb + lane];
        __syncwarp();
        if (lane == 0) {
          for (int q = 0; q < cnt; ++q) {
            uint4 en = sentA[q];
            const uint32_t cols = en.x >> 24;
            const bool wide = kWide && (en.w >> 31) != 0u;
            const int32_t k0 = static_cast<int32_t>(en.x & 0xFFFFu) * 32;
            en.w |= (eb + q == cur.e0 ? kFirst : 0u) | (eb + q + 1 == cur.e1 ? kLast : 0u);
            const unsigned long long tw0 = prof ? clock64() : 0;
            mbar_wait(&empty[s], ph ^ 1);
            if (prof) p_wait += clock64() - tw0;
            srun[s] = en;
            uint8_t* adst = smem + s * kStageBytes;
            if (dbg & 2) {
              mbar_arrive(&full[s]);   // debug: no loads
            } else if (use3d == 2) {
              // B in 64-column (128-byte-row) atoms: those covering the needed column tiles
              const int c0 = __ffs(cols) - 1, c1 = 32 - __clz(cols);
              const int na = ((c1 + 1) >> 1) - (c0 >> 1);
              mbar_arrive_expect_tx(&full[s], (wide ? 2 : 1) * (8192 + 4096 * na));
              tma_load_2d(adst, wide ? &mp.a2 : &mp.a1, &full[s], k0, I * 128);
            } else if (use3d) {
              const int c0 = __ffs(cols) - 1, len = (32 - __clz(cols)) - c0;
              mbar_arrive_expect_tx(&full[s], (wide ? 2 : 1) * (8192 + 2048 * len));
              tma_load_2d(adst, wide ? &mp.a2 : &mp.a1, &full[s], k0, I * 128);
            } else {
              mbar_arrive_expect_tx(&full[s], 8192 + 2048 * __popc(cols));
              tma_load_2d(adst, &mp.a1, &full[s], k0, I * 128);
            }
            next_stage();
          }
        }
        __syncwarp();   // (s, ph) are only used by lane 0
      }
    }
    if (prof && lane == 0) {
      prof[blockIdx.x * 16 + 1] = p_wait;
      prof[blockIdx.x * 16 + 7] = clock64() - p_t0;
      prof[blockIdx.x * 16 + 11] = p_claim;
    }
  } else if (warp == 3) {
    // --------------------------------------------------------------- producer B
    if (lane == 0) {
      if (use3d == 2) {
        tma_prefetch_desc(&mp.b64);
        tma_prefetch_desc(&mp.b64w);
      } else {
        for (int q = 0; q < 4; ++q) {
          tma_prefetch_desc(&mp.b1[q]);
          tma_prefetch_desc(&mp.b2[q]);
        }
      }
    }
    int s = 0;
    uint32_t ph = 0;
    int tq_s = 0;
    uint32_t tq_ph = 0;
    for (;;) {
      mbar_wait(&tq_full[tq_s], tq_ph);
      const TileInfo cur = tq[tq_s];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tq_empty[tq_s]);
      if (++tq_s == kTQ) {
        tq_s = 0;
        tq_ph ^= 1;
      }
      if (cur.t < 0) break;
      if (cur.e1 == cur.e0) {   // the no-k-step marker stage: nothing to load
        if (++s == kStages) {
          s = 0;
          ph ^= 1;
        }
        continue;
      }
      const int32_t J = static_cast<int32_t>(cur.t % GN);
      for (int64_t eb = cur.e0; eb < cur.e1; eb += 32) {
        const int cnt = static_cast<int>(cur.e1 - eb < 32 ? cur.e1 - eb : 32);
        if (lane < cnt) sentB[lane] = ment[eb + lane];
        __syncwarp();
        if (lane == 0) {
          for (int q = 0; q < cnt; ++q) {
            const uint4 en = sentB[q];
            const uint32_t cols = en.x >> 24;
            const bool wide = kWide && (en.w >> 31) != 0u;
            const int32_t k0 = static_cast<int32_t>(en.x & 0xFFFFu) * 32;
            uint8_t* bdst = smem + s * kStageBytes + kASlot;
            mbar_wait(&empty[s], ph ^ 1);
            if (dbg & 2) {
            } else if (use3d == 2) {
              // atom a (columns [64a, 64a+64) of the macro-tile) lands at bdst + a * atom bytes;
              // 2-D boxes [32|64 k x 64 n] SWIZZLE_128B, TMA zero fill beyond N
              const int c0 = __ffs(cols) - 1, c1 = 32 - __clz(cols);
              const int abytes = wide ? 8192 : 4096;
              const CUtensorMap* bm = wide ? &mp.b64w : &mp.b64;
              for (int a = c0 >> 1; a < ((c1 + 1) >> 1); ++a)
                tma_load_2d(bdst + a * abytes, bm, &full[s], J * 256 + a * 64, k0);
            } else if (use3d) {
              const int c0 = __ffs(cols) - 1, len = (32 - __clz(cols)) - c0;
              const int box = wide ? 4096 : 2048;
              const CUtensorMap* bm = wide ? mp.b2 : mp.b1;
              const int jb = J * 8;
              int off = c0;
              if (len == 8) {
                tma_load_3d(bdst, &bm[0], &full[s], 0, k0, jb);
              } else {
                if (len & 4) { tma_load_3d(bdst + off * box, &bm[1], &full[s], 0, k0, jb + off); off += 4; }
                if (len & 2) { tma_load_3d(bdst + off * box, &bm[2], &full[s], 0, k0, jb + off); off += 2; }
                if (len & 1) { tma_load_3d(bdst + off * box, &bm[3], &full[s], 0, k0, jb + off); }
              }
            } else {
              // ragged N: one 2-D TMA per needed box (only 32-deep k-steps are emitted)
#pragma unroll
              for (int lj = 0; lj < 8; ++lj)
                if ((cols >> lj) & 1u) tma_load_2d(bdst + lj * 2048, &mp.b2d, &full[s], J * 256 + lj * 32, k0);
            }
            if (++s == kStages) {
              s = 0;
              ph ^= 1;
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1 || (kCtas == 1 && warp == 2)) {
    // ------------------------------------------------------------- MMA issuer
    // kCtas == 2: one issuer, full 256-column tile.  kCtas == 1: warp 1 issues columns
    // [0, 128), warp 2 columns [128, 256) of every k-step (runs clipped to the half).
    const int hsel = kCtas == 1 ? warp - 1 : 0;
    if (lane == 0) {
      constexpr uint32_t idesc_base = idesc_f16(kFmt, 128, 0, 0, 1);
      constexpr uint32_t idesc_full = idesc_base | (8u << 19);   // N = 256, no lane mask
      const uint32_t base_addr = smem_u32(smem);
      const uint32_t srun_addr = smem_u32(srun);
      const uint64_t zdesc = smem_desc(smem_u32(sZero), 0, 0, kLayoutSW64);   // all strides 0: reads the zero atom
      const unsigned long long tk0 = clock64();
      unsigned long long m_te = 0, m_fu = 0, m_mma = 0, m_cm = 0, n_mma = 0;
      uint32_t ph = 0;
      int64_t tile_it = 0;
      int buf = 0;
      uint32_t dcol = tbase;
      bool fin = false;
      while (!fin) {
#pragma unroll 1
        for (int st = 0; st < kStages; ++st) {
          const unsigned long long t = prof ? clock64() : 0;
          mbar_wait(&full[st], ph);
          if (prof) m_fu += clock64() - t;
          tc_fence_after();
          uint4 rs;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(rs.x), "=r"(rs.y), "=r"(rs.z), "=r"(rs.w)
                       : "r"(srun_addr + st * 16));
          const uint32_t fl = rs.w;
          if (fl & kEnd) {
            fin = true;
            break;
          }
          if (fl & kFirst) {
            buf = static_cast<int>(tile_it % kBufs);
            const unsigned long long tw0 = prof ? clock64() : 0;
            mbar_wait(&tempty[buf], static_cast<uint32_t>((tile_it / kBufs) & 1));
            if (prof) m_te += clock64() - tw0;
            tc_fence_after();
            dcol = tbase + static_cast<uint32_t>(buf) * 256u + (kCtas == 1 ? static_cast<uint32_t>(hsel) * 128u : 0u);
            umma_f16(dcol, zdesc, zdesc, kCtas == 1 ? (idesc_base | (4u << 19)) : idesc_full, 0u, 0u, 0u, 0u, 0u);   // D = 0
          }
          const unsigned long long tm0 = prof ? clock64() : 0;
          if (!(fl & kNoStep) && !(dbg & 1)) {
            // A: K-major, SW64 rows of 32 (SBO 512) or SW128 rows of 64 (SBO 1024); +32 B per K=16
            // B: MN-major SW64 boxes of 32 columns, 32 or 64 rows deep (LBO = box size); +1024 B per K=16
            const uint32_t a_addr = base_addr + st * kStageBytes, b_addr = a_addr + kASlot;
            const bool wide = kWide && (fl >> 31) != 0u;
            const uint64_t ad = wide ? smem_desc(a_addr, 16, 1024, kLayoutSW128) : smem_desc(a_addr, 16, 512, kLayoutSW64);
            const bool b128 = use3d == 2;
            // bmode 2: B atoms of 64 columns x 32|64 k rows, SW128 (LBO = atom bytes, SBO = 1024,
            // +2048 B per K=16); bmode 0/1: 32-column SW64 boxes (LBO = box, SBO = 512, +1024 B)
            const uint32_t box = b128 ? (wide ? 8192u : 4096u) : (wide ? 4096u : 2048u);
            const uint64_t bd = b128 ? smem_desc(b_addr, box, 1024, kLayoutSW128) : smem_desc(b_addr, box, 512, kLayoutSW64);
            const uint32_t kstep = b128 ? 128u : 64u;   // descriptor units (16 B) per K=16
            const uint32_t nr = (rs.x >> 16) & 15u;
            if (kCtas == 1) {
              // split issuer: this warp's half [4h, 4h + 4) of the column tiles
              const uint32_t lo = 4u * static_cast<uint32_t>(hsel), hi = lo + 4u;
              const int nk = wide ? 4 : 2;
              if (nr == 1u && rs.y == kFullRun) {
                const uint32_t idesc = idesc_base | (4u << 19);   // N = 128
                const uint64_t bj = bd + static_cast<uint64_t>(lo * (box >> 4));
                for (int kk = 0; kk < nk; ++kk) umma_f16(dcol, ad + 2 * kk, bj + 64 * kk, idesc, 1u, 0u, 0u, 0u, 0u);
                if (prof) n_mma += nk;
              } else {
                uint32_t cw = rs.y;
                for (uint32_t rr = 0; rr < nr; ++rr) {
                  if (rr == 3) cw = rs.z;
                  if (rr == 6) cw = rs.w;
                  const uint32_t w = cw & 0x3FFu;
                  cw >>= 10;
                  const uint32_t r0 = w & 7u, r1 = r0 + ((w >> 3) & 7u) + 1u, pat = w >> 6;
                  const uint32_t j0 = r0 > lo ? r0 : lo, j1 = r1 < hi ? r1 : hi;
                  if (j1 <= j0) continue;
                  const uint32_t idesc = idesc_base | ((j1 - j0) << 19);
                  const uint32_t m0 = (pat & 1u) - 1u, m1 = ((pat >> 1) & 1u) - 1u;
                  const uint32_t m2 = ((pat >> 2) & 1u) - 1u, m3 = ((pat >> 3) & 1u) - 1u;
                  const uint64_t bj = bd + static_cast<uint64_t>(j0 * (box >> 4));
                  const uint32_t d = dcol + (j0 - lo) * 32u;
                  for (int kk = 0; kk < nk; ++kk) umma_f16(d, ad + 2 * kk, bj + 64 * kk, idesc, 1u, m0, m1, m2, m3);
                  if (prof) n_mma += nk;
                }
              }
            } else if (nr == 1u && rs.y == kFullRun) {
              umma_f16(dcol, ad, bd, idesc_full, 1u, 0u, 0u, 0u, 0u);
              umma_f16(dcol, ad + 2, bd + kstep, idesc_full, 1u, 0u, 0u, 0u, 0u);
              if (prof) n_mma += 2;
              if (wide) {
                umma_f16(dcol, ad + 4, bd + 2 * kstep, idesc_full, 1u, 0u, 0u, 0u, 0u);
                umma_f16(dcol, ad + 6, bd + 3 * kstep, idesc_full, 1u, 0u, 0u, 0u, 0u);
              }
            } else if (b128) {
              const int nk = wide ? 4 : 2;
              uint32_t cw = rs.y;
              for (uint32_t rr = 0; rr < nr; ++rr) {
                if (rr == 3) cw = rs.z;
                if (rr == 6) cw = rs.w;
                const uint32_t w = cw & 0x3FFu;
                cw >>= 10;
                uint32_t j0 = w & 7u, len = ((w >> 3) & 7u) + 1u;
                const uint32_t pat = w >> 6;
                const uint32_t m0 = (pat & 1u) - 1u, m1 = ((pat >> 1) & 1u) - 1u;   // 0 keep, ~0 disable
                const uint32_t m2 = ((pat >> 2) & 1u) - 1u, m3 = ((pat >> 3) & 1u) - 1u;
                // a run may start mid-atom (odd j0: +64 B inside the 128-byte swizzled row) but
                // the N walk only crosses atoms from an atom start: split odd starts of len > 1
                while (len) {
                  const uint32_t l = (j0 & 1u) ? 1u : len;
                  const uint32_t idesc = idesc_base | (l << 19);
                  const uint64_t bj = bd + (((j0 >> 1) * box + (j0 & 1u) * 64u) >> 4);
                  const uint32_t d = dcol + j0 * 32u;
                  for (int kk = 0; kk < nk; ++kk) umma_f16(d, ad + 2 * kk, bj + kstep * kk, idesc, 1u, m0, m1, m2, m3);
                  if (prof) n_mma += nk;
                  j0 += l;
                  len -= l;
                }
              }
            } else {
              const int nk = wide ? 4 : 2;
              uint32_t cw = rs.y;
              for (uint32_t rr = 0; rr < nr; ++rr) {
                if (rr == 3) cw = rs.z;
                if (rr == 6) cw = rs.w;
                const uint32_t w = cw & 0x3FFu;
                cw >>= 10;
                const uint32_t j0 = w & 7u, len = ((w >> 3) & 7u) + 1u, pat = w >> 6;
                const uint32_t idesc = idesc_base | (len << 19);        // N = 32*len -> N>>3 = 4*len at bit 17
                const uint32_t m0 = (pat & 1u) - 1u, m1 = ((pat >> 1) & 1u) - 1u;   // 0 keep, ~0 disable
                const uint32_t m2 = ((pat >> 2) & 1u) - 1u, m3 = ((pat >> 3) & 1u) - 1u;
                const uint64_t bj = bd + static_cast<uint64_t>(j0 * (box >> 4));
                const uint32_t d = dcol + j0 * 32u;
                for (int kk = 0; kk < nk; ++kk) umma_f16(d, ad + 2 * kk, bj + 64 * kk, idesc, 1u, m0, m1, m2, m3);
                if (prof) n_mma += nk;
              }
            }
          }
          const unsigned long long tm1 = prof ? clock64() : 0;
          umma_commit(&empty[st]);
          if (fl & kLast) {
            umma_commit(&tfull[buf]);
            ++tile_it;
          }
          if (prof) {
            const unsigned long long tm2 = clock64();
            m_mma += tm1 - tm0;
            m_cm += tm2 - tm1;
          }
        }
        ph ^= 1;
      }
      if (prof && warp == 1) {
        prof[blockIdx.x * 16 + 2] = m_te;
        prof[blockIdx.x * 16 + 3] = m_fu;
        prof[blockIdx.x * 16 + 6] = clock64() - tk0;
        prof[blockIdx.x * 16 + 12] = m_mma;
        prof[blockIdx.x * 16 + 13] = m_cm;
        prof[blockIdx.x * 16 + 14] = n_mma;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // --------------------------------------------------------------- epilogue
    const int q = warp & 3;            // TMEM lane quadrant (warp % 4)
    const int half = (warp - 4) >> 2;  // columns [128*half, 128*half + 128)
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      for (int b = 0; b < kBufs; ++b) mbar_arrive(&tempty[b]);
    }
    const int t0 = lane & 3, t1 = lane >> 2;
    unsigned long long e_w = 0, e_d = 0;
    // one zero-fill unit: 8 rows x 256 columns of an empty macro-tile; false when none is left
    // units are dealt round-robin to the grid's epilogue warps (no claim atomics: tens of
    // thousands of same-address atomics serialise in L2)
    const int64_t n_units = n_empty * 16;
    const int64_t u_stride = static_cast<int64_t>(gridDim.x) * kEpiWarps;
    int64_t u_next = static_cast<int64_t>(blockIdx.x) * kEpiWarps + (warp - 4);
    auto zero_unit = [&]() -> bool {
      if (u_next >= n_units) return false;
      const int64_t u = u_next;
      u_next += u_stride;
      const int64_t t = order[n_work + u / 16];
      const int64_t r0 = (t / GN) * 128 + (u % 16) * 8, c0 = (t % GN) * 256;
      // bulk (TMA-engine) stores of the 1 KB zero buffer: one instruction per row, so the
      // zero-fill costs the SM a handful of issues instead of 16-byte stores from every lane
      const int64_t ncol = N - c0 < 256 ? N - c0 : 256;
      const uint32_t bytes = static_cast<uint32_t>(ncol * 4) & ~15u;
      if (lane == 0) {
        for (int r = 0; r < 8; ++r) {
          const int64_t row = r0 + r;
          if (row >= M) break;
          if (bytes) bulk_store_1d(C + row * ldc + c0, sZero, bytes);
          for (int64_t cc = bytes / 4; cc < ncol; ++cc) C[row * ldc + c0 + cc] = 0.f;
        }
        bulk_commit_group();
      }
      return true;
    };
    int tq_s = 0;
    uint32_t tq_ph = 0;
    for (int64_t it = 0;; ++it) {
      mbar_wait(&tq_full[tq_s], tq_ph);
      const TileInfo cur = tq[tq_s];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tq_empty[tq_s]);
      if (++tq_s == kTQ) {
        tq_s = 0;
        tq_ph ^= 1;
      }
      if (cur.t < 0) break;
      const int64_t I = cur.t / GN, J = cur.t % GN;
      const int buf = static_cast<int>(it % kBufs);
      const unsigned long long te0 = prof ? clock64() : 0;
      if (!(dbg & 16)) {   // zero-fill empty tiles while waiting for the accumulator
        const uint32_t par = static_cast<uint32_t>((it / kBufs) & 1);
        while (!mbar_try_wait(&tfull[buf], par))
          if (!zero_unit()) {
            mbar_wait(&tfull[buf], par);
            break;
          }
      } else {
        mbar_wait(&tfull[buf], static_cast<uint32_t>((it / kBufs) & 1));
      }
      const unsigned long long te1 = prof ? clock64() : 0;
      e_w += te1 - te0;
      tc_fence_after();
      if (cur.part) {
        // ---- stream-K partial tile: own partial -> scratch, ticket, last contributor combines
        const int64_t w0 = wpre[cur.i], w1 = wpre[cur.i + 1];
        const int64_t w_last = entry_w(ment[mstart[cur.t] + mcount[cur.t] - 1]);
        const int64_t c_lo = sk_owner(w0, skW, skG), c_hi = sk_owner(w1 - w_last, skW, skG);
        float* mine = sk_scratch + sk_slot(skC, c_lo, w0, skW, skG) * (128 * 256);
#pragma unroll 1
        for (int hh = 0; hh < 4; ++hh) {
          const int lh = hh & 1;
          const int c0 = half * 128 + (hh >> 1) * 64;
          uint32_t v[32];
          tmem_ld_16x256b_x8(tbase + ((static_cast<uint32_t>(q * 32 + 16 * lh)) << 16) + buf * 256 + c0, v);
          tmem_wait_ld();
          const int ra = q * 32 + 16 * lh + t1, rb = ra + 8;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int col = c0 + 8 * i + 2 * t0;
            __stcg(reinterpret_cast<float2*>(mine + ra * 256 + col),
                   make_float2(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1])));
            __stcg(reinterpret_cast<float2*>(mine + rb * 256 + col),
                   make_float2(__uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3])));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);   // the accumulator is no longer needed
        asm volatile("bar.sync 1, 256;" ::: "memory");   // all 8 epilogue warps wrote their part
        if (warp == 4 && lane == 0) {
          __threadfence();
          const unsigned int old = atomicAdd(sk_ticket + cur.i, 1u);
          const bool last = static_cast<int64_t>(old) == c_hi - c_lo;
          if (last) sk_ticket[cur.i] = 0u;        // self-reset for the next launch
          __threadfence();
          *sk_flag = last ? 1u : 0u;
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (*sk_flag) {
          // partials summed in CTA order c_lo, c_lo+1, ... (deterministic): the first slot is
          // sk_slot(c_lo), every later contributor's is 2c (its first chunk).  Coalesced:
          // epilogue thread e handles float4 f = e + 256 m of the 128 x 256 tile.
          const int64_t I0 = I * 128, J0 = J * 256;
          const int nc = static_cast<int>(c_hi - c_lo + 1);
          const float4* src0 = reinterpret_cast<const float4*>(sk_scratch + sk_slot(c_lo, c_lo, w0, skW, skG) * (128 * 256));
          const float4* srcn = reinterpret_cast<const float4*>(sk_scratch + 2 * (c_lo + 1) * (128 * 256));
          const int e = static_cast<int>(threadIdx.x) - 128;
#pragma unroll 1
          for (int m0 = 0; m0 < 32; m0 += 4) {
            float4 acc[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) acc[m] = __ldcg(src0 + e + 256 * (m0 + m));
            for (int n = 1; n < nc; ++n) {
              const float4* src = srcn + static_cast<int64_t>(n - 1) * (2 * 128 * 256 / 4);
              float4 x[4];
#pragma unroll
              for (int m = 0; m < 4; ++m) x[m] = __ldcg(src + e + 256 * (m0 + m));
#pragma unroll
              for (int m = 0; m < 4; ++m) {
                acc[m].x += x[m].x;
                acc[m].y += x[m].y;
                acc[m].z += x[m].z;
                acc[m].w += x[m].w;
              }
            }
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const int f = e + 256 * (m0 + m);
              const int64_t row = I0 + (f >> 6), gc = J0 + (f & 63) * 4;
              if (row < M) {
                float* dst = C + row * ldc + gc;
                if (gc + 3 < N) {
                  __stcs(reinterpret_cast<float4*>(dst), kGen ? axpby4(ab, acc[m], dst) : acc[m]);
                } else {
                  if (gc < N) dst[0] = kGen ? axpby1(ab, acc[m].x, dst) : acc[m].x;
                  if (gc + 1 < N) dst[1] = kGen ? axpby1(ab, acc[m].y, dst + 1) : acc[m].y;
                  if (gc + 2 < N) dst[2] = kGen ? axpby1(ab, acc[m].z, dst + 2) : acc[m].z;
                }
              }
            }
          }
        }
        if (prof) e_d += clock64() - te1;
        continue;
      }
      if (kGen && (co.nC != nullptr || co.clow != nullptr)) {
        // ---- chained output: C (alpha/beta applied), optional rounded copy, tile norms
        double tsum[4] = {0.0, 0.0, 0.0, 0.0};   // tiles (I*4+q, J*8 + half*4 + t)
#pragma unroll 1
        for (int hh = 0; hh < 4; ++hh) {
          const int lh = hh & 1;
          const int c0 = half * 128 + (hh >> 1) * 64;
          uint32_t v[32];
          tmem_ld_16x256b_x8(tbase + ((static_cast<uint32_t>(q * 32 + 16 * lh)) << 16) + buf * 256 + c0, v);
          tmem_wait_ld();
          const int64_t ra = I * 128 + q * 32 + 16 * lh + t1;
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
              if (two) {
                x = axpby2(ab, x, cp);
                __stcs(reinterpret_cast<float2*>(cp), x);
              } else {
                x.x = axpby1(ab, x.x, cp);
                x.y = 0.f;
                *cp = x.x;
              }
              if (co.clow != nullptr) {   // round to the plan's input type; norms of what is stored
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
        if (lane == 0) mbar_arrive(&tempty[buf]);
        if (co.nC != nullptr) {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            double x = tsum[t];
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            const int64_t ti = I * 4 + q, tj = J * 8 + half * 4 + t;
            if (lane == 0 && ti * 32 < M && tj * 32 < N) co.nC[ti * co.ldn + tj] = sqrt(x);
          }
        }
        if (prof) e_d += clock64() - te1;
        continue;
      }
#pragma unroll 1
      for (int hh = 0; hh < 4; ++hh) {
        const int lh = hh & 1;                         // lanes [16*lh, 16*lh + 16) of the quadrant
        const int c0 = half * 128 + (hh >> 1) * 64;    // 64-column block
        uint32_t v[32];
        if (dbg & 8) continue;
        tmem_ld_16x256b_x8(tbase + ((static_cast<uint32_t>(q * 32 + 16 * lh)) << 16) + buf * 256 + c0, v);
        tmem_wait_ld();
        if ((dbg & 4) && v[0] != 0x7fc00001u) continue;
        const int64_t ra = I * 128 + q * 32 + 16 * lh + t1, rb = ra + 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int64_t col = J * 256 + c0 + 8 * i + 2 * t0;
          float* ca = C + ra * ldc + col;
          float* cb = C + rb * ldc + col;
          const float2 pa = make_float2(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]));
          const float2 pb = make_float2(__uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
          if (col + 1 < N) {
            if (ra < M) __stcs(reinterpret_cast<float2*>(ca), kGen ? axpby2(ab, pa, ca) : pa);
            if (rb < M) __stcs(reinterpret_cast<float2*>(cb), kGen ? axpby2(ab, pb, cb) : pb);
          } else if (col < N) {
            if (ra < M) *ca = kGen ? axpby1(ab, pa.x, ca) : pa.x;
            if (rb < M) *cb = kGen ? axpby1(ab, pb.x, cb) : pb.x;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      if (prof) e_d += clock64() - te1;
    }
    while (zero_unit()) {
    }
    if (lane == 0) bulk_wait_group<0>();   // zero-fill stores complete before the CTA retires
    if (prof && warp == 4 && lane == 0) {
      prof[blockIdx.x * 16 + 4] = e_w;
      prof[blockIdx.x * 16 + 5] = e_d;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<kTmemCols>(tbase);
  if (prof && threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    prof[blockIdx.x * 16 + 9] = g;
  }
}

// Stream-K weights: wt[i] = sum of entry_w over the entries of the tile at LPT position i
// (one warp per position), then wpre = exclusive prefix of wt in place (one block, each
// thread owns kPreR consecutive items), wpre[n] = total.  Empty tiles (the LPT tail) add 0.
__global__ void __launch_bounds__(256) tile_weight_kernel(const int32_t* __restrict__ order,
                                                          const int64_t* __restrict__ mstart,
                                                          const int64_t* __restrict__ mcount,
                                                          const uint4* __restrict__ ment, int64_t n,
                                                          int64_t* __restrict__ wt) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int64_t t = order[i], ms = mstart[t], cnt = mcount[t];
  int64_t w = 0;
  for (int64_t e = lane; e < cnt; e += 32) w += entry_w(ment[ms + e]);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
  if (lane == 0) wt[i] = w;
}

constexpr int kPreThreads = 1024, kPreR = 16;
__global__ void __launch_bounds__(kPreThreads) lpt_prefix_kernel(int64_t n, int64_t* __restrict__ wpre) {
  __shared__ int64_t s_warp[kPreThreads / 32];
  __shared__ int64_t s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += static_cast<int64_t>(kPreThreads) * kPreR) {
    const int64_t my0 = base + static_cast<int64_t>(threadIdx.x) * kPreR;
    int64_t v[kPreR], tot = 0;
#pragma unroll
    for (int r = 0; r < kPreR; ++r) {
      v[r] = my0 + r < n ? wpre[my0 + r] : 0;
      tot += v[r];
    }
    int64_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int64_t w = s_warp[lane];
      int64_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      s_warp[lane] = wi - w;   // exclusive warp offsets
    }
    __syncthreads();
    int64_t run = s_carry + s_warp[warp] + incl - tot;
#pragma unroll
    for (int r = 0; r < kPreR; ++r) {
      if (my0 + r < n) wpre[my0 + r] = run;
      run += v[r];
    }
    __syncthreads();
    if (threadIdx.x == kPreThreads - 1) s_carry = run;
    __syncthreads();
  }
  if (threadIdx.x == 0) wpre[n] = s_carry;
}

template <uint32_t kFmt, int kCtas, bool kWide, bool kGen>
spamm_status launch_cfg(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                        cudaStream_t s, CUtensorMapDataType dt) {
  Maps mp;
  std::memset(&mp, 0, sizeof(mp));
  SPAMM_TRY(encode_tmap_2d(&mp.a1, dt, 2, A, p.K, p.M, lda, 32, 128, CU_TENSOR_MAP_SWIZZLE_64B));
  SPAMM_TRY(encode_tmap_2d(&mp.a2, dt, 2, A, p.K, p.M, lda, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B));
  SPAMM_TRY(encode_tmap_2d(&mp.b2d, dt, 2, B, p.N, p.K, ldb, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B));
  // B as stacked [32|64 k][32 n] boxes: dims {32 n, K, N/32} with strides {ldb, 32} elements
  // (a non-monotonic stride; verified by scripts/probe_tma3d.cu).  Only when N % 32 == 0:
  // the inner 32 columns of the last box must exist.
  // B layout: 1 (default) = stacked 32-column 3-D boxes (needs N % 32 == 0, else 0 = one 2-D
  // 32-column box per needed tile); 2 = 64-column atoms with 128-byte rows (half the TMA
  // requests per byte; parity-green but measured slower at the bench point: 198 vs 182 us,
  // the extra columns of partially needed atoms and the split odd-start runs cost more)
  static const int bmode_env = getenv("SPAMM_UMMA_BMODE") ? atoi(getenv("SPAMM_UMMA_BMODE")) : 1;
  const int use3d = (bmode_env == 2 && kCtas == 2) ? 2 : (bmode_env >= 1 && (p.N % 32) == 0 ? 1 : 0);
  if (use3d == 2) {
    SPAMM_TRY(encode_tmap_2d(&mp.b64, dt, 2, B, p.N, p.K, ldb, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B));
    SPAMM_TRY(encode_tmap_2d(&mp.b64w, dt, 2, B, p.N, p.K, ldb, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B));
  }
  if (use3d == 1) {
    const uint32_t nbs[4] = {8, 4, 2, 1};
    for (int q = 0; q < 4; ++q) {
      SPAMM_TRY(encode_tmap_3d(&mp.b1[q], dt, B, 32, p.K, p.N / 32, static_cast<uint64_t>(ldb) * 2, 64, 32, 32,
                               nbs[q], CU_TENSOR_MAP_SWIZZLE_64B));
      SPAMM_TRY(encode_tmap_3d(&mp.b2[q], dt, B, 32, p.K, p.N / 32, static_cast<uint64_t>(ldb) * 2, 64, 32, 64,
                               nbs[q], CU_TENSOR_MAP_SWIZZLE_64B));
    }
  }
  constexpr size_t kSmemBytes = Cfg<kCtas, kWide>::kSmemBytes;
  auto kern = spamm_mul_umma_kernel<kFmt, kCtas, kWide, kGen>;
  static bool attr_set = false;
  if (!attr_set) {
    SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes)));
    attr_set = true;
  }
  const int64_t n_tiles = (p.row_end_macro - p.row_begin_macro) * p.GN;
  if (n_tiles <= 0) return SPAMM_OK;
  const int64_t slots = static_cast<int64_t>(p.num_sms) * kCtas;
  // stream-K (SPAMM_STREAMK=1) balances the k-step stream exactly but measured slower at the
  // bench point (partial-tile combine and zero-fill tails); dynamic LPT is default
  static const bool streamk_env = getenv("SPAMM_STREAMK") && atoi(getenv("SPAMM_STREAMK")) == 1;
  // (stream-K zero-fills empty tiles with bulk stores: only for beta == 0)
  const bool chain = p.out_norms || p.out_low != nullptr;
  const bool streamk = streamk_env && p.beta == 0.0 && !chain;
  // stream-K splits tiles, so it uses every slot even when there are fewer tiles than slots
  const int grid = static_cast<int>(streamk ? slots : (n_tiles < slots ? n_tiles : slots));
  constexpr int kProfMax = 512;
  static unsigned long long* prof = nullptr;
  if (getenv("SPAMM_DEBUG_UMMA_PROF") && !prof) cudaMalloc(&prof, kProfMax * 16 * 8);
  if (prof && grid > kProfMax) return fail(SPAMM_E_UNSUPPORTED, "profiling supports at most 512 CTAs");
  if (prof) cudaMemsetAsync(prof, 0, kProfMax * 16 * 8, s);
  SPAMM_CUDA_TRY(cudaMemsetAsync(p.sched, 0, 2 * sizeof(unsigned int), s));
  static const int dbg = getenv("SPAMM_DEBUG_UMMA_MODE") ? atoi(getenv("SPAMM_DEBUG_UMMA_MODE")) : 0;
  if (streamk) {
    const int64_t nmac = p.GM * p.GN;
    if (p.sk_cap_tiles < nmac + 1 || p.sk_cap_slots < 2 * slots) {
      if (p.sk_scratch) cudaFree(p.sk_scratch);
      if (p.sk_ticket) cudaFree(p.sk_ticket);
      if (p.sk_wpre) cudaFree(p.sk_wpre);
      p.sk_scratch = nullptr;
      p.sk_ticket = nullptr;
      p.sk_wpre = nullptr;
      p.sk_cap_tiles = p.sk_cap_slots = 0;
      if (cudaMalloc(&p.sk_scratch, sizeof(float) * 128 * 256 * static_cast<size_t>(2 * slots)) != cudaSuccess ||
          cudaMalloc(&p.sk_ticket, sizeof(unsigned int) * static_cast<size_t>(nmac + 1)) != cudaSuccess ||
          cudaMalloc(&p.sk_wpre, sizeof(int64_t) * static_cast<size_t>(nmac + 1)) != cudaSuccess) {
        cudaGetLastError();
        return fail(SPAMM_E_NOMEM, "stream-K workspace allocation failed");
      }
      SPAMM_CUDA_TRY(cudaMemset(p.sk_ticket, 0, sizeof(unsigned int) * static_cast<size_t>(nmac + 1)));
      p.sk_cap_tiles = nmac + 1;
      p.sk_cap_slots = 2 * slots;
    }
    // LPT order of the multiplied macro-row range: weights, then their prefix
    tile_weight_kernel<<<static_cast<unsigned>((n_tiles + 7) / 8), 256, 0, s>>>(p.order, p.mstart, p.Uw, p.macro_run,
                                                                             n_tiles, p.sk_wpre);
    lpt_prefix_kernel<<<1, kPreThreads, 0, s>>>(n_tiles, p.sk_wpre);
    count_launch(2);
    SPAMM_CUDA_TRY(cudaGetLastError());
  }
  kern<<<grid, kThreads, kSmemBytes, s>>>(mp, use3d, p.mstart, p.Uw, p.macro_run, p.order,
                                                                 n_tiles, p.GN, C, ldc, p.M, p.N, p.sched,
                                                                 (streamk || ((dbg & 32) && p.beta == 0.0)) ? p.hist : nullptr,
                                                                 streamk ? p.sk_wpre : nullptr, p.sk_scratch, p.sk_ticket,
                                                                 Axpby{static_cast<float>(p.alpha), static_cast<float>(p.beta)},
                                                                 ChainOut{p.out_norms ? p.nC : nullptr, p.BN, p.out_low, p.out_ldl},
                                                                 prof, dbg);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  if (prof) {
    static unsigned long long h[kProfMax * 16];
    cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double acc[16] = {0};
    double mn = 1e30, mx = 0;
    for (int c = 0; c < grid; ++c) {
      for (int k = 0; k < 16; ++k) acc[k] += static_cast<double>(h[c * 16 + k]) / grid;
      mn = std::min(mn, static_cast<double>(h[c * 16 + 6]));
      mx = std::max(mx, static_cast<double>(h[c * 16 + 6]));
    }
    unsigned long long g0 = ~0ull, g1 = 0;
    for (int c = 0; c < grid; ++c) {
      g0 = std::min(g0, h[c * 16 + 8]);
      g1 = std::max(g1, h[c * 16 + 9]);
    }
    int late = 0;
    double dur = 0, pro = 0;
    for (int c = 0; c < grid; ++c) pro += static_cast<double>(h[c * 16 + 10] - h[c * 16 + 8]) / grid;
    fprintf(stderr, "[umma prof] mean prologue (start -> TMEM allocated) %.2f us\n", pro * 1e-3);
    for (int c = 0; c < grid; ++c) {
      late += (h[c * 16 + 8] - g0) > 5000ull;
      dur += static_cast<double>(h[c * 16 + 9] - h[c * 16 + 8]) / grid;
    }
    fprintf(stderr, "[umma prof] grid %d: span %.1f us, mean CTA %.1f us, CTAs starting >5us late: %d\n", grid,
            (g1 - g0) * 1e-3, dur * 1e-3, late);
    fprintf(stderr,
            "[umma prof] cycles/CTA: MMA thread %.0f (min %.0f max %.0f) tmem-empty wait %.0f stage-full wait %.0f | "
            "producer %.0f stage-empty wait %.0f | epilogue tmem-full wait %.0f drain %.0f\n",
            acc[6], mn, mx, acc[2], acc[3], acc[7], acc[1], acc[4], acc[5]);
    fprintf(stderr, "[umma prof] producer claim %.0f | MMA-issue section %.0f commit %.0f MMAs/CTA %.0f\n", acc[11],
            acc[12], acc[13], acc[14]);
    if (getenv("SPAMM_DEBUG_UMMA_PROF_CTA")) {
      for (int c = 0; c < grid; ++c)
        fprintf(stderr, "[umma cta] %d mma %llu nmma %llu full %llu tempty %llu epi_wait %llu drain %llu start %.2f end %.2f\n", c,
                h[c * 16 + 6], h[c * 16 + 14], h[c * 16 + 3], h[c * 16 + 2], h[c * 16 + 4], h[c * 16 + 5],
                (h[c * 16 + 8] - g0) * 1e-3, (h[c * 16 + 9] - g0) * 1e-3);
    }
  }
  return SPAMM_OK;
}


template <uint32_t kFmt>
spamm_status launch_fmt(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                        cudaStream_t s, CUtensorMapDataType dt) {
  if (p.alpha != 1.0 || p.beta != 0.0 || p.out_norms || p.out_low != nullptr) {   // general epilogue
    if (umma_variant_wide(p.umma_variant)) return launch_cfg<kFmt, 2, true, true>(p, A, lda, B, ldb, C, ldc, s, dt);
    return launch_cfg<kFmt, 2, false, true>(p, A, lda, B, ldb, C, ldc, s, dt);
  }
  switch (p.umma_variant) {
    case 0:
      return launch_cfg<kFmt, 2, false, false>(p, A, lda, B, ldb, C, ldc, s, dt);
    case 1:
      return launch_cfg<kFmt, 2, true, false>(p, A, lda, B, ldb, C, ldc, s, dt);
    case 4:
      return launch_cfg<kFmt, 1, false, false>(p, A, lda, B, ldb, C, ldc, s, dt);
    default:
      return launch_cfg<kFmt, 1, true, false>(p, A, lda, B, ldb, C, ldc, s, dt);
  }
}

}  // namespace

int umma_variant_from_env() {
  const char* v = getenv("SPAMM_UMMA_VARIANT");
  // default 5: 256 x 256 macro-tiles with two MMA issuers (multiply_dual.cu; measured fastest at
  // the bench point).  Plans whose shape it cannot serve fall back to 0 (api.cu).
  const int x = v ? atoi(v) : 5;
  return x >= 0 && x <= 5 ? x : 5;
}
bool umma_variant_wide(int v) { return v == 1 || v == 2; }

spamm_status launch_multiply_umma(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C,
                                  int64_t ldc, cudaStream_t s) {
  if (p.prec == SPAMM_BF16) return launch_fmt<1>(p, A, lda, B, ldb, C, ldc, s, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
  return launch_fmt<0>(p, A, lda, B, ldb, C, ldc, s, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
}

}  // namespace spamm
