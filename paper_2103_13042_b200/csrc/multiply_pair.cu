// multiply_pair.cu -- stage 3, tensor-core path on CTA pairs (tensor-core multiplication
// kernel, Sec. 3.3, Alg. 3), BF16/FP16 inputs, FP32 accumulation.
//
// C[i,j] = sum_{kept k, ascending} A[i,k] * B[k,j]; the paper's FP32
// accumulator fragment becomes an FP32 accumulator in TMEM.
//
// B200 design: a cluster of two CTAs on one TPC computes 256 x 256 macro-tiles (8 x 8 C
// tiles of 32 x 32) with tcgen05.mma.cta_group::2 (M = 256): one thread of rank 0 issues
// every MMA for both SMs, each SM's tensor core reads its own 128 rows of A and the
// pair's B columns from both shared memories, and each SM accumulates its 128 x 256 half
// in its own TMEM.  Against one CTA per 128 x 256 tile this halves the MMA instructions
// per SM, cuts the bytes each SM pulls from L2 per k-step by a third (A 128 rows + half
// the B columns), and frees TMEM for two accumulators per SM (the epilogue of one tile
// overlaps the MMAs of the next).
//   * skip map (skipmap.cu, 8 x 8 keep masks): each k-step is a list of runs -- adjacent
//     C-tile columns with the same 8-bit row pattern; a run is ONE MMA of N = 32*len whose
//     disable-output-lane mask switches off the 32-row groups whose pair is skipped (exact
//     leaf-level skip semantics, Alg. 2 l.3-8).  Equal-mask k pairs are
//     merged into 64-deep k-steps;
//   * the rank-0 producer claims tiles (atomic counter, LPT order) and forwards each to the
//     peer through distributed shared memory; per k-step each CTA loads its A rows and its
//     half of every run's B columns (32-column SWIZZLE_64B boxes for even runs, 16-column
//     SWIZZLE_32B units for odd runs, as the pair MMA splits N in halves) with TMA that
//     completes on rank 0's stage barrier;
//   * MMA completion is multicast to both CTAs' stage / accumulator barriers; both CTAs'
//     epilogue warps drain their TMEM half with coalesced 8-byte stores and release the
//     accumulator on rank 0's barrier.
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

constexpr int kStages = 6;
constexpr int kASlot = 128 * 64 * 2;   // 16 KB: this CTA's A[128 x 32|64]
constexpr int kBSlot = 64 * 128 * 2;   // 16 KB: this CTA's halves of the runs' B columns (<= 128 x 64)
constexpr int kStageBytes = kASlot + kBSlot;
constexpr int kThreads = 384;          // w0 producer A + tile claims, w1 MMA (rank 0), w2 TMEM, w3 producer B,
                                       // w4-11 epilogue
constexpr int kEpiWarps = 8;
constexpr uint32_t kTmemCols = 512;    // 2 x (128 x 256 FP32) accumulators per SM
constexpr int kTQ = 4;                 // tile ring depth
// tile-queue consumers per tile: rank 0 producer B + epilogue, rank 1 producer A, B + epilogue
constexpr int kTqArrivals = (1 + kEpiWarps) + (2 + kEpiWarps);
constexpr size_t kSmemBytes = 1024 + static_cast<size_t>(kStages) * kStageBytes + 512 + 2048;

// entry x: k | nruns << 16 | wide << 19; stream flags added in shared memory (rank 0)
constexpr uint32_t kFirst = 1u << 24, kLast = 1u << 25, kNoStep = 1u << 26, kEnd = 1u << 27;
constexpr uint32_t kFullRun = 0u | (7u << 3) | (0xFFu << 6);   // j0 = 0, len = 8, all 8 row groups

struct TileInfo {
  int64_t t, e0, e1;
};

struct PairMaps {
  CUtensorMap a1, a2;     // A boxes {32, 128} SWIZZLE_64B, {64, 128} SWIZZLE_128B
  CUtensorMap b64[2][3];  // [32|64 deep][1, 2, 4 boxes]: 32-column SWIZZLE_64B boxes, dims {32, K, N/32}
  CUtensorMap b32[2][3];  // [32|64 deep][1, 2, 4 units]: 16-column SWIZZLE_32B units, dims {16, K, N/16}
};

__device__ __forceinline__ uint32_t run_word(const uint4& e, int q) {
  const uint32_t w = q < 2 ? e.y : (q < 4 ? e.z : e.w);
  return (q & 1) ? (w >> 16) : (w & 0xFFFFu);
}

template <uint32_t kFmt>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    spamm_mul_pair_kernel(const __grid_constant__ PairMaps mp, const int64_t* __restrict__ mcount,
                          const uint4* __restrict__ ment, const int32_t* __restrict__ order, int64_t n_tiles,
                          int64_t GN, int64_t BK, float* __restrict__ C, int64_t ldc, int64_t M, int64_t N,
                          unsigned int* __restrict__ sched, unsigned long long* __restrict__ prof) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sZero = smem + kStages * kStageBytes;   // 512-B zero atom (same offset in both CTAs)
  uint64_t* full = reinterpret_cast<uint64_t*>(sZero + 512);   // rank 0: stage loaded (both CTAs' bytes)
  uint64_t* empty = full + kStages;                              // each CTA: stage consumed
  uint64_t* tfull = empty + kStages;                             // each CTA: accumulator ready
  uint64_t* tempty = tfull + 2;                                  // rank 0: accumulator drained (both)
  uint64_t* tq_full = tempty + 2;                                // each CTA
  uint64_t* tq_empty = tq_full + kTQ;                            // rank 0
  uint4* srun = reinterpret_cast<uint4*>(tq_empty + kTQ);       // rank 0: [kStages] the stage's k-step
  uint4* sentA = srun + kStages;                                 // [32]
  uint4* sentB = sentA + 32;                                     // [32]
  TileInfo* tq = reinterpret_cast<TileInfo*>(sentB + 32);       // [kTQ]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq + kTQ);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  for (int i = threadIdx.x; i < 512 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sZero)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();   // the zero atom is read by tcgen05.mma (async proxy)
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * kEpiWarps);
    }
    for (int q = 0; q < kTQ; ++q) {
      mbar_init(&tq_full[q], 1);
      mbar_init(&tq_empty[q], kTqArrivals);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync();   // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  // rank 0's copies of the shared barriers, as cluster addresses
  const uint32_t full0 = mapa(smem_u32(full), 0), tempty0 = mapa(smem_u32(tempty), 0);
  const uint32_t tq_empty0 = mapa(smem_u32(tq_empty), 0);

  // consume tile-queue slot q (every role except rank 0's producer A)
  auto tq_take = [&](int q, uint32_t ph) -> TileInfo {
    mbar_wait(&tq_full[q], ph);
    const TileInfo ti = tq[q];
    __syncwarp();
    if (lane == 0) mbar_arrive_cluster(tq_empty0 + q * 8);
    return ti;
  };

  if (warp == 0) {
    // ------------------------------------------------- producer A (+ tile claims on rank 0)
    if (lane == 0) {
      tma_prefetch_desc(&mp.a1);
      tma_prefetch_desc(&mp.a2);
    }
    int s = 0;
    uint32_t ph = 0;
    int tq_s = 0;
    uint32_t tq_ph = 0;
    unsigned long long p_wait = 0;
    const unsigned long long p_t0 = clock64();
    auto claim = [&]() -> TileInfo {
      unsigned int idx = 0;
      if (lane == 0) idx = atomicAdd(sched, 1u);
      idx = __shfl_sync(0xffffffffu, idx, 0);
      TileInfo ti{-1, 0, 0};
      if (idx < n_tiles) {
        ti.t = order[idx];
        ti.e0 = ti.t * BK * 2;
        ti.e1 = ti.e0 + mcount[ti.t];
      }
      return ti;
    };
    TileInfo nxt{-1, 0, 0};
    if (rank == 0) nxt = claim();
    for (;;) {
      TileInfo cur;
      if (rank == 0) {
        cur = nxt;
        if (cur.t >= 0) nxt = claim();   // one ahead: the claim's latency hides behind this tile
        if (lane == 0) {
          mbar_wait(&tq_empty[tq_s], tq_ph ^ 1);
          tq[tq_s] = cur;
          const uint32_t peer = mapa(smem_u32(&tq[tq_s]), 1);
          st_cluster_u64(peer, static_cast<uint64_t>(cur.t));
          st_cluster_u64(peer + 8, static_cast<uint64_t>(cur.e0));
          st_cluster_u64(peer + 16, static_cast<uint64_t>(cur.e1));
          mbar_arrive(&tq_full[tq_s]);
          mbar_arrive_cluster(mapa(smem_u32(&tq_full[tq_s]), 1));   // release.cluster orders the stores
        }
        __syncwarp();
      } else {
        cur = tq_take(tq_s, tq_ph);
      }
      if (++tq_s == kTQ) {
        tq_s = 0;
        tq_ph ^= 1;
      }
      if (cur.t < 0 || cur.e1 == cur.e0) {   // end of stream, or a tile without k-steps (C = 0)
        if (rank == 0 && lane == 0) {
          mbar_wait(&empty[s], ph ^ 1);
          srun[s] = make_uint4(cur.t < 0 ? kEnd : (kFirst | kLast | kNoStep), 0u, 0u, 0u);
          mbar_arrive(&full[s]);
        }
        if (++s == kStages) {
          s = 0;
          ph ^= 1;
        }
        if (cur.t < 0) break;
        continue;
      }
      const int32_t arow = static_cast<int32_t>((cur.t / GN) * 256 + rank * 128);
      for (int64_t eb = cur.e0; eb < cur.e1; eb += 32) {
        const int cnt = static_cast<int>(cur.e1 - eb < 32 ? cur.e1 - eb : 32);
        if (lane < cnt) sentA[lane] = ment[eb + lane];
        __syncwarp();
        if (lane == 0) {
          for (int q = 0; q < cnt; ++q) {
            uint4 en = sentA[q];
            const bool wide = ((en.x >> 19) & 1u) != 0u;
            const int32_t k0 = static_cast<int32_t>(en.x & 0xFFFFu) * 32;
            const unsigned long long tw0 = prof ? clock64() : 0;
            mbar_wait(&empty[s], ph ^ 1);
            if (prof) p_wait += clock64() - tw0;
            if (rank == 0) {
              // expected bytes of both CTAs: A rows + B halves of every run
              const uint32_t nr = (en.x >> 16) & 7u;
              uint32_t units = 0;   // 16-column B units per CTA
              for (uint32_t r = 0; r < nr; ++r) units += ((run_word(en, static_cast<int>(r)) >> 3) & 7u) + 1u;
              const uint32_t kd = wide ? 64u : 32u;
              en.x |= (eb + q == cur.e0 ? kFirst : 0u) | (eb + q + 1 == cur.e1 ? kLast : 0u);
              srun[s] = en;
              mbar_arrive_expect_tx(&full[s], 2u * (128u * kd * 2u + units * kd * 32u));
            }
            tma_load_2d_pair(smem + s * kStageBytes, wide ? &mp.a2 : &mp.a1, full0 + s * 8, k0, arow);
            if (++s == kStages) {
              s = 0;
              ph ^= 1;
            }
          }
        }
        __syncwarp();
      }
    }
    if (prof && lane == 0) {
      prof[blockIdx.x * 16 + 1] = p_wait;
      prof[blockIdx.x * 16 + 7] = clock64() - p_t0;
    }
  } else if (warp == 3) {
    // -------------------------------------------------------------------- producer B
    if (lane == 0)
      for (int d = 0; d < 2; ++d)
        for (int q = 0; q < 3; ++q) {
          tma_prefetch_desc(&mp.b64[d][q]);
          tma_prefetch_desc(&mp.b32[d][q]);
        }
    int s = 0;
    uint32_t ph = 0;
    int tq_s = 0;
    uint32_t tq_ph = 0;
    for (;;) {
      const TileInfo cur = tq_take(tq_s, tq_ph);
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
            const int wide = static_cast<int>((en.x >> 19) & 1u);
            const int32_t k0 = static_cast<int32_t>(en.x & 0xFFFFu) * 32;
            const uint32_t nr = (en.x >> 16) & 7u;
            const uint32_t unit_bytes = (wide ? 64u : 32u) * 32u;   // one 16-column unit, kd rows
            uint8_t* bdst = smem + s * kStageBytes + kASlot;
            const uint32_t bar = full0 + s * 8;
            mbar_wait(&empty[s], ph ^ 1);
            uint32_t off = 0;
            for (uint32_t r = 0; r < nr; ++r) {
              const uint32_t w = run_word(en, static_cast<int>(r));
              const int j0 = static_cast<int>(w & 7u), len = static_cast<int>((w >> 3) & 7u) + 1;
              if ((len & 1) == 0) {
                // this CTA's half: 32-column boxes [j0 + rank*len/2, +len/2) of the tile's columns
                int c = J * 8 + j0 + static_cast<int>(rank) * (len >> 1);
                int nb = len >> 1;
                uint8_t* d = bdst + off;
                if (nb & 4) { tma_load_3d_pair(d, &mp.b64[wide][2], bar, 0, k0, c); d += 4 * 2 * unit_bytes; c += 4; }
                if (nb & 2) { tma_load_3d_pair(d, &mp.b64[wide][1], bar, 0, k0, c); d += 2 * 2 * unit_bytes; c += 2; }
                if (nb & 1) { tma_load_3d_pair(d, &mp.b64[wide][0], bar, 0, k0, c); }
              } else {
                // 16-column units [2*j0 + rank*len, +len)
                int c = (J * 8 + j0) * 2 + static_cast<int>(rank) * len;
                uint8_t* d = bdst + off;
                if (len & 4) { tma_load_3d_pair(d, &mp.b32[wide][2], bar, 0, k0, c); d += 4 * unit_bytes; c += 4; }
                if (len & 2) { tma_load_3d_pair(d, &mp.b32[wide][1], bar, 0, k0, c); d += 2 * unit_bytes; c += 2; }
                if (len & 1) { tma_load_3d_pair(d, &mp.b32[wide][0], bar, 0, k0, c); }
              }
              off += static_cast<uint32_t>(len) * unit_bytes;
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
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer (rank 0)
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc_base = idesc_f16(kFmt, 256, 0, 0, 1);
      constexpr uint32_t idesc_full = idesc_base | (32u << 17);   // N = 256
      const uint32_t base_addr = smem_u32(smem);
      const uint32_t srun_addr = smem_u32(srun);
      const uint64_t zdesc = smem_desc(smem_u32(sZero), 0, 0, kLayoutSW64);   // all strides 0: the zero atom
      const unsigned long long tk0 = clock64();
      unsigned long long m_te = 0, m_fu = 0;
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
          const uint32_t fl = rs.x;
          if (fl & kEnd) {
            fin = true;
            break;
          }
          if (fl & kFirst) {
            buf = static_cast<int>(tile_it & 1);
            const unsigned long long tw0 = prof ? clock64() : 0;
            mbar_wait(&tempty[buf], static_cast<uint32_t>((tile_it >> 1) & 1));
            if (prof) m_te += clock64() - tw0;
            tc_fence_after();
            dcol = tbase + static_cast<uint32_t>(buf) * 256u;
            umma_f16_pair(dcol, zdesc, zdesc, idesc_full, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u);   // D = 0
          }
          if (!(fl & kNoStep)) {
            const uint32_t a_addr = base_addr + st * kStageBytes, b_addr = a_addr + kASlot;
            const bool wide = ((fl >> 19) & 1u) != 0u;
            const uint32_t kd = wide ? 64u : 32u;
            // A: K-major, SW64 rows of 32 (SBO 512) or SW128 rows of 64 (SBO 1024); +32 B per K=16
            const uint64_t ad = wide ? smem_desc(a_addr, 16, 1024, kLayoutSW128) : smem_desc(a_addr, 16, 512, kLayoutSW64);
            const int nk = wide ? 4 : 2;
            const uint32_t nr = (fl >> 16) & 7u;
            if (nr == 1u && (rs.y & 0xFFFFu) == kFullRun) {
              // B: MN-major SW64 32-column boxes (LBO = box bytes, SBO 512); +1024 B per K=16
              const uint64_t bd = smem_desc(b_addr, kd * 64u, 512, kLayoutSW64);
              for (int kk = 0; kk < nk; ++kk)
                umma_f16_pair(dcol, ad + 2 * kk, bd + 64 * kk, idesc_full, 1u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u);
            } else {
              uint32_t off = 0;
              for (uint32_t r = 0; r < nr; ++r) {
                const uint32_t w = run_word(rs, static_cast<int>(r));
                const uint32_t j0 = w & 7u, len = ((w >> 3) & 7u) + 1u, pat = (w >> 6) & 0xFFu;
                const uint32_t idesc = idesc_base | ((4u * len) << 17);   // N = 32*len
                uint32_t m[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) m[q] = ((pat >> q) & 1u) - 1u;   // 0 keep, ~0 disable
                // even runs: SW64 32-column boxes; odd runs: SW32 16-column units
                const uint64_t bd = (len & 1u) ? smem_desc(b_addr + off, kd * 32u, 256, kLayoutSW32)
                                               : smem_desc(b_addr + off, kd * 64u, 512, kLayoutSW64);
                const uint32_t bstep = (len & 1u) ? 32u : 64u;   // K=16 rows: 512 or 1024 bytes
                const uint32_t d = dcol + j0 * 32u;
                for (int kk = 0; kk < nk; ++kk)
                  umma_f16_pair(d, ad + 2 * kk, bd + bstep * kk, idesc, 1u, m[0], m[1], m[2], m[3], m[4], m[5], m[6],
                                m[7]);
                off += len * kd * 32u;
              }
            }
          }
          umma_commit_pair(&empty[st]);
          if (fl & kLast) {
            umma_commit_pair(&tfull[buf]);
            ++tile_it;
          }
        }
        ph ^= 1;
      }
      if (prof) {
        prof[blockIdx.x * 16 + 2] = m_te;
        prof[blockIdx.x * 16 + 3] = m_fu;
        prof[blockIdx.x * 16 + 6] = clock64() - tk0;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // --------------------------------------------------------------- epilogue (both CTAs)
    const int q = warp & 3;            // TMEM lane quadrant (warp % 4)
    const int half = (warp - 4) >> 2;  // columns [128*half, 128*half + 128)
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      mbar_arrive_cluster(tempty0);
      mbar_arrive_cluster(tempty0 + 8);
    }
    const int t0 = lane & 3, t1 = lane >> 2;
    unsigned long long e_w = 0, e_d = 0;
    int tq_s = 0;
    uint32_t tq_ph = 0;
    for (int64_t it = 0;; ++it) {
      const TileInfo cur = tq_take(tq_s, tq_ph);
      if (++tq_s == kTQ) {
        tq_s = 0;
        tq_ph ^= 1;
      }
      if (cur.t < 0) break;
      const int64_t I = cur.t / GN, J = cur.t % GN;
      const int buf = static_cast<int>(it & 1);
      const unsigned long long te0 = prof ? clock64() : 0;
      mbar_wait(&tfull[buf], static_cast<uint32_t>((it >> 1) & 1));
      const unsigned long long te1 = prof ? clock64() : 0;
      e_w += te1 - te0;
      tc_fence_after();
#pragma unroll 1
      for (int hh = 0; hh < 4; ++hh) {
        const int lh = hh & 1;                         // lanes [16*lh, 16*lh + 16) of the quadrant
        const int c0 = half * 128 + (hh >> 1) * 64;    // 64-column block
        uint32_t v[32];
        tmem_ld_16x256b_x8(tbase + ((static_cast<uint32_t>(q * 32 + 16 * lh)) << 16) + buf * 256 + c0, v);
        tmem_wait_ld();
        const int64_t ra = I * 256 + rank * 128 + q * 32 + 16 * lh + t1, rb = ra + 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int64_t col = J * 256 + c0 + 8 * i + 2 * t0;
          if (col + 1 < N) {
            if (ra < M) __stcs(reinterpret_cast<float2*>(C + ra * ldc + col),
                               make_float2(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1])));
            if (rb < M) __stcs(reinterpret_cast<float2*>(C + rb * ldc + col),
                               make_float2(__uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3])));
          } else if (col < N) {
            if (ra < M) C[ra * ldc + col] = __uint_as_float(v[4 * i]);
            if (rb < M) C[rb * ldc + col] = __uint_as_float(v[4 * i + 2]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty0 + buf * 8);
      if (prof) e_d += clock64() - te1;
    }
    if (prof && warp == 4 && lane == 0) {
      prof[blockIdx.x * 16 + 4] = e_w;
      prof[blockIdx.x * 16 + 5] = e_d;
    }
  }
  tc_fence_before();
  cluster_sync();   // the peer's TMEM / barriers stay live until both CTAs are done
  if (warp == 2) tmem_dealloc_pair<kTmemCols>(tbase);
}

template <uint32_t kFmt>
spamm_status launch_fmt(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                        cudaStream_t s, CUtensorMapDataType dt) {
  if (p.N % 32 != 0) return fail(SPAMM_E_UNSUPPORTED, "pair tensor path needs N % 32 == 0");
  PairMaps mp;
  std::memset(&mp, 0, sizeof(mp));
  SPAMM_TRY(encode_tmap_2d(&mp.a1, dt, 2, A, p.K, p.M, lda, 32, 128, CU_TENSOR_MAP_SWIZZLE_64B));
  SPAMM_TRY(encode_tmap_2d(&mp.a2, dt, 2, A, p.K, p.M, lda, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B));
  // B as stacked column boxes: dims {w, K, N/w} with strides {ldb, w} elements (a
  // non-monotonic stride; verified by scripts/probe_tma3d.cu)
  const uint32_t nbs[3] = {1, 2, 4};
  for (int d = 0; d < 2; ++d)
    for (int q = 0; q < 3; ++q) {
      const uint32_t kd = d ? 64 : 32;
      SPAMM_TRY(encode_tmap_3d(&mp.b64[d][q], dt, B, 32, p.K, p.N / 32, static_cast<uint64_t>(ldb) * 2, 64, 32, kd,
                               nbs[q], CU_TENSOR_MAP_SWIZZLE_64B));
      SPAMM_TRY(encode_tmap_3d(&mp.b32[d][q], dt, B, 16, p.K, p.N / 16, static_cast<uint64_t>(ldb) * 2, 32, 16, kd,
                               nbs[q], CU_TENSOR_MAP_SWIZZLE_32B));
    }
  auto kern = spamm_mul_pair_kernel<kFmt>;
  static bool attr_set = false;
  if (!attr_set) {
    SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes)));
    attr_set = true;
  }
  const int64_t n_tiles = (p.row_end_macro - p.row_begin_macro) * p.GN;
  if (n_tiles <= 0) return SPAMM_OK;
  const int64_t pairs = std::max<int64_t>(1, std::min<int64_t>(n_tiles, p.num_sms / 2));
  const int grid = static_cast<int>(2 * pairs);
  constexpr int kProfMax = 512;
  static unsigned long long* prof = nullptr;
  if (getenv("SPAMM_DEBUG_UMMA_PROF") && !prof) cudaMalloc(&prof, kProfMax * 16 * 8);
  if (prof && grid > kProfMax) return fail(SPAMM_E_UNSUPPORTED, "profiling supports at most 512 CTAs");
  if (prof) cudaMemsetAsync(prof, 0, kProfMax * 16 * 8, s);
  SPAMM_CUDA_TRY(cudaMemsetAsync(p.sched, 0, sizeof(unsigned int), s));
  // tiles of macro rows [row_begin_macro, row_end_macro): order[] holds tile ids of that range
  kern<<<grid, kThreads, kSmemBytes, s>>>(mp, p.Uw, p.macro_run, p.order, n_tiles, p.GN, p.BK, C, ldc, p.M, p.N,
                                          p.sched, prof);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  if (prof) {
    static unsigned long long h[kProfMax * 16];
    cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double acc[16] = {0};
    double mx = 0;
    for (int c = 0; c < grid; c += 2) {   // rank 0 CTAs
      for (int k = 0; k < 16; ++k) acc[k] += static_cast<double>(h[c * 16 + k]) / (grid / 2);
      mx = std::max(mx, static_cast<double>(h[c * 16 + 6]));
    }
    fprintf(stderr,
            "[pair prof] cycles per rank-0 CTA: MMA thread %.0f (max %.0f) tmem-empty wait %.0f stage-full wait %.0f | "
            "producer A %.0f stage-empty wait %.0f | epilogue tmem-full wait %.0f drain %.0f\n",
            acc[6], mx, acc[2], acc[3], acc[7], acc[1], acc[4], acc[5]);
  }
  return SPAMM_OK;
}

}  // namespace

spamm_status launch_multiply_pair(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C,
                                  int64_t ldc, cudaStream_t s) {
  if (p.out_norms || p.out_low)
    return fail(SPAMM_E_UNSUPPORTED, "chained outputs are not implemented for the CTA-pair variant");
  if (p.alpha != 1.0 || p.beta != 0.0)
    return fail(SPAMM_E_UNSUPPORTED, "the CTA-pair variant (SPAMM_UMMA_VARIANT=3) implements alpha = 1, beta = 0 only");
  if (p.prec == SPAMM_BF16) return launch_fmt<1>(p, A, lda, B, ldb, C, ldc, s, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
  return launch_fmt<0>(p, A, lda, B, ldb, C, ldc, s, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
}

}  // namespace spamm
