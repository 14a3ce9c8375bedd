// multiply_umma.cu -- stage 3, tensor-core path (tensor-core multiplication kernel,
// Sec. 3.3, Alg. 3), BF16/FP16 inputs, FP32 accumulation.
//
// C[i,j] = sum_{kept k, ascending} A[i,k] * B[k,j]; the paper's FP32
// accumulator fragment becomes an FP32 accumulator in TMEM.
//
// B200 design (tcgen05, not the paper's wmma):
//   * persistent CTAs (one per SM) over an LPT-ordered list of 128x256 macro-tiles
//     (4 x 8 C tiles of 32x32), taken in snake order;
//   * warp 0: TMA producer.  Per kept k of the macro-tile's union list it loads
//     A[128 x 32] (K-major, SWIZZLE_64B) and the contiguous range of needed
//     B[32 x 32] boxes (MN-major, SWIZZLE_64B) with one 3-D TMA per power-of-two
//     piece.  Two k-steps share one ring stage (one mbarrier handshake per two
//     k-steps: the per-handshake cost, not the tensor pipe, bounded the 1-k design);
//   * warp 1 lane 0: issues tcgen05.mma kind::f16 M=128, K=16 (x2 per k-tile).  The
//     skip-map emit kernel pre-decoded each k-step's 4 x 8 keep bits into runs of
//     adjacent C-tile columns with the same 4-bit row pattern; each run is ONE MMA
//     with N = 32*run and the disable-output-lane mask switching off the 32-lane
//     groups (C-tile rows) whose pair is skipped -- exact leaf-level skip semantics
//     (Alg. 2 l.3-8) on a 128-row MMA;
//   * warps 4-7: epilogue -- TMEM -> registers -> swizzled smem -> TMA bulk store of
//     C (FP32), zeroing the accumulator for its next use; two TMEM accumulators
//     (2 x 256 columns) overlap the epilogue of one macro-tile with the next's MMAs.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>

#include "internal.h"
#include "sm100.cuh"

namespace spamm {
namespace {

using namespace sm100;

constexpr int kStages = 3;                      // ring stages, each holding kPer k-steps
constexpr int kPer = 1;
constexpr int kABytes = 128 * 32 * 2;           // 8 KB per k-step
constexpr int kBBoxBytes = 32 * 32 * 2;         // 2 KB per 32 x 32 box
constexpr int kBBytes = 8 * kBBoxBytes;         // 16 KB per k-step
constexpr int kThreads = 256;
constexpr int kCStageBytes = 32 * 32 * 4;       // one 32x32 FP32 C box (SWIZZLE_128B); 2 per epilogue warp
constexpr size_t kRingBytes = static_cast<size_t>(kStages) * kPer * (kABytes + kBBytes);
constexpr size_t kSmemBytes = 1024 + kRingBytes + 8 * kCStageBytes + 1280;   // 2 CTAs per SM
constexpr uint32_t kTmemCols = 256;             // one 128x256 FP32 accumulator per CTA (2 CTAs per SM)

// run word of a k-step whose 4 x 8 keep bits are all set: j0 = 0, len = 8, pattern 1111
constexpr uint32_t kFullRun = 0u | (7u << 3) | (15u << 6);
constexpr int kTQ = 4;   // tile ring depth (dynamic LPT scheduling)

__device__ __forceinline__ int64_t snake(int64_t r, int G, int b) { return r * G + ((r & 1) ? (G - 1 - b) : b); }

// number of ring stages the producer uses for a tile with E entries (batches of 32, kPer per stage)
__device__ __forceinline__ int64_t stages_for(int64_t E) {
  return (E / 32) * (32 / kPer) + ((E % 32) + kPer - 1) / kPer;
}

struct TileInfo {
  int64_t t, e0, e1;
};
__device__ __forceinline__ TileInfo tile_info(const int32_t* order, const int64_t* mstart, const int64_t* mcount,
                                              int64_t idx, int64_t n_tiles) {
  TileInfo ti{-1, 0, 0};
  if (idx < n_tiles) {
    ti.t = order[idx];
    ti.e0 = mstart[ti.t];
    ti.e1 = ti.e0 + mcount[ti.t];
  }
  return ti;
}

template <uint32_t kFmt>
__global__ void __launch_bounds__(kThreads, 2)
    spamm_mul_umma_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                          const __grid_constant__ CUtensorMap tB8, const __grid_constant__ CUtensorMap tB4,
                          const __grid_constant__ CUtensorMap tB2, const __grid_constant__ CUtensorMap tB1,
                          const __grid_constant__ CUtensorMap tC, int use3d, int dbg_mode,
                          const int64_t* __restrict__ mstart, const int64_t* __restrict__ mcount, const uint4* __restrict__ ment,
                          const int32_t* __restrict__ order, int64_t n_tiles, int64_t GN,
                          unsigned int* __restrict__ sched, unsigned long long* __restrict__ prof) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                           // [stage][slot] 8 KB
  uint8_t* sB = smem + kStages * kPer * kABytes;                // [stage][slot] 16 KB
  uint8_t* sC = smem + kRingBytes;                              // [4 warps][2 bufs] 4 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(sC + 8 * kCStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint4* srun = reinterpret_cast<uint4*>(tempty + 2);           // [stage][slot]: pre-decoded runs
  uint32_t* scount = reinterpret_cast<uint32_t*>(srun + kStages * kPer);   // k-steps in the stage
  uint4* sent = reinterpret_cast<uint4*>((reinterpret_cast<uintptr_t>(scount + kStages) + 15) & ~uintptr_t(15));
  TileInfo* tq = reinterpret_cast<TileInfo*>(sent + 32);       // [kTQ] tiles claimed by the producer
  uint64_t* tq_full = reinterpret_cast<uint64_t*>(tq + kTQ);
  uint64_t* tq_empty = tq_full + kTQ;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq_empty + kTQ);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tempty[0], 4);
    for (int q = 0; q < kTQ; ++q) {
      mbar_init(&tq_full[q], 1);
      mbar_init(&tq_empty[q], 5);   // MMA thread + 4 epilogue warps
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tA);
      tma_prefetch_desc(&tC);
      if (use3d) {
        tma_prefetch_desc(&tB8);
        tma_prefetch_desc(&tB4);
        tma_prefetch_desc(&tB2);
        tma_prefetch_desc(&tB1);
      } else {
        tma_prefetch_desc(&tB);
      }
    }
    int s = 0;
    uint32_t ph = 0;
    unsigned long long p_load = 0, p_wait = 0;
    const unsigned long long p_t0 = clock64();
    // Dynamic LPT scheduling: tiles are claimed in global order (descending work) from an
    // atomic counter, one tile ahead, and published to the MMA / epilogue roles via tq[].
    int tq_s = 0;
    uint32_t tq_ph = 0;
    TileInfo nxt;
    {
      unsigned int idx = 0;
      if (lane == 0) idx = atomicAdd(sched, 1u);
      idx = __shfl_sync(0xffffffffu, idx, 0);
      nxt = tile_info(order, mstart, mcount, idx, n_tiles);
    }
    for (;;) {
      const TileInfo cur = nxt;
      if (cur.t >= 0) {
        unsigned int idx = 0;
        if (lane == 0) idx = atomicAdd(sched, 1u);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        nxt = tile_info(order, mstart, mcount, idx, n_tiles);   // consumed next iteration
      }
      if (lane == 0) {
        mbar_wait(&tq_empty[tq_s], tq_ph ^ 1);
        tq[tq_s] = cur;
        mbar_arrive(&tq_full[tq_s]);
      }
      if (++tq_s == kTQ) {
        tq_s = 0;
        tq_ph ^= 1;
      }
      if (cur.t < 0) break;
      const int32_t I = static_cast<int32_t>(cur.t / GN), J = static_cast<int32_t>(cur.t % GN);
      for (int64_t eb = cur.e0; eb < cur.e1; eb += 32) {
        const int cnt = static_cast<int>(cur.e1 - eb < 32 ? cur.e1 - eb : 32);
        unsigned long long tb0 = prof ? clock64() : 0;
        if (lane < cnt) sent[lane] = ment[eb + lane];
        __syncwarp();
        if (prof) p_load += clock64() - tb0;
        if (lane == 0) {
          for (int q0 = 0; q0 < cnt; q0 += kPer) {
            const int nq = cnt - q0 < kPer ? cnt - q0 : kPer;
            unsigned long long tw0 = prof ? clock64() : 0;
            mbar_wait(&empty[s], ph ^ 1);
            if (prof) p_wait += clock64() - tw0;
            if (kPer == 1 && use3d && dbg_mode == 0) {
              // lean path: one k-step per stage
              const uint4 en = sent[q0];
              srun[s] = en;
              const uint32_t cols = en.x >> 24;
              const int32_t k0 = static_cast<int32_t>(en.x & 0xFFFFu) * 32;
              uint8_t* adst = sA + s * kABytes;
              uint8_t* bdst = sB + s * kBBytes;
              const int jb = J * 8;
              if (cols == 0xFFu) {
                mbar_arrive_expect_tx(&full[s], kABytes + kBBytes);
                tma_load_2d(adst, &tA, &full[s], k0, I * 128);
                tma_load_3d(bdst, &tB8, &full[s], 0, k0, jb);
              } else {
                const int c0 = __ffs(cols) - 1, len = (32 - __clz(cols)) - c0;
                int off = c0;
                mbar_arrive_expect_tx(&full[s], kABytes + kBBoxBytes * len);
                tma_load_2d(adst, &tA, &full[s], k0, I * 128);
                if (len & 4) { tma_load_3d(bdst + off * kBBoxBytes, &tB4, &full[s], 0, k0, jb + off); off += 4; }
                if (len & 2) { tma_load_3d(bdst + off * kBBoxBytes, &tB2, &full[s], 0, k0, jb + off); off += 2; }
                if (len & 1) { tma_load_3d(bdst + off * kBBoxBytes, &tB1, &full[s], 0, k0, jb + off); }
              }
              if (++s == kStages) {
                s = 0;
                ph ^= 1;
              }
              continue;
            }
            uint32_t bytes = 0;
            for (int q = 0; q < nq; ++q) {
              const uint32_t cols = sent[q0 + q].x >> 24;
              bytes += kABytes + kBBoxBytes * (use3d ? (32 - __clz(cols)) - (__ffs(cols) - 1) : __popc(cols));
            }
            scount[s] = static_cast<uint32_t>(nq);
            for (int q = 0; q < nq; ++q) srun[s * kPer + q] = sent[q0 + q];
            if (dbg_mode == 1 || dbg_mode == 3 || dbg_mode >= 5) {   // debug: no operand traffic
              mbar_arrive(&full[s]);
            } else {
              mbar_arrive_expect_tx(&full[s], bytes);
              for (int q = 0; q < nq; ++q) {
                const uint4 en = sent[q0 + q];
                const uint32_t cols = en.x >> 24;
                const int32_t k0 = static_cast<int32_t>(en.x & 0xFFFFu) * 32;
                uint8_t* adst = sA + (s * kPer + q) * kABytes;
                uint8_t* bdst = sB + (s * kPer + q) * kBBytes;
                tma_load_2d(adst, &tA, &full[s], k0, I * 128);
                if (use3d) {
                  const int c0 = __ffs(cols) - 1, c1 = 31 - __clz(cols);
                  int off = c0;
                  const int len = c1 - c0 + 1;
                  const int jb = J * 8;
                  if (len == 8) {
                    tma_load_3d(bdst, &tB8, &full[s], 0, k0, jb);
                  } else {
                    if (len & 4) { tma_load_3d(bdst + off * kBBoxBytes, &tB4, &full[s], 0, k0, jb + off); off += 4; }
                    if (len & 2) { tma_load_3d(bdst + off * kBBoxBytes, &tB2, &full[s], 0, k0, jb + off); off += 2; }
                    if (len & 1) { tma_load_3d(bdst + off * kBBoxBytes, &tB1, &full[s], 0, k0, jb + off); }
                  }
                } else {
#pragma unroll
                  for (int lj = 0; lj < 8; ++lj)
                    if ((cols >> lj) & 1u) tma_load_2d(bdst + lj * kBBoxBytes, &tB, &full[s], J * 256 + lj * 32, k0);
                }
              }
            }
            if (++s == kStages) {
              s = 0;
              ph ^= 1;
            }
          }
        }
        __syncwarp();   // (s, ph) are only used by lane 0
      }
    }
    if (prof && lane == 0) {
      prof[blockIdx.x * 16 + 0] = p_load;
      prof[blockIdx.x * 16 + 1] = p_wait;
      prof[blockIdx.x * 16 + 7] = clock64() - p_t0;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    const unsigned long long tk0 = clock64();
    if (lane == 0) {
      constexpr uint32_t idesc_base = idesc_f16(kFmt, 128, 0, 0, 1);
      const uint32_t a_addr0 = smem_u32(sA), b_addr0 = smem_u32(sB);
      const uint32_t srun_addr = smem_u32(srun), scount_addr = smem_u32(scount);
      int s = 0;
      uint32_t ph = 0;
      int64_t it = 0;
      unsigned long long m_te = 0, m_fu = 0;
      int tq_s = 0;
      uint32_t tq_ph = 0;
      for (;; ++it) {
        mbar_wait(&tq_full[tq_s], tq_ph);
        const TileInfo cur = tq[tq_s];
        mbar_arrive(&tq_empty[tq_s]);
        if (++tq_s == kTQ) {
          tq_s = 0;
          tq_ph ^= 1;
        }
        if (cur.t < 0) break;
        const int buf = 0;
        unsigned long long tw0 = prof ? clock64() : 0;
        mbar_wait(&tempty[0], static_cast<uint32_t>(it & 1));
        if (prof) m_te += clock64() - tw0;
        tc_fence_after();
        const uint32_t dcol = tbase;
        const int64_t nst = stages_for(cur.e1 - cur.e0);
        for (int64_t st = 0; st < nst; ++st) {
          unsigned long long tf0 = prof ? clock64() : 0;
          mbar_wait(&full[s], ph);
          if (prof) m_fu += clock64() - tf0;
          tc_fence_after();
          uint32_t nq;
          if (kPer == 1) {
            uint4 rs;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(rs.x), "=r"(rs.y), "=r"(rs.z), "=r"(rs.w)
                         : "r"(srun_addr + s * 16));
            if (((rs.x >> 16) & 15u) == 1u && rs.y == kFullRun && dbg_mode == 0) {
              // full 4 x 8 keep mask: two N=256 MMAs, no lane mask
              constexpr uint32_t idesc_full = idesc_base | (8u << 19);
              const uint64_t ad0 = smem_desc(a_addr0 + s * kABytes, 16, 512, kLayoutSW64);
              const uint64_t bd0 = smem_desc(b_addr0 + s * kBBytes, kBBoxBytes, 512, kLayoutSW64);
              umma_f16(dcol, ad0, bd0, idesc_full, 1u, 0u, 0u, 0u, 0u);
              umma_f16(dcol, ad0 + (32 >> 4), bd0 + (1024 >> 4), idesc_full, 1u, 0u, 0u, 0u, 0u);
              nq = 0;
            } else {
              nq = 1;
            }
          } else {
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(nq) : "r"(scount_addr + s * 4));
          }
          for (uint32_t q = 0; q < nq; ++q) {
            uint4 rs;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(rs.x), "=r"(rs.y), "=r"(rs.z), "=r"(rs.w)
                         : "r"(srun_addr + (s * kPer + q) * 16));
            const uint32_t nr = (dbg_mode == 2 || dbg_mode == 3 || dbg_mode >= 5) ? 0u : ((rs.x >> 16) & 15u);
            const uint64_t ad0 = smem_desc(a_addr0 + (s * kPer + q) * kABytes, 16, 512, kLayoutSW64);
            const uint64_t bd0 = smem_desc(b_addr0 + (s * kPer + q) * kBBytes, kBBoxBytes, 512, kLayoutSW64);
            uint32_t cw = rs.y;
            for (uint32_t rr = 0; rr < nr; ++rr) {
              if (rr == 3) cw = rs.z;
              if (rr == 6) cw = rs.w;
              const uint32_t w = cw & 0x3FFu;
              cw >>= 10;
              const uint32_t j0 = w & 7u, len = ((w >> 3) & 7u) + 1u, pat = w >> 6;
              const uint32_t idesc = idesc_base | (len << 19);          // N = 32*len -> N>>3 = 4*len at bit 17
              const uint32_t m0 = (pat & 1u) - 1u, m1 = ((pat >> 1) & 1u) - 1u;   // 0 keep, ~0 disable
              const uint32_t m2 = ((pat >> 2) & 1u) - 1u, m3 = ((pat >> 3) & 1u) - 1u;
              const uint64_t bd = bd0 + static_cast<uint64_t>(j0 * (kBBoxBytes >> 4));
              const uint32_t d = dcol + j0 * 32u;
              umma_f16(d, ad0, bd, idesc, 1u, m0, m1, m2, m3);
              umma_f16(d, ad0 + (32 >> 4), bd + (1024 >> 4), idesc, 1u, m0, m1, m2, m3);
            }
          }
          umma_commit(&empty[s]);
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
        umma_commit(&tfull[0]);
      }
      if (prof) {
        prof[blockIdx.x * 16 + 2] = m_te;
        prof[blockIdx.x * 16 + 3] = m_fu;
        prof[blockIdx.x * 16 + 6] = clock64() - tk0;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // --------------------------------------------------------------- epilogue
    const int q = warp & 3;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    for (int c = 0; c < 8; ++c) tmem_st_32x32b_x32_zero(tbase + lane_off + c * 32);
    tmem_wait_st();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&tempty[0]);
    int64_t it = 0;
    unsigned long long e_w = 0, e_d = 0;
    int tq_s = 0;
    uint32_t tq_ph = 0;
    for (;; ++it) {
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
      const int buf = 0;
      unsigned long long te0 = prof ? clock64() : 0;
      mbar_wait(&tfull[0], static_cast<uint32_t>(it & 1));
      unsigned long long te1 = prof ? clock64() : 0;
      e_w += te1 - te0;
      tc_fence_after();
      // TMEM -> registers -> swizzled smem box -> TMA bulk store (coalesced, clipped at M, N)
#pragma unroll 1
      for (int c = 0; c < (dbg_mode == 6 ? 0 : 8); ++c) {   // debug 6: empty epilogue
        const uint32_t taddr = tbase + lane_off + buf * 256 + c * 32;
        uint32_t v[32];
        tmem_ld_32x32b_x32(taddr, v);
        tmem_wait_ld();
        if (dbg_mode == 7) continue;                          // debug 7: TMEM loads only
        tmem_st_32x32b_x32_zero(taddr);
        if (dbg_mode == 8) continue;                          // debug 8: TMEM load + zero store
        uint8_t* box = sC + (q * 2 + (c & 1)) * kCStageBytes;
        if (c >= 2) {
          if (lane == 0) bulk_wait_group_read<1>();   // the store issued from this buffer two chunks ago
          __syncwarp();
        }
        // row = lane (128 B); 16-byte chunk j stored at j ^ (row % 8)  (SWIZZLE_128B)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int pj = j ^ (lane & 7);
          *reinterpret_cast<uint4*>(box + lane * 128 + pj * 16) =
              make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && dbg_mode != 4 && dbg_mode < 5) {   // debug 4/5: no C store
          tma_store_2d(&tC, box, static_cast<int32_t>(J * 256 + c * 32), static_cast<int32_t>(I * 128 + q * 32));
          bulk_commit_group();
        }
      }
      if (lane == 0) bulk_wait_group_read<0>();
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[0]);
      if (prof) e_d += clock64() - te1;
    }
    if (prof && q == 0 && lane == 0) {
      prof[blockIdx.x * 16 + 4] = e_w;
      prof[blockIdx.x * 16 + 5] = e_d;
    }
    if (lane == 0) bulk_wait_group<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<kTmemCols>(tbase);
}

template <uint32_t kFmt>
spamm_status launch_fmt(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                        cudaStream_t s, CUtensorMapDataType dt) {
  CUtensorMap tA, tB, tB8, tB4, tB2, tB1, tC;
  SPAMM_TRY(encode_tmap_2d(&tC, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, C, p.N, p.M, ldc, 32, 32,
                           CU_TENSOR_MAP_SWIZZLE_128B));
  SPAMM_TRY(encode_tmap_2d(&tA, dt, 2, A, p.K, p.M, lda, 32, 128, CU_TENSOR_MAP_SWIZZLE_64B));
  SPAMM_TRY(encode_tmap_2d(&tB, dt, 2, B, p.N, p.K, ldb, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B));
  // B as stacked [32 k][32 n] boxes: dims {32 n, K, N/32} with strides {ldb, 32} elements.
  // Only when N % 32 == 0 (the inner 32 columns of the last box must exist).
  const int use3d = (p.N % 32) == 0;
  if (use3d) {
    const uint32_t nbs[4] = {8, 4, 2, 1};
    CUtensorMap* maps[4] = {&tB8, &tB4, &tB2, &tB1};
    for (int q = 0; q < 4; ++q)
      SPAMM_TRY(encode_tmap_3d(maps[q], dt, B, 32, p.K, p.N / 32, static_cast<uint64_t>(ldb) * 2, 64, 32, 32,
                               nbs[q], CU_TENSOR_MAP_SWIZZLE_64B));
  } else {
    tB8 = tB4 = tB2 = tB1 = tB;
  }
  static bool attr_set = false;
  if (!attr_set) {
    SPAMM_CUDA_TRY(cudaFuncSetAttribute(spamm_mul_umma_kernel<kFmt>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kSmemBytes)));
    attr_set = true;
  }
  const int64_t n_tiles = (p.row_end_macro - p.row_begin_macro) * p.GN;
  if (n_tiles <= 0) return SPAMM_OK;
  const int64_t slots = 2 * static_cast<int64_t>(p.num_sms);   // 2 CTAs per SM
  const int grid = static_cast<int>(n_tiles < slots ? n_tiles : slots);
  static const int dbg_mode = getenv("SPAMM_DEBUG_UMMA_MODE") ? atoi(getenv("SPAMM_DEBUG_UMMA_MODE")) : 0;
  static unsigned long long* prof = nullptr;
  if (getenv("SPAMM_DEBUG_UMMA_PROF") && !prof) {
    cudaMalloc(&prof, 296 * 16 * 8);
  }
  if (prof) cudaMemsetAsync(prof, 0, 296 * 16 * 8, s);
  SPAMM_CUDA_TRY(cudaMemsetAsync(p.sched, 0, sizeof(unsigned int), s));
  spamm_mul_umma_kernel<kFmt><<<grid, kThreads, kSmemBytes, s>>>(tA, tB, tB8, tB4, tB2, tB1, tC, use3d, dbg_mode,
                                                                 p.mstart, p.U, p.macro_run, p.order, n_tiles, p.GN,
                                                                 p.sched, prof);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  if (prof) {
    unsigned long long h[296 * 16];
    cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double acc[16] = {0};
    double mn = 1e30, mx = 0;
    for (int c = 0; c < grid; ++c) {
      for (int k = 0; k < 16; ++k) acc[k] += static_cast<double>(h[c * 16 + k]) / grid;
      mn = std::min(mn, static_cast<double>(h[c * 16 + 6]));
      mx = std::max(mx, static_cast<double>(h[c * 16 + 6]));
    }
    fprintf(stderr, "[umma prof] per-CTA MMA-thread cycles: min %.0f max %.0f mean %.0f\n", mn, mx, acc[6]);
    fprintf(stderr,
            "[umma prof] mean cycles/CTA: total %.0f | producer batch-load %.0f empty-wait %.0f | mma tempty-wait %.0f "
            "full-wait %.0f | epi tfull-wait %.0f drain %.0f\n",
            acc[6], acc[0], acc[1], acc[2], acc[3], acc[4], acc[5]);
  }
  return SPAMM_OK;
}

}  // namespace

spamm_status launch_multiply_umma(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C,
                                  int64_t ldc, cudaStream_t s) {
  if (p.prec == SPAMM_BF16) return launch_fmt<1>(p, A, lda, B, ldb, C, ldc, s, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
  return launch_fmt<0>(p, A, lda, B, ldb, C, ldc, s, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
}

}  // namespace spamm
