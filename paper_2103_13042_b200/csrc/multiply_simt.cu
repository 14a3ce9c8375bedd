// multiply_simt.cu -- stage 3, FP32 CUDA-core path (multiplication kernel, Sec. 3.3,
// Alg. 2 lines 17-28).
//
// C[i,j] = sum_{kept k, ascending} A[i,k] * B[k,j], FP32 FMA.
//
// B200 design.  Persistent CTAs (one per SM) walk an LPT-ordered list of 128x128
// macro-tiles (4x4 C tiles).  For every k in the macro-tile's union list a TMA
// producer warp stages A[128 x 32] (SWIZZLE_128B) and B[32 x 128] in a 6-deep
// shared-memory ring guarded by mbarriers (replacing the paper's two half-block
// double buffer).  Eight compute warps each own a pair of adjacent 32x32
// C tiles; the pair's keep bits for this k are warp-uniform, so a skipped pair costs a warp
// nothing but the barrier.  Each lane computes an 8x8 register micro-tile (4 columns in
// each tile of the pair).  Two-level accumulation: a 32-term register partial per kept k-tile
// is added into a running sum, also in registers, which keeps
// N=65536 within 1e-5.
#include "internal.h"
#include "skipdecide.cuh"
#include "sm100.cuh"

namespace spamm {
namespace {

using namespace sm100;

#ifndef SPAMM_SIMT_QUNROLL
#define SPAMM_SIMT_QUNROLL 2
#endif
constexpr int kQUnroll = SPAMM_SIMT_QUNROLL;   // k-slice loop unroll (experiments: -DSPAMM_SIMT_QUNROLL)
constexpr int kStages = 6;
constexpr int kComputeWarps = 8;   // one C-tile pair (32 x 64) each
// warpgroup 0: the TMA producer (warp 0; its registers handed to the compute warps with setmaxnreg),
// warpgroups 1-2: the 8 compute warps (232 registers each: 128 accumulators of the 8 x 8 micro-tile)
constexpr int kThreads = (4 + kComputeWarps) * 32;
constexpr int kAFloats = 128 * 32;
constexpr int kBFloats = 32 * 128;
constexpr int kStageBytes = (kAFloats + kBFloats) * 4;
constexpr size_t kSmemBytes = 1024 + static_cast<size_t>(kStages) * kStageBytes + 512;

__device__ __forceinline__ int64_t snake(int64_t r, int G, int b) { return r * G + ((r & 1) ? (G - 1 - b) : b); }

__device__ __forceinline__ float comp(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// kFuse (small problems, spamm_run): the producer warp decides each tile's skip list itself
// (skipdecide.cuh fuse_tile_list: the skip kernel's predicate and list format, plus U, L, row work,
// totals and the identity order for the getters) and hands (tile, k-steps) to the compute warps
// through a 2-slot shared-memory queue; the compute warps read the just-written masks coherently.
template <bool kFuse>
__global__ void __launch_bounds__(kThreads, 1)
    spamm_mul_simt_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                          float* __restrict__ C, int64_t ldc, int64_t M, int64_t N,
                          const int64_t* __restrict__ mstart, const int64_t* __restrict__ mcount, const uint2* ment,
                          const int32_t* __restrict__ order, int64_t n_tiles, const int64_t* __restrict__ rng,
                          int64_t GN, const Axpby ab, double* __restrict__ nC, int64_t ldn, int64_t BM, int64_t BN,
                          const XFuse fz) {
  if (rng != nullptr) n_tiles = (rng[1] - rng[0]) * GN;   // multi-GPU range decided on the device
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned base derived from smem_raw by an offset (not an integer round trip), so the compiler
  // keeps the shared address space: LDS/STS instead of generic LD/ST for the operand and sum reads
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  float* sA = reinterpret_cast<float*>(smem);
  float* sB = sA + kStages * kAFloats;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(kStages) * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tl_full = empty + kStages;    // kFuse: 2-slot tile queue (tile, k-step count)
  uint64_t* tl_empty = tl_full + 2;
  int64_t* tl_info = reinterpret_cast<int64_t*>(tl_empty + 2);   // [2][2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kComputeWarps);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&tl_full[q], 1);
      mbar_init(&tl_empty[q], kComputeWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int G = gridDim.x, b = blockIdx.x;

  if (warp < 4) {
    // ------------------------------------------------------ TMA producer (warpgroup 0)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;" ::: "memory");
    if constexpr (kFuse) {
      if (warp == 0) {   // the whole warp decides the lists; lane 0 issues the loads
        if (lane == 0) {
          tma_prefetch_desc(&tA);
          tma_prefetch_desc(&tB);
        }
        int s = 0;
        uint32_t ph = 0;
        for (int64_t r = 0;; ++r) {
          const int64_t t = snake(r, G, b);   // static assignment, identity order
          const int slot = static_cast<int>(r & 1);
          const uint32_t tph = static_cast<uint32_t>((r >> 1) & 1);
          uint2 reg = make_uint2(0u, 0u);
          uint32_t any = 0u;
          const int64_t u = t < n_tiles ? fuse_tile_list(fz, t, GN, lane, &reg, &any) : 0;
          if (lane == 0) {   // publish (tile, k-steps), or the end marker
            mbar_wait(&tl_empty[slot], tph ^ 1);
            tl_info[2 * slot] = t < n_tiles ? t : -1;
            tl_info[2 * slot + 1] = u;
            mbar_arrive(&tl_full[slot]);   // release: the list written above is visible to the CTA
          }
          if (t >= n_tiles) break;
          const int32_t I = static_cast<int32_t>(t / GN), J = static_cast<int32_t>(t % GN);
          for (int64_t q = 0; q < u; ++q) {
            uint32_t kx;
            if (fz.BK <= 32) kx = __shfl_sync(0xffffffffu, reg.x, static_cast<int>(__fns(any, 0u, static_cast<int>(q) + 1)));
            else kx = __ldcg(ment + t * fz.BK + q).x;
            if (lane == 0) {
              mbar_wait(&empty[s], ph ^ 1);
              mbar_arrive_expect_tx(&full[s], kStageBytes);
              tma_load_2d(sA + s * kAFloats, &tA, &full[s], static_cast<int32_t>(kx) * 32, I * 128);
              tma_load_2d(sB + s * kBFloats, &tB, &full[s], J * 128, static_cast<int32_t>(kx) * 32);
            }
            if (++s == kStages) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
      return;
    }
    if (warp == 0 && lane == 0) {
      tma_prefetch_desc(&tA);
      tma_prefetch_desc(&tB);
      int s = 0;
      uint32_t ph = 0;
      for (int64_t r = 0;; ++r) {
        const int64_t idx = snake(r, G, b);
        if (idx >= n_tiles) break;
        const int64_t t = order[idx];
        const int32_t I = static_cast<int32_t>(t / GN), J = static_cast<int32_t>(t % GN);
        const int64_t e0 = mstart[t], e1 = e0 + mcount[t];
        for (int64_t e = e0; e < e1; ++e) {
          const uint2 en = ment[e];
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], kStageBytes);
          tma_load_2d(sA + s * kAFloats, &tA, &full[s], static_cast<int32_t>(en.x) * 32, I * 128);
          tma_load_2d(sB + s * kBFloats, &tB, &full[s], J * 128, static_cast<int32_t>(en.x) * 32);
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------- compute warps (warpgroups 1-2)
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;" ::: "memory");
  // Warp w owns the C-tile pair (li, 2 jp), (li, 2 jp + 1), li = w / 2, jp = w % 2: 32 rows x 64
  // columns.  Lane (g, cg) = (lane / 8, lane % 8) holds rows g + 4 rr (rr < 8) and, in each tile
  // of the pair, the 4 columns 4 cg .. 4 cg + 3: an 8 x 8 register micro-tile.  Per 4-deep k slice
  // a warp reads 8 A and 8 B float4 from shared memory for 256 FFMA (the 4 x 8 one-tile-per-warp
  // layout read 12 for 128 and was bound by the shared pipe).  A k-step is computed when
  // either tile of the pair is kept (adjacent tiles are kept together: 1-3 % of the pair-steps of
  // the N = 16384 lambda = 0.99 sweep keep exactly one) and each tile's partial is added only if
  // kept.  Two-level accumulation in registers: the 32-term partial of a kept k-tile is added into
  // the running sum (first kept k: the partial itself), in ascending k.
  const int cw = warp - 4;
  const int li = cw >> 1, jp = cw & 1;
  const int bit_a = li * 4 + 2 * jp, bit_b = bit_a + 1;
  const int g = lane >> 3, cg = lane & 7;
  int s = 0;
  uint32_t ph = 0;
  for (int64_t r = 0;; ++r) {
    int64_t t, e0, e1;
    if constexpr (kFuse) {
      const int slot = static_cast<int>(r & 1);
      mbar_wait(&tl_full[slot], static_cast<uint32_t>((r >> 1) & 1));
      t = tl_info[2 * slot];
      e0 = t * fz.BK;
      e1 = e0 + tl_info[2 * slot + 1];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tl_empty[slot]);
      if (t < 0) break;
    } else {
      const int64_t idx = snake(r, G, b);
      if (idx >= n_tiles) break;
      t = order[idx];
      e0 = mstart[t];
      e1 = e0 + mcount[t];
    }
    const int64_t I = t / GN, J = t % GN;
    float run[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) run[i][j] = 0.f;
    bool first_a = true, first_b = true;
    for (int64_t e = e0; e < e1; ++e) {
      mbar_wait(&full[s], ph);
      // the k-step's keep bits (kFuse: written by this CTA's producer warp, read coherently)
      const uint32_t mask = kFuse ? __ldcg(&ment[e].y) : __ldg(&ment[e].y);
      const bool ka = (mask >> bit_a) & 1u, kb = (mask >> bit_b) & 1u;
      if (ka || kb) {
        const float* a_base = sA + s * kAFloats + (li * 32 + g) * 32;
        const float* b_base = sB + s * kBFloats + jp * 64 + cg * 4;
        float part[8][8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) part[i][j] = 0.f;
#pragma unroll kQUnroll
        for (int q = 0; q < 8; ++q) {   // partial unroll: the fully unrolled body (2048 FFMA) missed the i-cache
          float4 a4[8];
#pragma unroll
          for (int rr = 0; rr < 8; ++rr)   // row li*32 + g + 4 rr: its SWIZZLE_128B chunk is q ^ (row & 7)
            a4[rr] = *reinterpret_cast<const float4*>(a_base + rr * 4 * 32 + ((q ^ (g + 4 * (rr & 1))) << 2));
#pragma unroll
          for (int kq = 0; kq < 4; ++kq) {
            const float* brow = b_base + (q * 4 + kq) * 128;
            const float4 b0 = *reinterpret_cast<const float4*>(brow);        // tile 2 jp
            const float4 b1 = *reinterpret_cast<const float4*>(brow + 32);   // tile 2 jp + 1
#pragma unroll
            for (int rr = 0; rr < 8; ++rr) {
              const float av = comp(a4[rr], kq);
              part[rr][0] = fmaf(av, b0.x, part[rr][0]);
              part[rr][1] = fmaf(av, b0.y, part[rr][1]);
              part[rr][2] = fmaf(av, b0.z, part[rr][2]);
              part[rr][3] = fmaf(av, b0.w, part[rr][3]);
              part[rr][4] = fmaf(av, b1.x, part[rr][4]);
              part[rr][5] = fmaf(av, b1.y, part[rr][5]);
              part[rr][6] = fmaf(av, b1.z, part[rr][6]);
              part[rr][7] = fmaf(av, b1.w, part[rr][7]);
            }
          }
        }
        // second level: running sum += 32-term partial, for each kept tile of the pair
#pragma unroll
        for (int rr = 0; rr < 8; ++rr)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (ka) run[rr][j] = first_a ? part[rr][j] : run[rr][j] + part[rr][j];
            if (kb) run[rr][4 + j] = first_b ? part[rr][4 + j] : run[rr][4 + j] + part[rr][4 + j];
          }
        first_a = first_a && !ka;
        first_b = first_b && !kb;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == kStages) {
        s = 0;
        ph ^= 1;
      }
    }
    // epilogue: rows I*128 + li*32 + g + 4 rr; columns J*128 + jp*64 + 32 h + 4 cg .. + 3 for tile
    // 2 jp + h -- the 8 lanes of a row write 128 contiguous bytes per tile
    double tsq[2] = {0.0, 0.0};   // chained SpAMM: this lane's share of each tile's sum of squares
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      const int64_t m = I * 128 + li * 32 + g + 4 * rr;
      if (m >= M) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t n0 = J * 128 + jp * 64 + 32 * h + 4 * cg;
        const float4 v = make_float4(run[rr][4 * h], run[rr][4 * h + 1], run[rr][4 * h + 2], run[rr][4 * h + 3]);
        float* crow = C + m * ldc + n0;
        if (n0 + 4 <= N) {
          const float4 w = axpby4(ab, v, crow);
          __stcs(reinterpret_cast<float4*>(crow), w);
          if (nC != nullptr)
            tsq[h] += static_cast<double>(w.x) * static_cast<double>(w.x) + static_cast<double>(w.y) * static_cast<double>(w.y) +
                      static_cast<double>(w.z) * static_cast<double>(w.z) + static_cast<double>(w.w) * static_cast<double>(w.w);
        } else {
          const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (n0 + j < N) {
              const float w = axpby1(ab, vv[j], crow + j);
              crow[j] = w;
              tsq[h] += static_cast<double>(w) * static_cast<double>(w);
            }
        }
      }
    }
    if (nC != nullptr) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double x = tsq[h];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        const int64_t ti = I * 4 + li, tj = J * 4 + 2 * jp + h;
        if (lane == 0 && ti < BM && tj < BN) nC[ti * ldn + tj] = sqrt(x);
      }
    }
  }
}

}  // namespace

spamm_status launch_multiply_simt(Plan& p, const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                                  int64_t ldc, bool fuse, cudaStream_t s) {
  CUtensorMap tA, tB;
  SPAMM_TRY(encode_tmap_2d(&tA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, A, p.K, p.M, lda, 32, 128,
                           CU_TENSOR_MAP_SWIZZLE_128B));
  SPAMM_TRY(encode_tmap_2d(&tB, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, B, p.N, p.K, ldb, 128, 32,
                           CU_TENSOR_MAP_SWIZZLE_NONE));
  auto kern = fuse ? spamm_mul_simt_kernel<true> : spamm_mul_simt_kernel<false>;
  SPAMM_SET_SMEM(spamm_mul_simt_kernel<true>, static_cast<int>(kSmemBytes), p.device);
  SPAMM_SET_SMEM(spamm_mul_simt_kernel<false>, static_cast<int>(kSmemBytes), p.device);
  const int64_t n_tiles = p.range_on_device ? 0 : static_cast<int64_t>(p.row_end_macro - p.row_begin_macro) * p.GN;
  if (!p.range_on_device && n_tiles <= 0) return SPAMM_OK;
  const int grid = static_cast<int>(!p.range_on_device && n_tiles < p.num_sms ? n_tiles : p.num_sms);
  kern<<<grid, kThreads, kSmemBytes, s>>>(tA, tB, C, ldc, p.M, p.N, p.mstart, p.U, static_cast<const uint2*>(p.macro_ent),
                                          p.order, n_tiles, p.range_on_device ? p.d_range : nullptr, p.GN,
                                          Axpby{static_cast<float>(p.alpha), static_cast<float>(p.beta)},
                                          p.out_norms ? p.nC : nullptr, p.BN, p.BM, p.BN,
                                          XFuse{p.nA, p.nBt, p.BM, p.BK, p.BN, p.tau, p.U, p.L,
                                                static_cast<uint2*>(p.macro_ent), p.order,
                                                reinterpret_cast<unsigned long long*>(p.row_work),
                                                reinterpret_cast<unsigned long long*>(p.totals)});
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, spamm_mul_simt_kernel<false>);
    return fail(SPAMM_E_CUDA, std::string("spamm_mul_simt_kernel launch: ") + cudaGetErrorString(e) +
                                  " (regs " + std::to_string(fa.numRegs) + ", maxThreads " +
                                  std::to_string(fa.maxThreadsPerBlock) + ", static smem " +
                                  std::to_string(fa.sharedSizeBytes) + ", dyn smem " + std::to_string(kSmemBytes) +
                                  ", max dyn " + std::to_string(fa.maxDynamicSharedSizeBytes) + ")");
  }
  return SPAMM_OK;
}

}  // namespace spamm
