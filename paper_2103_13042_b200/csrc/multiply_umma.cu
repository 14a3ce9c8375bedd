// multiply_umma.cu -- stage 3, tensor-core path (tensor-core multiplication kernel,
// Sec. 3.3, Alg. 3), BF16/FP16 inputs, FP32 accumulation.
//
// C[i,j] = sum_{kept k, ascending} A[i,k] * B[k,j]; the paper's FP32
// accumulator fragment becomes an FP32 accumulator in TMEM.
//
// B200 design (tcgen05, not the paper's wmma):
//   * persistent CTAs (one per SM) over an LPT-ordered list of 128x256 macro-tiles
//     (4 x 8 C tiles of 32x32);
//   * warp 0: TMA producer -- per kept k of the macro-tile's union list, A[128 x 32]
//     (K-major, SWIZZLE_64B) and only the B[32 x 32] boxes (MN-major, SWIZZLE_64B)
//     whose C-tile column has a kept pair, into an 8-deep smem ring (mbarriers);
//   * warp 1: one elected thread issues tcgen05.mma kind::f16 M=128, K=16 (x2 per
//     k-tile).  The 4 x 8 keep bits of the k-step are split into runs of adjacent
//     C-tile columns with the same 4-bit row pattern; each run is ONE MMA with
//     N = 32*run and the disable-output-lane mask switching off the 32-lane groups
//     (C-tile rows) whose pair is skipped -- exact leaf-level skip semantics
//     (Alg. 2 l.3-8) on a 128-row MMA;
//   * warps 4-7: epilogue -- TMEM -> registers -> C (FP32), then zero the
//     accumulator for its next use; two TMEM accumulator buffers (2 x 256 columns)
//     overlap the epilogue of one macro-tile with the MMAs of the next.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "internal.h"
#include "sm100.cuh"

namespace spamm {
namespace {

using namespace sm100;

constexpr int kStages = 8;
constexpr int kABytes = 128 * 32 * 2;           // 8 KB
constexpr int kBBoxBytes = 32 * 32 * 2;         // 2 KB per 32 x 32 box
constexpr int kBBytes = 8 * kBBoxBytes;         // 16 KB
constexpr int kThreads = 256;
constexpr size_t kSmemBytes = 1024 + static_cast<size_t>(kStages) * (kABytes + kBBytes) + 256;

__device__ __forceinline__ int64_t snake(int64_t r, int G, int b) { return r * G + ((r & 1) ? (G - 1 - b) : b); }

__device__ __forceinline__ uint32_t row_pattern(uint32_t mask, int lj) {
  return ((mask >> lj) & 1u) | (((mask >> (8 + lj)) & 1u) << 1) | (((mask >> (16 + lj)) & 1u) << 2) |
         (((mask >> (24 + lj)) & 1u) << 3);
}

template <uint32_t kFmt>
__global__ void __launch_bounds__(kThreads, 1)
    spamm_mul_umma_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                          float* __restrict__ C, int64_t ldc, int64_t M, int64_t N,
                          const int64_t* __restrict__ mptr, const uint2* __restrict__ ment,
                          const int32_t* __restrict__ order, int64_t n_tiles, int64_t GN) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(kStages) * (kABytes + kBBytes));
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* smask = reinterpret_cast<uint32_t*>(tempty + 2);
  uint32_t* tmem_slot = smask + kStages;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int G = gridDim.x, b = blockIdx.x;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tA);
      tma_prefetch_desc(&tB);
      int s = 0;
      uint32_t ph = 0;
      for (int64_t r = 0;; ++r) {
        const int64_t idx = snake(r, G, b);
        if (idx >= n_tiles) break;
        const int64_t t = order[idx];
        const int32_t I = static_cast<int32_t>(t / GN), J = static_cast<int32_t>(t % GN);
        const int64_t e1 = mptr[t + 1];
        for (int64_t e = mptr[t]; e < e1; ++e) {
          const uint2 en = ment[e];
          const uint32_t cols = (en.y | (en.y >> 8) | (en.y >> 16) | (en.y >> 24)) & 0xFFu;
          mbar_wait(&empty[s], ph ^ 1);
          smask[s] = en.y;
          mbar_arrive_expect_tx(&full[s], kABytes + kBBoxBytes * __popc(cols));
          const int32_t k0 = static_cast<int32_t>(en.x) * 32;
          tma_load_2d(sA + s * kABytes, &tA, &full[s], k0, I * 128);
#pragma unroll
          for (int lj = 0; lj < 8; ++lj)
            if ((cols >> lj) & 1u)
              tma_load_2d(sB + s * kBBytes + lj * kBBoxBytes, &tB, &full[s], J * 256 + lj * 32, k0);
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    int s = 0;
    uint32_t ph = 0;
    int64_t it = 0;
    for (int64_t r = 0;; ++r, ++it) {
      const int64_t idx = snake(r, G, b);
      if (idx >= n_tiles) break;
      const int64_t t = order[idx];
      const int buf = static_cast<int>(it & 1);
      mbar_wait(&tempty[buf], static_cast<uint32_t>((it >> 1) & 1));
      tc_fence_after();
      const uint32_t dcol = tbase + static_cast<uint32_t>(buf) * 256u;
      const int64_t e1 = mptr[t + 1];
      for (int64_t e = mptr[t]; e < e1; ++e) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t mask = smask[s];
          const uint32_t a_addr = smem_u32(sA + s * kABytes);
          const uint32_t b_addr = smem_u32(sB + s * kBBytes);
          int j = 0;
          while (j < 8) {
            const uint32_t pat = row_pattern(mask, j);
            if (pat == 0u) {
              ++j;
              continue;
            }
            int j1 = j + 1;
            while (j1 < 8 && row_pattern(mask, j1) == pat) ++j1;
            const uint32_t run = static_cast<uint32_t>(j1 - j);
            const uint32_t idesc = idesc_f16(kFmt, 128, 32u * run, 0, 1);
            const uint32_t w0 = (pat & 1u) ? 0u : 0xFFFFFFFFu;
            const uint32_t w1 = (pat & 2u) ? 0u : 0xFFFFFFFFu;
            const uint32_t w2 = (pat & 4u) ? 0u : 0xFFFFFFFFu;
            const uint32_t w3 = (pat & 8u) ? 0u : 0xFFFFFFFFu;
#pragma unroll
            for (int kh = 0; kh < 2; ++kh) {
              const uint64_t ad = smem_desc(a_addr + kh * 32, 16, 512, kLayoutSW64);
              const uint64_t bd = smem_desc(b_addr + j * kBBoxBytes + kh * 1024, kBBoxBytes, 512, kLayoutSW64);
              umma_f16(dcol + static_cast<uint32_t>(j) * 32u, ad, bd, idesc, 1u, w0, w1, w2, w3);
            }
            j = j1;
          }
          umma_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == kStages) {
          s = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) umma_commit(&tfull[buf]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // --------------------------------------------------------------- epilogue
    const int q = warp & 3;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    for (int buf = 0; buf < 2; ++buf)
      for (int c = 0; c < 8; ++c) tmem_st_32x32b_x32_zero(tbase + lane_off + buf * 256 + c * 32);
    tmem_wait_st();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&tempty[0]);
      mbar_arrive(&tempty[1]);
    }
    int64_t it = 0;
    for (int64_t r = 0;; ++r, ++it) {
      const int64_t idx = snake(r, G, b);
      if (idx >= n_tiles) break;
      const int64_t t = order[idx];
      const int64_t I = t / GN, J = t % GN;
      const int buf = static_cast<int>(it & 1);
      mbar_wait(&tfull[buf], static_cast<uint32_t>((it >> 1) & 1));
      tc_fence_after();
      const int64_t row = I * 128 + q * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        const uint32_t taddr = tbase + lane_off + buf * 256 + c * 32;
        uint32_t v[32];
        tmem_ld_32x32b_x32(taddr, v);
        tmem_wait_ld();
        tmem_st_32x32b_x32_zero(taddr);
        const int64_t n0 = J * 256 + c * 32;
        if (row < M && n0 < N) {
          float* crow = C + row * ldc + n0;
          if (n0 + 32 <= N) {
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              __stcs(reinterpret_cast<float4*>(crow + e),
                     make_float4(__uint_as_float(v[e]), __uint_as_float(v[e + 1]), __uint_as_float(v[e + 2]),
                                 __uint_as_float(v[e + 3])));
          } else {
            for (int e = 0; e < 32; ++e)
              if (n0 + e < N) crow[e] = __uint_as_float(v[e]);
          }
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tbase);
}

template <uint32_t kFmt>
spamm_status launch_fmt(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                        cudaStream_t s, CUtensorMapDataType dt) {
  CUtensorMap tA, tB;
  SPAMM_TRY(encode_tmap_2d(&tA, dt, 2, A, p.K, p.M, lda, 32, 128, CU_TENSOR_MAP_SWIZZLE_64B));
  SPAMM_TRY(encode_tmap_2d(&tB, dt, 2, B, p.N, p.K, ldb, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B));
  static bool attr_set = false;
  if (!attr_set) {
    SPAMM_CUDA_TRY(cudaFuncSetAttribute(spamm_mul_umma_kernel<kFmt>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kSmemBytes)));
    attr_set = true;
  }
  const int64_t n_tiles = (p.row_end_macro - p.row_begin_macro) * p.GN;
  if (n_tiles <= 0) return SPAMM_OK;
  const int grid = static_cast<int>(n_tiles < p.num_sms ? n_tiles : p.num_sms);
  spamm_mul_umma_kernel<kFmt><<<grid, kThreads, kSmemBytes, s>>>(tA, tB, C, ldc, p.M, p.N, p.macro_ptr,
                                                                 p.macro_ent, p.order, n_tiles, p.GN);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

}  // namespace

spamm_status launch_multiply_umma(Plan& p, const void* A, int64_t lda, const void* B, int64_t ldb, float* C,
                                  int64_t ldc, cudaStream_t s) {
  if (p.prec == SPAMM_BF16) return launch_fmt<1>(p, A, lda, B, ldb, C, ldc, s, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
  return launch_fmt<0>(p, A, lda, B, ldb, C, ldc, s, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
}

}  // namespace spamm
