// multiply_simt.cu -- stage 3, FP32 CUDA-core path (multiplication kernel, Sec. 3.3,
// Alg. 2 lines 17-28).
//
// C[i,j] = sum_{kept k, ascending} A[i,k] * B[k,j], FP32 FMA.
//
// B200 design.  Persistent CTAs (one per SM) walk an LPT-ordered list of 128x128
// macro-tiles (4x4 C tiles).  For every k in the macro-tile's union list a TMA
// producer warp stages A[128 x 32] (SWIZZLE_128B) and B[32 x 128] in a 5-deep
// shared-memory ring guarded by mbarriers (replacing the paper's two half-block
// double buffer).  Sixteen compute warps each own one 32x32 C tile;
// the tile's keep bit for this k is warp-uniform, so a skipped pair costs a warp
// nothing but the barrier.  Each lane computes a 4x8 register micro-tile.
// Two-level accumulation: a 32-term register partial per kept k-tile is added into a
// running sum kept in shared memory, which keeps N=65536
// within 1e-5 and leaves registers for 17 warps (4 SMSPs x <=5 warps x 96 regs).
#include "internal.h"
#include "sm100.cuh"

namespace spamm {
namespace {

using namespace sm100;

constexpr int kStages = 5;
constexpr int kComputeWarps = 16;
constexpr int kThreads = (kComputeWarps + 1) * 32;
constexpr int kAFloats = 128 * 32;
constexpr int kBFloats = 32 * 128;
constexpr int kStageBytes = (kAFloats + kBFloats) * 4;
constexpr int kAccBytes = kComputeWarps * 32 * 32 * 4;   // running sums, [warp][8 float4][32 lanes]
constexpr size_t kSmemBytes = 1024 + static_cast<size_t>(kStages) * kStageBytes + kAccBytes + 256;

__device__ __forceinline__ int64_t snake(int64_t r, int G, int b) { return r * G + ((r & 1) ? (G - 1 - b) : b); }

__device__ __forceinline__ float comp(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

__global__ void __launch_bounds__(kThreads, 1)
    spamm_mul_simt_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                          float* __restrict__ C, int64_t ldc, int64_t M, int64_t N,
                          const int64_t* __restrict__ mstart, const int64_t* __restrict__ mcount, const uint2* __restrict__ ment,
                          const int32_t* __restrict__ order, int64_t n_tiles, const int64_t* __restrict__ rng,
                          int64_t GN, const Axpby ab, double* __restrict__ nC, int64_t ldn, int64_t BM, int64_t BN) {
  if (rng != nullptr) n_tiles = (rng[1] - rng[0]) * GN;   // multi-GPU range decided on the device
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned base derived from smem_raw by an offset (not an integer round trip), so the compiler
  // keeps the shared address space: LDS/STS instead of generic LD/ST for the operand and sum reads
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  float* sA = reinterpret_cast<float*>(smem);
  float* sB = sA + kStages * kAFloats;
  float4* sAcc = reinterpret_cast<float4*>(smem + static_cast<size_t>(kStages) * kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(kStages) * kStageBytes + kAccBytes);
  uint64_t* empty = full + kStages;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kComputeWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int G = gridDim.x, b = blockIdx.x;

  if (warp == kComputeWarps) {
    // ------------------------------------------------------ TMA producer
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

  // -------------------------------------------------------- compute warps
  const int li = warp >> 2, lj = warp & 3, bit = li * 4 + lj;
  // lane -> (row g, column group cg) = (lane / 4, lane % 4): the epilogue's row segments are 128-byte
  // contiguous.  Measured at N = 16384 (profiles/r02zf_*): with LDS (see smem above) 6.26 ms vs 6.47 ms
  // for (lane % 8, lane / 8) and 6.90 ms with generic loads; the shared pipe stays the limiter (A loads
  // 2, B loads 4 wavefronts per LDS.128 here; 4 and 2 with the other mapping)
  const int g = lane >> 2, cg = lane & 3;
  int s = 0;
  uint32_t ph = 0;
  for (int64_t r = 0;; ++r) {
    const int64_t idx = snake(r, G, b);
    if (idx >= n_tiles) break;
    const int64_t t = order[idx];
    const int64_t I = t / GN, J = t % GN;
    float4* acc = sAcc + warp * 8 * 32 + lane;   // acc[j4 * 32]: outputs 4*j4 .. 4*j4+3 of this lane
    bool first = true;
    const int64_t e0 = mstart[t], e1 = e0 + mcount[t];
    for (int64_t e = e0; e < e1; ++e) {
      mbar_wait(&full[s], ph);
      const uint32_t mask = __ldg(&ment[e].y);   // the k-step's keep bits (read-only, L1-resident)
      if ((mask >> bit) & 1u) {
        const float* a_base = sA + s * kAFloats + (li * 32 + g) * 32;
        const float* b_base = sB + s * kBFloats + lj * 32 + cg * 8;
        float part[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) part[i][j] = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 a4[4];
#pragma unroll
          for (int rr = 0; rr < 4; ++rr)
            a4[rr] = *reinterpret_cast<const float4*>(a_base + rr * 8 * 32 + ((q ^ g) << 2));
#pragma unroll
          for (int kq = 0; kq < 4; ++kq) {
            const float* brow = b_base + (q * 4 + kq) * 128;
            const float4 b0 = *reinterpret_cast<const float4*>(brow);
            const float4 b1 = *reinterpret_cast<const float4*>(brow + 4);
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
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
        // second level: running sum += 32-term partial
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const int rr = j4 >> 1, c0 = (j4 & 1) * 4;
          float4 v = make_float4(part[rr][c0], part[rr][c0 + 1], part[rr][c0 + 2], part[rr][c0 + 3]);
          if (!first) {
            const float4 o = acc[j4 * 32];
            v.x += o.x;
            v.y += o.y;
            v.z += o.z;
            v.w += o.w;
          }
          acc[j4 * 32] = v;
        }
        first = false;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == kStages) {
        s = 0;
        ph ^= 1;
      }
    }
    // epilogue: rows I*128 + li*32 + g + 8*rr, cols J*128 + lj*32 + cg*8 .. +7
    const int64_t n0 = J * 128 + lj * 32 + cg * 8;
    double tsq = 0.0;   // chained SpAMM: this lane's share of the tile's sum of squares
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const int64_t m = I * 128 + li * 32 + g + 8 * rr;
      const float4 v0 = first ? make_float4(0.f, 0.f, 0.f, 0.f) : acc[(2 * rr) * 32];
      const float4 v1 = first ? make_float4(0.f, 0.f, 0.f, 0.f) : acc[(2 * rr + 1) * 32];
      if (m >= M) continue;
      float* crow = C + m * ldc + n0;
      if (n0 + 8 <= N) {
        const float4 w0 = axpby4(ab, v0, crow), w1 = axpby4(ab, v1, crow + 4);
        __stcs(reinterpret_cast<float4*>(crow), w0);
        __stcs(reinterpret_cast<float4*>(crow + 4), w1);
        if (nC != nullptr) {
          const float ww[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
          for (int j = 0; j < 8; ++j) tsq += static_cast<double>(ww[j]) * static_cast<double>(ww[j]);
        }
      } else {
        const float vv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (n0 + j < N) {
            const float w = axpby1(ab, vv[j], crow + j);
            crow[j] = w;
            tsq += static_cast<double>(w) * static_cast<double>(w);
          }
      }
    }
    if (nC != nullptr) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) tsq += __shfl_xor_sync(0xffffffffu, tsq, o);
      const int64_t ti = I * 4 + li, tj = J * 4 + lj;
      if (lane == 0 && ti < BM && tj < BN) nC[ti * ldn + tj] = sqrt(tsq);
    }
  }
}

}  // namespace

spamm_status launch_multiply_simt(Plan& p, const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                                  int64_t ldc, cudaStream_t s) {
  CUtensorMap tA, tB;
  SPAMM_TRY(encode_tmap_2d(&tA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, A, p.K, p.M, lda, 32, 128,
                           CU_TENSOR_MAP_SWIZZLE_128B));
  SPAMM_TRY(encode_tmap_2d(&tB, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, B, p.N, p.K, ldb, 128, 32,
                           CU_TENSOR_MAP_SWIZZLE_NONE));
  SPAMM_SET_SMEM(spamm_mul_simt_kernel, static_cast<int>(kSmemBytes), p.device);
  const int64_t n_tiles = p.range_on_device ? 0 : static_cast<int64_t>(p.row_end_macro - p.row_begin_macro) * p.GN;
  if (!p.range_on_device && n_tiles <= 0) return SPAMM_OK;
  const int grid = static_cast<int>(!p.range_on_device && n_tiles < p.num_sms ? n_tiles : p.num_sms);
  spamm_mul_simt_kernel<<<grid, kThreads, kSmemBytes, s>>>(tA, tB, C, ldc, p.M, p.N, p.mstart, p.U,
                                                           static_cast<const uint2*>(p.macro_ent), p.order, n_tiles,
                                                           p.range_on_device ? p.d_range : nullptr, p.GN,
                                                           Axpby{static_cast<float>(p.alpha), static_cast<float>(p.beta)},
                                                           p.out_norms ? p.nC : nullptr, p.BN, p.BM, p.BN);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, spamm_mul_simt_kernel);
    return fail(SPAMM_E_CUDA, std::string("spamm_mul_simt_kernel launch: ") + cudaGetErrorString(e) +
                                  " (regs " + std::to_string(fa.numRegs) + ", maxThreads " +
                                  std::to_string(fa.maxThreadsPerBlock) + ", static smem " +
                                  std::to_string(fa.sharedSizeBytes) + ", dyn smem " + std::to_string(kSmemBytes) +
                                  ", max dyn " + std::to_string(fa.maxDynamicSharedSizeBytes) + ")");
  }
  return SPAMM_OK;
}

}  // namespace spamm
