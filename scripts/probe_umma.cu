// probe_umma.cu -- one-CTA hardware probe of the building blocks the BF16 SpAMM
// multiply relies on (run on a B200 before trusting the kernel):
//   * TMA 2-D loads with SWIZZLE_64B of a K-major A tile [128 x 32] and of
//     8 MN-major B boxes [32 k x 32 n];
//   * UMMA smem descriptors for both, K advanced by 16 inside the 64-B swizzle row;
//   * N = 32*run starting at any 32-column box;
//   * tcgen05.mma disable-output-lane: which bit/word masks which TMEM lane.
// Prints one PASS/FAIL line per case and exits non-zero on failure.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cmath>
#include "../paper_2103_13042_b200/csrc/sm100.cuh"

using namespace spamm::sm100;

struct Case { int j0, run; uint32_t m[4]; int accumulate_twice; };

__global__ void probe_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                             float* out, int j0, int run, uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;               // 8 KB
  uint8_t* sB = smem + 8192;        // 16 KB
  __shared__ uint64_t bar_full, bar_mma;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar_full, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<256>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar_full, 8192 + 16384);
    tma_load_2d(sA, &tA, &bar_full, 0, 0);
    for (int b = 0; b < 8; ++b) tma_load_2d(sB + b * 2048, &tB, &bar_full, b * 32, 0);
  }
  // zero the accumulator columns first (all 4 warps)
  for (int c = 0; c < 256; c += 32) tmem_st_32x32b_x32_zero(tbase + ((warp * 32u) << 16) + c);
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    mbar_wait(&bar_full, 0);
    tc_fence_after();
    if (elect_one()) {
      const uint32_t idesc = idesc_f16(1, 128, 32u * run, 0, 1);
      for (int kh = 0; kh < 2; ++kh) {
        uint64_t ad = smem_desc(smem_u32(sA) + kh * 32, 16, 512, kLayoutSW64);
        uint64_t bd = smem_desc(smem_u32(sB) + j0 * 2048 + kh * 1024, 2048, 512, kLayoutSW64);
        umma_f16(tbase + j0 * 32, ad, bd, idesc, 1u, m0, m1, m2, m3);
      }
      umma_commit(&bar_mma);
    }
    __syncwarp();
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  for (int c = 0; c < 256; c += 32) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tbase + ((warp * 32u) << 16) + c, r);
    tmem_wait_ld();
    for (int e = 0; e < 32; ++e) out[(warp * 32 + threadIdx.x % 32) * 256 + c + e] = __uint_as_float(r[e]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<256>(tbase);
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

int main() {
  auto encode = get_encode();
  if (!encode) { printf("FAIL no cuTensorMapEncodeTiled\n"); return 2; }
  const int M = 128, K = 32, N = 256;
  std::vector<__nv_bfloat16> hA(M * K), hB(K * N);
  std::vector<float> fA(M * K), fB(K * N);
  for (int i = 0; i < M * K; ++i) { float v = (float)((i * 37 % 17) - 8) / 8.0f; hA[i] = __float2bfloat16(v); fA[i] = __bfloat162float(hA[i]); }
  for (int i = 0; i < K * N; ++i) { float v = (float)((i * 53 % 13) - 6) / 4.0f; hB[i] = __float2bfloat16(v); fB[i] = __bfloat162float(hB[i]); }
  __nv_bfloat16 *dA, *dB; float* dO;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, K * N * 2); cudaMalloc(&dO, 128 * 256 * 4);
  cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), K * N * 2, cudaMemcpyHostToDevice);
  CUtensorMap tA, tB;
  {
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    CUresult r = encode(&tA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dA, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("FAIL encode A %d\n", (int)r); return 2; }
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)K};
    cuuint64_t strides[1] = {(cuuint64_t)N * 2};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    CUresult r = encode(&tB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dB, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("FAIL encode B %d\n", (int)r); return 2; }
  }
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 1024);
  // reference full product
  std::vector<double> ref(128 * 256, 0.0);
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 256; ++j) {
      double s = 0; for (int k = 0; k < 32; ++k) s += (double)fA[i * K + k] * fB[k * N + j];
      ref[i * 256 + j] = s;
    }
  Case cases[] = {
      {0, 8, {0, 0, 0, 0}, 0},
      {2, 2, {0, 0, 0, 0}, 0},
      {7, 1, {0, 0, 0, 0}, 0},
      {1, 3, {0xFFFFFFFFu, 0, 0xFFFFFFFFu, 0}, 0},
      {0, 4, {0, 0xFFFFFFFFu, 0, 0}, 0},
      {3, 5, {0x0000FFFFu, 0, 0, 0x80000001u}, 0},
  };
  int fails = 0;
  std::vector<float> out(128 * 256);
  for (auto& c : cases) {
    cudaMemset(dO, 0xFF, 128 * 256 * 4);
    probe_kernel<<<1, 128, 32768 + 1024>>>(tA, tB, dO, c.j0, c.run, c.m[0], c.m[1], c.m[2], c.m[3]);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("FAIL case j0=%d run=%d cuda %s\n", c.j0, c.run, cudaGetErrorString(e)); return 3; }
    cudaMemcpy(out.data(), dO, 128 * 256 * 4, cudaMemcpyDeviceToHost);
    // hypothesis H1: word w bit b disables lane 32*w+b
    int bad = 0, bad_alt = 0;
    for (int i = 0; i < 128; ++i) {
      bool dis = (c.m[i / 32] >> (i % 32)) & 1u;
      bool dis_alt = (c.m[3 - i / 32] >> (i % 32)) & 1u;  // alternative: reversed word order
      for (int j = 0; j < 256; ++j) {
        bool in_run = j >= c.j0 * 32 && j < (c.j0 + c.run) * 32;
        double e1 = (in_run && !dis) ? ref[i * 256 + j] : 0.0;
        double e2 = (in_run && !dis_alt) ? ref[i * 256 + j] : 0.0;
        if (std::fabs(out[i * 256 + j] - e1) > 1e-3 * (1 + std::fabs(e1))) ++bad;
        if (std::fabs(out[i * 256 + j] - e2) > 1e-3 * (1 + std::fabs(e2))) ++bad_alt;
      }
    }
    printf("%s case j0=%d run=%d mask=%08x,%08x,%08x,%08x mismatches=%d (reversed-word hypothesis: %d)\n",
           bad ? "FAIL" : "PASS", c.j0, c.run, c.m[0], c.m[1], c.m[2], c.m[3], bad, bad_alt);
    if (bad) {
      ++fails;
      int shown = 0;
      for (int i = 0; i < 128 && shown < 6; i += 17) { printf("   row %d: out[j0*32]=%g ref=%g\n", i, out[i*256+c.j0*32], ref[i*256+c.j0*32]); ++shown; }
    }
  }
  printf("%s probe_umma (%d failing cases)\n", fails ? "FAIL" : "PASS", fails);
  return fails ? 1 : 0;
}
