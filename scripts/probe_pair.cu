// probe_pair.cu -- semantics of tcgen05.mma.cta_group::2 (CTA pair, M = 256) as used by the
// pair kernel: which B columns each CTA must hold, how the 8-word disable-output-lane mask
// maps onto the two CTAs' TMEM lanes, and MN-major SWIZZLE_32B B halves of 16 columns.
//   A: 256 x 16 (K-major SW64; CTA r holds rows 128r..128r+127)
//   B: 16 x N  (MN-major; CTA r holds B columns [r*N/2, (r+1)*N/2) -- hypothesis H1)
// Test 1: N=256 SW64 boxes, all lanes; Test 2: N=64; Test 3: mask; Test 4: N=32 with SW32.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstring>
#include <vector>
#include "../paper_2103_13042_b200/csrc/sm100.cuh"
using namespace spamm::sm100;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void umma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc, const uint32_t* m) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, {%5, %6, %7, %8, %9, %10, %11, %12}, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(m[0]), "r"(m[1]), "r"(m[2]), "r"(m[3]), "r"(m[4]), "r"(m[5]),
      "r"(m[6]), "r"(m[7])
      : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)), "h"((uint16_t)3)
               : "memory");
}

struct Maps { CUtensorMap a, b64, b32; };

// mode 0: N=256 (SW64, 4 boxes per CTA); 1: N=64 (1 box per CTA); 2: N=256 + masked second MMA;
// 3: N=32, SW32 16-column halves
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) pair_kernel(const __grid_constant__ Maps mp, int mode, float* D) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full, done;
  __shared__ uint32_t tslot;
  const uint32_t r = cta_rank();
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&full, 1); mbar_init(&done, 1); fence_mbar_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tbase = tslot;
  uint8_t* sA = sm;            // 128 x 32 k (we use k 0..15), 8 KB
  uint8_t* sB = sm + 8192;     // B half
  if (threadIdx.x == 0) {
    int bytes = 8192;
    if (mode == 0 || mode == 2) bytes += 4 * 2048;
    if (mode == 1) bytes += 2048;
    if (mode == 3) bytes += 1024;
    mbar_arrive_expect_tx(&full, bytes);
    tma_load_2d(sA, &mp.a, &full, 0, 128 * r);
    if (mode == 0 || mode == 2) tma_load_3d(sB, &mp.b64, &full, 0, 0, 4 * r);
    if (mode == 1) tma_load_3d(sB, &mp.b64, &full, 0, 0, r);
    if (mode == 3) tma_load_3d(sB, &mp.b32, &full, 0, 0, r);
  }
  mbar_wait(&full, 0);
  tc_fence_before();
  cluster_sync_all();   // both halves resident
  tc_fence_after();
  if (r == 0 && threadIdx.x == 0) {
    const int N = (mode == 1) ? 64 : (mode == 3 ? 32 : 256);
    const uint32_t idesc = idesc_f16(1, 256, N, 0, 1);
    const uint64_t ad = smem_desc(smem_u32(sA), 16, 512, kLayoutSW64);
    const uint64_t bd = (mode == 3) ? smem_desc(smem_u32(sB), 1024, 256, 6u) : smem_desc(smem_u32(sB), 2048, 512, kLayoutSW64);
    uint32_t m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    umma2(tbase, ad, bd, idesc, 0u, m);
    if (mode == 2) {   // second MMA, accumulate, only words 1 and 6 enabled
      for (int w = 0; w < 8; ++w) m[w] = (w == 1 || w == 6) ? 0u : 0xFFFFFFFFu;
      umma2(tbase, ad, bd, idesc, 1u, m);
    }
    commit2(&done);
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  // each CTA: its 128 lanes x 256 columns -> D[128 r + lane][col]
  uint32_t v[32];
  for (int c = 0; c < 256; c += 32) {
    tmem_ld_32x32b_x32(tbase + ((warp * 32) << 16) + c, v);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) D[(128 * r + warp * 32 + (threadIdx.x & 31)) * 256 + c + i] = __uint_as_float(v[i]);
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tbase) : "memory");
}

int main() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int M = 256, K = 64, NN = 512;
  std::vector<__nv_bfloat16> hA(M * K), hB(K * NN);
  std::vector<float> fA(M * K), fB(K * NN);
  for (int i = 0; i < M * K; ++i) { float x = (float)((i * 7 + 3) % 5 - 2); fA[i] = x; hA[i] = __float2bfloat16(x); }
  for (int i = 0; i < K * NN; ++i) { float x = (float)((i * 5 + 1) % 7 - 3); fB[i] = x; hB[i] = __float2bfloat16(x); }
  void *dA, *dB; float* dD;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, K * NN * 2); cudaMalloc(&dD, 256 * 256 * 4);
  cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), K * NN * 2, cudaMemcpyHostToDevice);
  Maps mp;
  {
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M}, str[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    printf("enc a %d\n", (int)encode(&mp.a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dA, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                     CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  {
    cuuint64_t dims[3] = {32, (cuuint64_t)K, (cuuint64_t)(NN / 32)}, str[2] = {(cuuint64_t)NN * 2, 64};
    cuuint32_t box[3] = {32, 32, 4}, es[3] = {1, 1, 1};
    printf("enc b64 %d\n", (int)encode(&mp.b64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dB, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                       CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    // box count per TMA: 4 for modes 0/2, 1 for mode 1 -> separate map with 1 box
  }
  CUtensorMap b64_1;
  {
    cuuint64_t dims[3] = {32, (cuuint64_t)K, (cuuint64_t)(NN / 32)}, str[2] = {(cuuint64_t)NN * 2, 64};
    cuuint32_t box[3] = {32, 32, 1}, es[3] = {1, 1, 1};
    encode(&b64_1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dB, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t dims[3] = {16, (cuuint64_t)K, (cuuint64_t)(NN / 16)}, str[2] = {(cuuint64_t)NN * 2, 32};
    cuuint32_t box[3] = {16, 32, 1}, es[3] = {1, 1, 1};
    printf("enc b32 %d\n", (int)encode(&mp.b32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dB, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                       CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  cudaFuncSetAttribute(pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  std::vector<float> hD(256 * 256);
  for (int mode = 0; mode < 4; ++mode) {
    Maps m2 = mp;
    if (mode == 1) m2.b64 = b64_1;
    cudaMemset(dD, 0, 256 * 256 * 4);
    pair_kernel<<<2, 128, 40000>>>(m2, mode, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(hD.data(), dD, 256 * 256 * 4, cudaMemcpyDeviceToHost);
    const int N = mode == 1 ? 64 : (mode == 3 ? 32 : 256);
    // hypothesis H1: D[m][n] = sum_k A[m][k] * B[k][n] for n < N, k < 16
    int bad = 0;
    for (int mm = 0; mm < 256; ++mm)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < 16; ++k) ref += (double)fA[mm * K + k] * fB[k * NN + n];
        double want = ref;
        if (mode == 2) { const int w = mm / 32; if (w == 1 || w == 6) want = 2 * ref; }
        if (hD[mm * 256 + n] != (float)want) { if (bad < 5) printf("  mode %d D[%d][%d] = %g want %g\n", mode, mm, n, hD[mm * 256 + n], want); ++bad; }
      }
    printf("mode %d (N=%d): %d mismatches of %d\n", mode, N, bad, 256 * N);
  }
  return 0;
}
