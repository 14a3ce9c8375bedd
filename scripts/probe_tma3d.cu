// probe_tma3d.cu -- can a 3-D tensor map with a non-monotonic stride (n_inner=32, k, n_outer)
// load B[32 k x (32*nb) n] as nb stacked [32 k][32 n] SWIZZLE_64B boxes in one TMA?
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <vector>
#include "../paper_2103_13042_b200/csrc/sm100.cuh"
using namespace spamm::sm100;

__global__ void k3d(const __grid_constant__ CUtensorMap t3, const __grid_constant__ CUtensorMap t2, int nb, int c0,
                    uint16_t* out3, uint16_t* out2) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 2 * nb * 2048);
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
        ::"r"(smem_u32(sm)), "l"(reinterpret_cast<uint64_t>(&t3)), "r"(smem_u32(&bar)), "r"(0), "r"(0), "r"(c0)
        : "memory");
    for (int q = 0; q < nb; ++q) tma_load_2d(sm + 16384 + q * 2048, &t2, &bar, (c0 + q) * 32, 0);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < nb * 1024; i += blockDim.x) {
    out3[i] = reinterpret_cast<uint16_t*>(sm)[i];
    out2[i] = reinterpret_cast<uint16_t*>(sm + 16384)[i];
  }
}

int main() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int K = 64, N = 512;
  std::vector<uint16_t> h(K * N);
  for (int i = 0; i < K * N; ++i) h[i] = (uint16_t)(i * 7 + 3);
  uint16_t *dB, *o3, *o2; cudaMalloc(&dB, K * N * 2); cudaMalloc(&o3, 8 * 2048); cudaMalloc(&o2, 8 * 2048);
  cudaMemcpy(dB, h.data(), K * N * 2, cudaMemcpyHostToDevice);
  CUtensorMap t3, t2;
  int fails = 0;
  for (int nb : {8, 4, 2, 1}) {
    cuuint64_t dims[3] = {32, (cuuint64_t)K, (cuuint64_t)(N / 32)};
    cuuint64_t strides[2] = {(cuuint64_t)N * 2, 64};
    cuuint32_t box[3] = {32, 32, (cuuint32_t)nb}, es[3] = {1, 1, 1};
    CUresult r = encode(&t3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dB, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode 3d nb=%d -> %d\n", nb, (int)r);
    if (r != CUDA_SUCCESS) { ++fails; continue; }
    cuuint64_t d2[2] = {(cuuint64_t)N, (cuuint64_t)K};
    cuuint64_t s2[1] = {(cuuint64_t)N * 2};
    cuuint32_t b2[2] = {32, 32}, e2[2] = {1, 1};
    encode(&t2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dB, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k3d, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    for (int c0 : {0, 3, 16 - nb}) {
      k3d<<<1, 128, 40000>>>(t3, t2, nb, c0, o3, o2);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<uint16_t> a(nb * 1024), b(nb * 1024);
      cudaMemcpy(a.data(), o3, nb * 2048, cudaMemcpyDeviceToHost);
      cudaMemcpy(b.data(), o2, nb * 2048, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int i = 0; i < nb * 1024; ++i) bad += a[i] != b[i];
      printf("%s nb=%d c0=%d cuda=%s mismatches=%d\n", bad || e ? "FAIL" : "PASS", nb, c0, cudaGetErrorString(e), bad);
      fails += bad != 0 || e != cudaSuccess;
    }
  }
  printf("%s probe_tma3d\n", fails ? "FAIL" : "PASS");
  return fails != 0;
}
