// probe_tma_rings.cu -- is L2 -> SMEM TMA throughput limited per CTA or per ring (issuing
// thread + its in-flight stages)?  1 CTA/SM with R independent rings (own producer warp, own
// consumer warp, S stages of A 8 KB [128 x 32] SW64 + B 16 KB 3-D {32,32,8} SW64 each), vs
// 2 CTAs/SM with one ring.  The consumer only releases stages.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include "../paper_2103_13042_b200/csrc/sm100.cuh"
using namespace spamm::sm100;

constexpr int kStageBytes = 24576;

__global__ void rings(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int R, int S,
                      int iters, int ymax, int zmax) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[4][8], empty[4][8];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int r = 0; r < R; ++r)
      for (int s = 0; s < S; ++s) { mbar_init(&full[r][s], 1); mbar_init(&empty[r][s], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int r = warp / 2;
  if (r >= R || lane != 0) return;
  uint8_t* base = sm + r * S * kStageBytes;
  if ((warp & 1) == 0) {
    uint32_t h = (blockIdx.x * 4 + r) * 2654435761u;
    for (int i = 0; i < iters; ++i) {
      const int s = i % S;
      mbar_wait(&empty[r][s], ((i / S) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[r][s], kStageBytes);
      h = h * 1664525u + 1013904223u;
      const int y = (h >> 16) % ymax, z = (h >> 4) % zmax, x = ((h >> 8) % 200) * 32;
      tma_load_2d(base + s * kStageBytes, &ta, &full[r][s], x, y * 128);
      tma_load_3d(base + s * kStageBytes + 8192, &tb, &full[r][s], 0, y * 32, z);
    }
  } else {
    for (int i = 0; i < iters; ++i) {
      const int s = i % S;
      mbar_wait(&full[r][s], (i / S) & 1);
      mbar_arrive(&empty[r][s]);
    }
  }
}

int main() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int W = 8192, H = 2048;      // bf16, 32 MB: L2 resident after the warm-up launch
  uint16_t* d; cudaMalloc(&d, (size_t)W * H * 2); cudaMemset(d, 0, (size_t)W * H * 2);
  CUtensorMap ta{}, tb{};
  {
    cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H}, str[1] = {(cuuint64_t)W * 2};
    cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    encode(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t dims[3] = {32, (cuuint64_t)H, (cuuint64_t)(W / 32)}, str[2] = {(cuuint64_t)W * 2, 64};
    cuuint32_t box[3] = {32, 32, 8}, es[3] = {1, 1, 1};
    encode(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct Case { int grid, R, S; } cases[] = {{148, 1, 4}, {148, 1, 8}, {148, 2, 4}, {148, 4, 2}, {296, 1, 4},
                                             {148, 2, 3}, {296, 2, 2}, {148, 1, 6}, {148, 3, 3}};
  const int iters = 2000;
  for (auto c : cases) {
    const int smem = c.R * c.S * kStageBytes + 1024;
    if (smem > 220 * 1024) continue;
    cudaFuncSetAttribute(rings, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    rings<<<c.grid, 256, smem>>>(ta, tb, c.R, c.S, 50, H / 128 - 1, W / 32 - 8);
    cudaEventRecord(e0);
    rings<<<c.grid, 256, smem>>>(ta, tb, c.R, c.S, iters, H / 128 - 1, W / 32 - 8);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)kStageBytes * iters * c.R * c.grid;
    printf("grid %3d rings/CTA %d stages %d (in flight/CTA %3d KB): %6.2f TB/s (%.0f B/clk/SM @1.965GHz)\n", c.grid, c.R,
           c.S, c.R * c.S * 24, bytes / (ms * 1e-3) / 1e12, bytes / (ms * 1e-3) / 148 / 1.965e9);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
