// probe_tma_bw.cu -- L2 -> SMEM TMA load throughput by box shape (inner row bytes),
// 2 CTAs/SM, 4-stage ring, the consumer only releases stages (no math).  Source: a 32 MB
// bf16 matrix (L2 resident after the first pass).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include "../paper_2103_13042_b200/csrc/sm100.cuh"
using namespace spamm::sm100;

constexpr int kStages = 4, kStageBytes = 24576;

struct Cfg { int dims; int bx, by, bz; int bytes; };

__global__ void bw(const __grid_constant__ CUtensorMap t, const __grid_constant__ CUtensorMap t2, int nl, int bytes,
                   int use2, int R, int xmax, int ymax, int zmax, int xstep) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kStages], empty[kStages];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t h = blockIdx.x * 2654435761u;
    for (int r = 0; r < R; ++r) {
      const int s = r % kStages;
      mbar_wait(&empty[s], ((r / kStages) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], bytes * nl + (use2 ? 16384 : 0));
      h = h * 1664525u + 1013904223u;
      const int x = ((h >> 8) % xmax) * xstep, y = (h >> 16) % ymax, z = (h >> 4) % zmax;
      for (int l = 0; l < nl; ++l) {
        if (zmax > 0 && t.opaque[0] == t.opaque[0] && bytes == 16384 && use2 < 0) {}
        if (zmax > 1) tma_load_3d(sm + s * kStageBytes + l * bytes, &t, &full[s], 0, y * 32, z);
        else tma_load_2d(sm + s * kStageBytes + l * bytes, &t, &full[s], x + l * 64, y * 32);
      }
      if (use2) tma_load_3d(sm + s * kStageBytes + 8192, &t2, &full[s], 0, y * 32, (h >> 3) % 248);
    }
  } else if (threadIdx.x == 32) {
    for (int r = 0; r < R; ++r) {
      const int s = r % kStages;
      mbar_wait(&full[s], (r / kStages) & 1);
      mbar_arrive(&empty[s]);
    }
  }
}

int main() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int W = 8192, H = 2048;      // bf16, 32 MB
  uint16_t* d; cudaMalloc(&d, (size_t)W * H * 2); cudaMemset(d, 0, (size_t)W * H * 2);
  cudaFuncSetAttribute(bw, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kStageBytes + 2048);
  auto enc2 = [&](CUtensorMap* m, int bx, int by, CUtensorMapSwizzle sw, CUtensorMapL2promotion pr) {
    cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H}, str[1] = {(cuuint64_t)W * 2};
    cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by}, es[2] = {1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, pr,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  auto enc3 = [&](CUtensorMap* m, int kb, int nb, CUtensorMapL2promotion pr) {
    cuuint64_t dims[3] = {32, (cuuint64_t)H, (cuuint64_t)(W / 32)}, str[2] = {(cuuint64_t)W * 2, 64};
    cuuint32_t box[3] = {32, (cuuint32_t)kb, (cuuint32_t)nb}, es[3] = {1, 1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_64B, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int R = 2000;
  for (int grid : {148, 296}) {
    for (auto pr : {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B}) {
      CUtensorMap t{}, t2{};
      struct Case { const char* name; int kind; } cases[] = {
        {"A 2D {32 el=64B,128 rows} SW64 8KB", 0}, {"A 2D {64 el=128B,128 rows} SW128 16KB", 1},
        {"A 2D {128 el=256B,64 rows} none 16KB", 2}, {"B 3D {32,32,8} SW64 16KB (64B rows)", 3},
        {"A 8KB + B 3D 16KB (narrow entry)", 4}, {"2D {64 el,64 rows} SW128 x2 16KB", 5}};
      for (auto& c : cases) {
        int nl = 1, bytes = 0, use2 = 0, zmax = 1, xmax = W / 64 - 2, ymax = H / 32 - 8, xstep = 64;
        if (c.kind == 0) { enc2(&t, 32, 128, CU_TENSOR_MAP_SWIZZLE_64B, pr); bytes = 8192; nl = 2; }
        if (c.kind == 1) { enc2(&t, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B, pr); bytes = 16384; }
        if (c.kind == 2) { enc2(&t, 128, 64, CU_TENSOR_MAP_SWIZZLE_NONE, pr); bytes = 16384; xstep = 128; xmax = W / 128 - 1; ymax = H / 32 - 4; }
        if (c.kind == 3) { enc3(&t, 32, 8, pr); bytes = 16384; zmax = W / 32 - 8; }
        if (c.kind == 4) { enc2(&t, 32, 128, CU_TENSOR_MAP_SWIZZLE_64B, pr); enc3(&t2, 32, 8, pr); bytes = 8192; use2 = 1; }
        if (c.kind == 5) { enc2(&t, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B, pr); bytes = 8192; nl = 2; ymax = H / 32 - 4; }
        const int tot = bytes * nl + (use2 ? 16384 : 0);
        bw<<<grid, 64, kStages * kStageBytes + 2048>>>(t, t2, nl, bytes, use2, 50, xmax, ymax, zmax, xstep);
        cudaEventRecord(e0);
        bw<<<grid, 64, kStages * kStageBytes + 2048>>>(t, t2, nl, bytes, use2, R, xmax, ymax, zmax, xstep);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("grid %3d promo %d  %-40s %6.2f TB/s  (%.0f B/clk/SM @1.965GHz)\n", grid, (int)pr, c.name,
               (double)tot * R * grid / (ms * 1e-3) / 1e12, (double)tot * R * grid / (ms * 1e-3) / 148 / 1.965e9);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
