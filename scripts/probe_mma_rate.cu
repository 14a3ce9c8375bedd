// probe_mma_rate.cu -- tcgen05.mma kind::f16 issue-rate microbenchmark on one B200.
// Every CTA (one per SM) issues R MMAs on zero-filled smem operands into TMEM, then
// commits and waits; cycles per MMA are reported for operand layouts, N and lane masks.
#include <cuda.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2103_13042_b200/csrc/sm100.cuh"

using namespace spamm::sm100;

struct Cfg {
  const char* name;
  uint32_t a_layout, a_lbo, a_sbo, a_kstep;      // A K-major
  uint32_t b_layout, b_lbo, b_sbo, b_kstep;      // B
  uint32_t b_mn_major;
  uint32_t N;
  uint32_t masked;    // disable lanes of quadrants 1 and 3
  uint32_t ksub;      // MMAs per "k-step" cycling over the K sub-blocks
  uint32_t same_acc;  // 1: every MMA accumulates into the same TMEM tile (a dependent chain)
};

__global__ void __launch_bounds__(128, 1) rate_kernel(Cfg c, int R, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 1) tmem_alloc<512>(&tslot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (warp == 0) {
    unsigned long long t0 = 0, t1 = 0;
    if (elect_one()) {
      const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 32 * 1024);
      const uint32_t idesc = idesc_f16(1, 128, c.N, 0, c.b_mn_major);
      const uint32_t m1 = c.masked ? 0xFFFFFFFFu : 0u, m3 = c.masked ? 0xFFFFFFFFu : 0u;
      t0 = clock64();
      for (int r = 0; r < R; ++r) {
        const uint32_t ks = r % c.ksub;
        const uint64_t ad = smem_desc(a0 + ks * c.a_kstep, c.a_lbo, c.a_sbo, c.a_layout);
        const uint64_t bd = smem_desc(b0 + ks * c.b_kstep, c.b_lbo, c.b_sbo, c.b_layout);
        umma_f16(tb + (c.same_acc ? 0u : (r & 1) * 256), ad, bd, idesc, 1u, 0u, m1, 0u, m3);
      }
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      t1 = clock64();
      if (blockIdx.x == 0) { out[0] = t1 - t0; }
      atomicMax(out + 1, t1 - t0);
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tb);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int R = 4096;
  // A: [128 rows][32 k] SW64 K-major: SBO 512, K step 32 B.  A SW128 [128][64]: SBO 1024, K step 32 B.
  // B MN-major SW64 boxes [32 k][32 n]: LBO 2048 (next 32 n), SBO 512 (next 8 k), K step 1024 B.
  // B K-major SW64 [N rows][32 k]: SBO 512, K step 32 B.  B K-major SW128 [N][64 k]: SBO 1024.
  Cfg cfgs[] = {
      {"A-K-SW64 / B-MN-SW64  N=256", kLayoutSW64, 16, 512, 32, kLayoutSW64, 2048, 512, 1024, 1, 256, 0, 2},
      {"A-K-SW64 / B-MN-SW64  N=256 masked", kLayoutSW64, 16, 512, 32, kLayoutSW64, 2048, 512, 1024, 1, 256, 1, 2},
      {"A-K-SW64 / B-MN-SW64  N=128", kLayoutSW64, 16, 512, 32, kLayoutSW64, 2048, 512, 1024, 1, 128, 0, 2},
      {"A-K-SW64 / B-MN-SW64  N=64", kLayoutSW64, 16, 512, 32, kLayoutSW64, 2048, 512, 1024, 1, 64, 0, 2},
      {"A-K-SW64 / B-MN-SW64  N=32", kLayoutSW64, 16, 512, 32, kLayoutSW64, 2048, 512, 1024, 1, 32, 0, 2},
      {"A-K-SW64 / B-K-SW64   N=256", kLayoutSW64, 16, 512, 32, kLayoutSW64, 16, 512, 32, 0, 256, 0, 2},
      {"A-K-SW128/ B-K-SW128  N=256", kLayoutSW128, 16, 1024, 32, kLayoutSW128, 16, 1024, 32, 0, 256, 0, 4},
      {"A-K-SW128/ B-MN-SW128 N=256", kLayoutSW128, 16, 1024, 32, kLayoutSW128, 8192, 1024, 2048, 1, 256, 0, 4},
      {"A-K-SW128/ B-K-SW128  N=128", kLayoutSW128, 16, 1024, 32, kLayoutSW128, 16, 1024, 32, 0, 128, 0, 4},
      {"A-K-SW128/ B-K-SW128  N=64", kLayoutSW128, 16, 1024, 32, kLayoutSW128, 16, 1024, 32, 0, 64, 0, 4},
      {"A-K-SW64 / B-MN-SW64  N=256 same acc", kLayoutSW64, 16, 512, 32, kLayoutSW64, 2048, 512, 1024, 1, 256, 0, 2, 1},
      {"A-K-SW64 / B-MN-SW64  N=128 same acc", kLayoutSW64, 16, 512, 32, kLayoutSW64, 2048, 512, 1024, 1, 128, 0, 2, 1},
      {"A-K-SW64 / B-MN-SW64  N=128 masked same acc", kLayoutSW64, 16, 512, 32, kLayoutSW64, 2048, 512, 1024, 1, 128, 1, 2, 1},
  };
  for (auto& c : cfgs) {
    for (int grid : {1, 148}) {
      cudaMemset(d, 0, 16);
      rate_kernel<<<grid, 128, 100 * 1024>>>(c, R, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s: %s\n", c.name, cudaGetErrorString(e)); return 1; }
      unsigned long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      const double cyc = (double)h[1] / R;
      const double floor = 128.0 * c.N / 256.0;
      printf("%-40s grid=%3d  cycles/MMA=%7.1f  floor=%6.1f  eff=%5.2f\n", c.name, grid, cyc, floor, floor / cyc);
    }
  }
  return 0;
}
