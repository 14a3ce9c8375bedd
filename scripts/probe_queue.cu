// probe_queue.cu -- does a single thread block when issuing tcgen05.mma back to back?
// Issue R MMAs (N=256, 128 cycles each) and record the clock after each issue.
#include <cstdio>
#include <cstdint>
#include "../paper_2103_13042_b200/csrc/sm100.cuh"
using namespace spamm::sm100;

__global__ void qk(unsigned long long* out, int R, int gap) {
  extern __shared__ uint8_t zraw[];
  uint8_t* z = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(zraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t ts;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(z)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x / 32 == 1) tmem_alloc<256>(&ts);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) {
    const uint64_t ad = smem_desc(smem_u32(z), 16, 512, kLayoutSW64);
    const uint64_t bd = smem_desc(smem_u32(z + 8192), 2048, 512, kLayoutSW64);
    const uint32_t idesc = idesc_f16(1, 128, 256, 0, 1);
    unsigned long long t0 = clock64();
    uint32_t x = 1;
    for (int r = 0; r < R; ++r) {
      umma_f16(ts, ad, bd, idesc, 1u, 0, 0, 0, 0);
      for (int g = 0; g < gap; ++g) x = x * 1664525u + 1013904223u;   // dependent ALU chain
      out[r] = clock64() - t0;
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[R] = clock64() - t0;
    out[R + 1] = x;
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x / 32 == 1) tmem_dealloc<256>(ts);
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 200);
  cudaFuncSetAttribute(qk, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int gap : {0, 20, 50, 100}) {
    const int R = 64;
    qk<<<1, 64, 40000>>>(d, R, gap);
    cudaDeviceSynchronize();
    unsigned long long h[200];
    cudaMemcpy(h, d, 8 * (R + 2), cudaMemcpyDeviceToHost);
    printf("gap=%3d: issue clocks after MMA #1..#8: ", gap);
    for (int r = 0; r < 8; ++r) printf("%llu ", h[r]);
    printf(" ... #32: %llu #64: %llu  total(with drain): %llu  (%.1f cyc/MMA)\n", h[31], h[63], h[R], (double)h[R] / R);
  }
  return 0;
}
