// probe_queue3.cu -- single issuing thread: is the per-MMA blocking caused by the
// accumulator dependency?  R MMAs, `gap` dependent IMADs between issues, D alternating
// over `nacc` different TMEM column ranges (N columns each).
#include <cstdio>
#include <cstdint>
#include "../paper_2103_13042_b200/csrc/sm100.cuh"
using namespace spamm::sm100;

__global__ void qk(unsigned long long* out, int R, int gap, int nacc, int N) {
  extern __shared__ uint8_t zraw[];
  uint8_t* z = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(zraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t ts;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(z)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x / 32 == 0) tmem_alloc<512>(&ts);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) {
    const uint64_t ad = smem_desc(smem_u32(z), 16, 512, kLayoutSW64);
    const uint64_t bd = smem_desc(smem_u32(z + 8192), 2048, 512, kLayoutSW64);
    const uint32_t idesc = idesc_f16(1, 128, N, 0, 1);
    uint32_t x = 1;
    const unsigned long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
      umma_f16(ts + (r % nacc) * N, ad, bd, idesc, 1u, 0, 0, 0, 0);
      for (int g = 0; g < gap; ++g) x = x * 1664525u + 1013904223u;
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[0] = clock64() - t0 + (x == 12345u);
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x / 32 == 0) tmem_dealloc<512>(ts);
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(qk, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  const int R = 256;
  for (int N : {256, 128})
    for (int nacc : {1, 2})
      for (int gap : {0, 10, 30}) {
        if (nacc * N > 512) continue;
        qk<<<1, 64, 40000>>>(d, R, gap, nacc, N);
        cudaDeviceSynchronize();
        unsigned long long h;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("N=%d accumulators=%d gap=%2d: %.1f cyc/MMA (pipe floor %d)\n", N, nacc, gap, (double)h / R, N / 2);
      }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
