// probe_queue2.cu -- can several warps of one CTA (or several CTAs of one SM) keep the
// tensor pipe busy while each issuing thread does ALU work between its MMAs?
// W issuing warps, each R MMAs (N=256, 128 cycles) into its own TMEM columns, gap ALU ops
// between consecutive MMAs.  Reports cycles per MMA over all warps.
#include <cstdio>
#include <cstdint>
#include "../paper_2103_13042_b200/csrc/sm100.cuh"
using namespace spamm::sm100;

__global__ void qk(unsigned long long* out, int R, int gap, int W, int N) {
  extern __shared__ uint8_t zraw[];
  uint8_t* z = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(zraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[4];
  __shared__ uint32_t ts;
  __shared__ unsigned long long tt[8];
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(z)[i] = 0;
  if (threadIdx.x == 0) { for (int w = 0; w < 4; ++w) mbar_init(&bar[w], 1); fence_mbar_init(); }
  if (threadIdx.x / 32 == 0) tmem_alloc<512>(&ts);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const int warp = threadIdx.x / 32;
  unsigned long long t0 = clock64();
  if (warp < W && (threadIdx.x & 31) == 0) {
    const uint64_t ad = smem_desc(smem_u32(z), 16, 512, kLayoutSW64);
    const uint64_t bd = smem_desc(smem_u32(z + 8192), 2048, 512, kLayoutSW64);
    const uint32_t idesc = idesc_f16(1, 128, N, 0, 1);
    uint32_t x = 1;
    const uint32_t col = ts + (warp * 128) % 512;
    for (int r = 0; r < R; ++r) {
      umma_f16(col, ad, bd, idesc, 1u, 0, 0, 0, 0);
      for (int g = 0; g < gap; ++g) x = x * 1664525u + 1013904223u;   // dependent ALU chain
    }
    umma_commit(&bar[warp]);
    mbar_wait(&bar[warp], 0);
    tt[warp] = clock64() - t0 + (x == 12345u);
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long m = 0;
    for (int w = 0; w < W; ++w) m = tt[w] > m ? tt[w] : m;
    out[blockIdx.x] = m;
  }
  if (threadIdx.x / 32 == 0) tmem_dealloc<512>(ts);
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 200);
  cudaFuncSetAttribute(qk, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  const int R = 256;
  for (int N : {256, 128})
  for (int W : {1, 2, 4})
    for (int gap : {0, 10, 30, 60}) {
      qk<<<1, 128, 40000>>>(d, R, gap, W, N);
      cudaDeviceSynchronize();
      unsigned long long h;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("N=%d warps=%d gap=%3d: %.1f cyc/MMA (all warps; pipe floor %d)\n", N, W, gap, (double)h / (R * W), N / 2);
    }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
