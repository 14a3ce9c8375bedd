// probe_sync.cu -- latency of mbarrier handshakes and tcgen05.commit arrivals on B200.
#include <cstdio>
#include <cstdint>
#include "../paper_2103_13042_b200/csrc/sm100.cuh"
using namespace spamm::sm100;

__global__ void sync_kernel(unsigned long long* out, int iters) {
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  extern __shared__ uint8_t zraw[];
  uint8_t* zbuf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(zraw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(zbuf)[i] = 0;
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  if (warp == 1) tmem_alloc<256>(&tslot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tb = tslot;
  // (1) commit with nothing pending -> wait, same thread
  if (warp == 0 && lane == 0) {
    uint32_t ph = 0;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { umma_commit(&bar[0]); mbar_wait(&bar[0], ph); ph ^= 1; }
    out[0] = (clock64() - t0) / iters;
    // (3) one N=256 MMA then commit -> wait
    const uint64_t ad = smem_desc(smem_u32(zbuf), 16, 512, kLayoutSW64);
    const uint64_t bd = smem_desc(smem_u32(zbuf + 8192), 2048, 512, kLayoutSW64);
    const uint32_t idesc = idesc_f16(1, 128, 256, 0, 1);
    uint32_t ph3 = 0;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { umma_f16(tb, ad, bd, idesc, 1u, 0, 0, 0, 0); umma_commit(&bar[3]); mbar_wait(&bar[3], ph3); ph3 ^= 1; }
    out[2] = (clock64() - t0) / iters;
  }
  __syncthreads();
  // (2) ping-pong between warp 0 lane 0 and warp 2 lane 0 via mbarrier arrive / wait
  if (lane == 0 && (warp == 0 || warp == 2)) {
    uint32_t ph = 0;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (warp == 0) { mbar_arrive(&bar[1]); mbar_wait(&bar[2], ph); }
      else { mbar_wait(&bar[1], ph); mbar_arrive(&bar[2]); }
      ph ^= 1;
    }
    if (warp == 0) out[1] = (clock64() - t0) / iters;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 1) tmem_dealloc<256>(tb);
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(sync_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  sync_kernel<<<1, 128, 40000>>>(d, 1000);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[4];
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("cuda=%s  commit(no MMA)->wait: %llu cyc   arrive/wait ping-pong round trip: %llu cyc   MMA(N=256)+commit->wait: %llu cyc\n",
         cudaGetErrorString(e), h[0], h[1], h[2]);
  sync_kernel<<<148, 128, 40000>>>(d, 1000);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("148 CTAs: commit->wait %llu  ping-pong %llu  MMA+commit %llu\n", h[0], h[1], h[2]);
  return 0;
}
