// probe_ffma.cu -- measured FP32 CUDA-core (FFMA) peak of this B200, the denominator of the
// FP32 SIMT multiply's roofline (bench.py reads profiles/ffma_peak.json).
// Every thread runs 16 independent FFMA chains (enough ILP to cover the 4-cycle FMA latency
// with 4 warps per SM sub-partition); grid = 148 SMs x 4 CTAs x 512 threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_ffma probe_ffma.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) ffma_kernel(float* out, int iters, float a, float b) {
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678f) out[blockIdx.x] = s;   // keep the chains alive
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4096 * sizeof(float));
  const int blocks = sms * 4, threads = 512, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  ffma_kernel<<<blocks, threads>>>(out, iters, 0.999999f, 1e-7f);   // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 10; ++rep) {
    cudaEventRecord(e0);
    ffma_kernel<<<blocks, threads>>>(out, iters, 0.999999f, 1e-7f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * blocks * threads * (double)iters * 8 * 16;
  const double tf = flops / (best * 1e-3) / 1e12;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"tflops\": %.2f, \"ms\": %.3f, \"sms\": %d, \"how\": \"scripts/probe_ffma.cu: %d CTAs x %d threads x %d x 128 "
         "independent FFMA, best of 10, CUDA events\"}\n", tf, best, sms, blocks, threads, iters);
  return cudaGetLastError() != cudaSuccess;
}
