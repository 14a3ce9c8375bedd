// norms.cu -- stage 1: tile Frobenius norms (Eq. 2; get-norm kernel Sec. 3.2,
// PAPER.md:105-123).
//
// B200 design (not the paper's one-block-per-tile reduction): the matrix is read
// exactly once, fully coalesced, with 16-byte streaming loads; a CTA covers one
// 32-row tile strip and a chunk of columns.  Each lane owns 16 B of a row (4 FP32
// or 8 BF16/FP16 values), accumulates x*x in float64 over its 4 rows, the lanes of
// one tile combine with an xor-shuffle butterfly and the 8 warps combine in smem
// in warp order.  The operation sequence per tile does not depend on the tile's
// position, so equal tiles give bit-identical norms (Toeplitz inputs).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "internal.h"

namespace spamm {
namespace {

constexpr int kWarps = 8;         // rows w, w+8, w+16, w+24 of the strip
constexpr int kGroups = 8;        // 32*V-column groups per CTA

template <typename T>
__device__ __forceinline__ double sq_sum_vec(const T* p, int n_valid);

template <>
__device__ __forceinline__ double sq_sum_vec<float>(const float* p, int n_valid) {
  double s = 0.0;
  if (n_valid >= 4) {
    float4 v = __ldcs(reinterpret_cast<const float4*>(p));
    s = fma((double)v.x, (double)v.x, s);
    s = fma((double)v.y, (double)v.y, s);
    s = fma((double)v.z, (double)v.z, s);
    s = fma((double)v.w, (double)v.w, s);
  } else {
    for (int e = 0; e < 4; ++e) {
      double x = e < n_valid ? (double)p[e] : 0.0;
      s = fma(x, x, s);
    }
  }
  return s;
}

template <typename H>
__device__ __forceinline__ double to_d(H h);
template <>
__device__ __forceinline__ double to_d<__nv_bfloat16>(__nv_bfloat16 h) { return (double)__bfloat162float(h); }
template <>
__device__ __forceinline__ double to_d<__half>(__half h) { return (double)__half2float(h); }

template <typename H>
__device__ __forceinline__ double sq_sum_vec16(const H* p, int n_valid) {
  double s = 0.0;
  if (n_valid >= 8) {
    int4 raw = __ldcs(reinterpret_cast<const int4*>(p));
    const H* h = reinterpret_cast<const H*>(&raw);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      double x = to_d<H>(h[e]);
      s = fma(x, x, s);
    }
  } else {
    for (int e = 0; e < 8; ++e) {
      double x = e < n_valid ? to_d<H>(p[e]) : 0.0;
      s = fma(x, x, s);
    }
  }
  return s;
}
template <>
__device__ __forceinline__ double sq_sum_vec<__nv_bfloat16>(const __nv_bfloat16* p, int n_valid) {
  return sq_sum_vec16<__nv_bfloat16>(p, n_valid);
}
template <>
__device__ __forceinline__ double sq_sum_vec<__half>(const __half* p, int n_valid) {
  return sq_sum_vec16<__half>(p, n_valid);
}

// grid = (ceil(cols / (kGroups*32*V)), tile rows); block = 256.
template <typename T>
__global__ void __launch_bounds__(kWarps * 32) tile_norms_kernel(const T* __restrict__ X, int64_t rows,
                                                                  int64_t cols, int64_t ld,
                                                                  double* __restrict__ out, int64_t out_rs,
                                                                  int64_t out_cs, int64_t tile_row0) {
  constexpr int V = 16 / sizeof(T);   // elements per lane-load
  constexpr int LPT = kTile / V;      // lanes per tile
  constexpr int TPG = 32 / LPT;       // tiles per warp group (= V)
  __shared__ double part[kWarps][kGroups * TPG];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t it = tile_row0 + blockIdx.y;
  const int64_t col_base = static_cast<int64_t>(blockIdx.x) * kGroups * 32 * V;
  const int64_t row0 = it * kTile + warp;

#pragma unroll 2
  for (int g = 0; g < kGroups; ++g) {
    const int64_t c = col_base + static_cast<int64_t>(g) * 32 * V + lane * V;
    double s = 0.0;
    const int64_t nv64 = cols - c;
    const int nv = nv64 <= 0 ? 0 : (nv64 >= V ? V : static_cast<int>(nv64));
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t row = row0 + 8 * r;
      if (row < rows && nv > 0) s += sq_sum_vec<T>(X + row * ld + c, nv);
    }
    // combine the LPT lanes of each tile (butterfly; order independent of tile position)
#pragma unroll
    for (int o = LPT / 2; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((lane % LPT) == 0) part[warp][g * TPG + lane / LPT] = s;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < kGroups * TPG; t += blockDim.x) {
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) tot += part[w][t];
    const int64_t kt = (col_base / kTile) + t;
    if (kt * kTile < cols) out[it * out_rs + kt * out_cs] = sqrt(tot);
  }
}

template <typename T>
spamm_status launch_t(const void* X, int64_t rows, int64_t cols, int64_t ld, double* out, int64_t out_rs,
                      int64_t out_cs, int64_t r0, int64_t r1, cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  const int64_t per_block = static_cast<int64_t>(kGroups) * 32 * V;
  const int64_t gx = (cols + per_block - 1) / per_block;
  const int64_t gy = r1 - r0;
  if (gx <= 0 || gy <= 0) return SPAMM_OK;
  if (gy > 65535) {
    // chunk the tile rows over several launches (grid.y limit)
    for (int64_t a = r0; a < r1; a += 65535) {
      SPAMM_TRY(launch_t<T>(X, rows, cols, ld, out, out_rs, out_cs, a, a + 65535 < r1 ? a + 65535 : r1, s));
    }
    return SPAMM_OK;
  }
  dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
  tile_norms_kernel<T><<<grid, kWarps * 32, 0, s>>>(static_cast<const T*>(X), rows, cols, ld, out, out_rs,
                                                    out_cs, r0);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

}  // namespace

spamm_status launch_norms(const Plan& p, const void* X, int64_t rows, int64_t cols, int64_t ld, double* out,
                          int64_t out_rs, int64_t out_cs, int64_t r0, int64_t r1, cudaStream_t s) {
  switch (p.prec) {
    case SPAMM_FP32: return launch_t<float>(X, rows, cols, ld, out, out_rs, out_cs, r0, r1, s);
    case SPAMM_BF16: return launch_t<__nv_bfloat16>(X, rows, cols, ld, out, out_rs, out_cs, r0, r1, s);
    case SPAMM_FP16: return launch_t<__half>(X, rows, cols, ld, out, out_rs, out_cs, r0, r1, s);
  }
  return fail(SPAMM_E_UNSUPPORTED, "precision");
}

}  // namespace spamm
