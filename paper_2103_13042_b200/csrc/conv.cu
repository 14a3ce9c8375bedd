// conv.cu -- SpAMM convolution drop-in (Sec. 4.3.2): a convolution layer as the
// GEMM Y = W * im2col(X) whose product is the SpAMM of the plan.
//
// The paper applies cuSpAMM to the im2col GEMMs of VGG13 (128 x 576 x 25600 and
// 256 x 1152 x 6400), with weight pruning and ReLU making both operands near-sparse.  Here the
// im2col matrix is formed on the device by one coalesced kernel into plan-owned storage (HBM-bound:
// one write of K x N elements, reads of X mostly from L2), then the plan's three stages run with
// A = W, B = im2col(X), C = Y.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "internal.h"

namespace spamm {
namespace {

// B[r][c], r = (ci*kh + ky)*kw + kx, c = (n*Ho + y)*Wo + x  =  X[n][ci][y*s - pad + ky][x*s - pad + kx]
// (0 outside the image).  One thread per 8 consecutive columns of one row: 16-byte (bf16/fp16) or
// 32-byte (float) stores.
template <typename T>
__global__ void __launch_bounds__(256)
    im2col_kernel(const T* __restrict__ X, int64_t batch, int64_t C_in, int64_t H, int64_t W, int kh, int kw,
                  int stride, int pad, int64_t Ho, int64_t Wo, T* __restrict__ B, int64_t ldb) {
  const int64_t N = batch * Ho * Wo;
  const int64_t groups = (N + 7) / 8;
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t r = blockIdx.y + static_cast<int64_t>(blockIdx.z) * gridDim.y;
  if (gid >= groups || r >= C_in * kh * kw) return;
  const int kx = static_cast<int>(r % kw), ky = static_cast<int>((r / kw) % kh);
  const int64_t ci = r / (static_cast<int64_t>(kh) * kw);
  T v[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int64_t c = gid * 8 + e;
    v[e] = T(0.f);
    if (c < N) {
      const int64_t x = c % Wo, y = (c / Wo) % Ho, n = c / (Wo * Ho);
      const int64_t iy = y * stride - pad + ky, ix = x * stride - pad + kx;
      if (iy >= 0 && iy < H && ix >= 0 && ix < W) v[e] = X[((n * C_in + ci) * H + iy) * W + ix];
    }
  }
  T* dst = B + r * ldb + gid * 8;   // ldb is a multiple of 8: whole vector stores (padding columns = 0)
  if constexpr (sizeof(T) == 2) {
    *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(v);
  } else {
    reinterpret_cast<uint4*>(dst)[0] = reinterpret_cast<const uint4*>(v)[0];
    reinterpret_cast<uint4*>(dst)[1] = reinterpret_cast<const uint4*>(v)[1];
  }
}

}  // namespace
}  // namespace spamm

using namespace spamm;

extern "C" spamm_status spamm_conv2d_im2col(spamm_plan_t h, const void* W, int64_t ldw, const void* X, int64_t batch,
                                           int64_t C_in, int64_t H, int64_t Wd, int32_t kh, int32_t kw,
                                           int32_t stride, int32_t pad, float* Y, int64_t ldy, void* stream) {
  if (!h || !W || !X || !Y) return fail(SPAMM_E_INVALID, "NULL argument");
  Plan& p = *reinterpret_cast<Plan*>(h);
  if (batch <= 0 || C_in <= 0 || H <= 0 || Wd <= 0 || kh <= 0 || kw <= 0 || stride <= 0 || pad < 0)
    return fail(SPAMM_E_INVALID, "bad convolution geometry");
  const int64_t Ho = (H + 2 * pad - kh) / stride + 1, Wo = (Wd + 2 * pad - kw) / stride + 1;
  if (Ho <= 0 || Wo <= 0) return fail(SPAMM_E_INVALID, "empty convolution output");
  const int64_t K = C_in * kh * kw, N = batch * Ho * Wo;
  if (p.K != K || p.N != N)
    return fail(SPAMM_E_INVALID, "plan shape must be M = C_out, K = C_in*kh*kw, N = batch*Ho*Wo (got K = " +
                                     std::to_string(p.K) + ", N = " + std::to_string(p.N) + ")");
  const size_t es = f32_inputs(p.prec) ? 4 : 2;
  SPAMM_TRY(check_matrix(X, 1, 1, 8, es, "X"));
  const int64_t ldb = (N + 7) / 8 * 8;
  if (!p.im2col) {
    if (cudaMalloc(&p.im2col, es * static_cast<size_t>(K * ldb)) != cudaSuccess) {
      cudaGetLastError();
      return fail(SPAMM_E_NOMEM, "im2col storage");
    }
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t groups = (ldb + 7) / 8;
  const int64_t gy = std::min<int64_t>(K, 65535), gz = (K + gy - 1) / gy;
  const dim3 grid(static_cast<unsigned>((groups + 255) / 256), static_cast<unsigned>(gy), static_cast<unsigned>(gz));
  if (es == 4)
    im2col_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(X), batch, C_in, H, Wd, kh, kw, stride, pad, Ho,
                                               Wo, static_cast<float*>(p.im2col), ldb);
  else
    im2col_kernel<__half><<<grid, 256, 0, s>>>(static_cast<const __half*>(X), batch, C_in, H, Wd, kh, kw, stride, pad,
                                                Ho, Wo, static_cast<__half*>(p.im2col), ldb);   // 16-bit moves only
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  return spamm_run(h, W, ldw, p.im2col, ldb, Y, ldy, stream);
}
