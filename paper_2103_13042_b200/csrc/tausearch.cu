// tausearch.cu -- the Sec. 3.5.2 tau search on the device norm maps.
//
// The paper picks tau for a target valid ratio by binary search: start at ave = the mean of
// the norm products of all sub-matrix pairs, search [0, k*ave] and grow k while the upper end
// still keeps too many pairs; stop when |vr - target| < 1 % (readings R16, R17).
// Every evaluation of vr(tau) is a count of kept triples (i,k,j), i.e. the skip-map predicate
// !(nA[i,k] * nB[k,j] < tau) in float64 (reading R2) over all BM*BK*BN triples, done here by a
// brute-force tiled kernel without writing any list.  The control flow of the search is the
// paper's scalar loop and stays on the host (one synchronisation per evaluation).
#include <algorithm>
#include <cmath>

#include "internal.h"

namespace spamm {
namespace {

constexpr int kCI = 64, kCJ = 64, kCK = 32, kCountThreads = 256;

// Count !(nA[i,k] * nBt[j,k] < tau) over a 64 (i) x 64 (j) block of C tiles, all k.
// Thread (ty, tx) of a 16 x 16 layout owns i = i0 + ty + 16 r, j = j0 + tx + 16 c (r, c < 4).
__global__ void __launch_bounds__(kCountThreads)
    count_kept_kernel(const double* __restrict__ nA, const double* __restrict__ nBt, int64_t BM, int64_t BK,
                      int64_t BN, double tau, unsigned long long* __restrict__ out) {
  __shared__ double sa[kCK][kCI + 1];
  __shared__ double sb[kCK][kCJ + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t i0 = static_cast<int64_t>(blockIdx.y) * kCI, j0 = static_cast<int64_t>(blockIdx.x) * kCJ;
  unsigned int cnt = 0, valid = 0;   // bit 4r+c: (i, j) inside [0,BM) x [0,BN)
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (i0 + ty + 16 * r < BM && j0 + tx + 16 * c < BN) valid |= 1u << (4 * r + c);
  for (int64_t k0 = 0; k0 < BK; k0 += kCK) {
    const int kn = static_cast<int>(BK - k0 < kCK ? BK - k0 : kCK);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < (kCI * kCK) / kCountThreads; ++q) {
      const int idx = threadIdx.x + q * kCountThreads;
      const int r = idx / kCK, kk = idx % kCK;
      const int64_t i = i0 + r, j = j0 + r;
      sa[kk][r] = (i < BM && kk < kn) ? nA[i * BK + k0 + kk] : 0.0;
      sb[kk][r] = (j < BN && kk < kn) ? nBt[j * BK + k0 + kk] : 0.0;
    }
    __syncthreads();
    for (int kk = 0; kk < kn; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = sa[kk][ty + 16 * r];
#pragma unroll
      for (int c = 0; c < 4; ++c) b[c] = sb[kk][tx + 16 * c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) cnt += ((valid >> (4 * r + c)) & 1u) & !(__dmul_rn(a[r], b[c]) < tau);
    }
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, static_cast<unsigned long long>(cnt));
}

// Column sums over i of nA (sA[k] = sum_i nA[i,k]) and over j of nBt (sB[k] = sum_j nB[k,j]),
// in fixed order per chunk of 64 rows: part[(chunk * 2 + which) * BK + k].
__global__ void colsum_kernel(const double* __restrict__ nA, const double* __restrict__ nBt, int64_t BM,
                              int64_t BK, int64_t BN, double* __restrict__ part) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= BK) return;
  const int which = blockIdx.z;
  const double* src = which == 0 ? nA : nBt;
  const int64_t rows = which == 0 ? BM : BN;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 64, r1 = rows < r0 + 64 ? rows : r0 + 64;
  if (r0 >= rows) return;   // the scratch is zeroed; chunks past this map's rows stay 0
  double s = 0.0;
  for (int64_t r = r0; r < r1; ++r) s += src[r * BK + k];
  part[(static_cast<int64_t>(blockIdx.y) * 2 + which) * BK + k] = s;
}

// ave = sum_k sA[k] * sB[k] / (BM * BK * BN), one block, fixed reduction order.
__global__ void __launch_bounds__(1024) ave_kernel(const double* __restrict__ part, int64_t nchunkA,
                                                  int64_t nchunkB, int64_t BK, double denom,
                                                  double* __restrict__ out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int64_t k = threadIdx.x; k < BK; k += blockDim.x) {
    double sa = 0.0, sb = 0.0;
    for (int64_t c = 0; c < nchunkA; ++c) sa += part[(c * 2 + 0) * BK + k];
    for (int64_t c = 0; c < nchunkB; ++c) sb += part[(c * 2 + 1) * BK + k];
    s += sa * sb;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (static_cast<int>(threadIdx.x) < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0] / denom;
}

// plan-owned scratch of the search (allocated on the first search, reused afterwards)
spamm_status ensure_scratch(Plan& p, int64_t nch) {
  if (!p.ts_cnt) SPAMM_CUDA_TRY(cudaMalloc(&p.ts_cnt, sizeof(unsigned long long)));
  if (nch > 0 && !p.ts_part)
    SPAMM_CUDA_TRY(cudaMalloc(&p.ts_part, sizeof(double) * static_cast<size_t>(nch * 2 * p.BK + 1)));
  return SPAMM_OK;
}

spamm_status count_on(const Plan& p, double tau, unsigned long long* d_cnt, cudaStream_t s, int64_t* kept) {
  SPAMM_CUDA_TRY(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), s));
  const dim3 grid(static_cast<unsigned>((p.BN + kCJ - 1) / kCJ), static_cast<unsigned>((p.BM + kCI - 1) / kCI));
  count_kept_kernel<<<grid, kCountThreads, 0, s>>>(p.nA, p.nBt, p.BM, p.BK, p.BN, tau, d_cnt);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  unsigned long long h = 0;
  SPAMM_CUDA_TRY(cudaMemcpyAsync(&h, d_cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
  SPAMM_CUDA_TRY(cudaStreamSynchronize(s));
  *kept = static_cast<int64_t>(h);
  return SPAMM_OK;
}

}  // namespace
}  // namespace spamm

using namespace spamm;

extern "C" {

spamm_status spamm_count_kept(spamm_plan_t h, double tau, int64_t* kept, void* stream) {
  if (!h || !kept) return fail(SPAMM_E_INVALID, "plan or output is NULL");
  if (!(std::isfinite(tau) && tau >= 0.0)) return fail(SPAMM_E_INVALID, "tau must be finite and >= 0");
  Plan& p = *reinterpret_cast<Plan*>(h);
  if (!p.norms_ready) return fail(SPAMM_E_STATE, "spamm_count_kept before spamm_norms");
  SPAMM_TRY(ensure_scratch(p, 0));
  p.last_stream = static_cast<cudaStream_t>(stream);
  return count_on(p, tau, p.ts_cnt, static_cast<cudaStream_t>(stream), kept);
}

spamm_status spamm_tau_search(spamm_plan_t h, double target, double tol, int32_t max_iter, double* tau_out,
                              double* vr_out, int32_t* iters_out, void* stream) {
  if (!h || !tau_out) return fail(SPAMM_E_INVALID, "plan or tau output is NULL");
  if (!(target >= 0.0 && target <= 1.0) || !(tol > 0.0) || max_iter < 1)
    return fail(SPAMM_E_INVALID, "need 0 <= target <= 1, tol > 0, max_iter >= 1");
  Plan& p = *reinterpret_cast<Plan*>(h);
  if (!p.norms_ready) return fail(SPAMM_E_STATE, "spamm_tau_search before spamm_norms");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t nchA = (p.BM + 63) / 64, nchB = (p.BN + 63) / 64, nch = std::max(nchA, nchB);
  SPAMM_TRY(ensure_scratch(p, nch));
  struct {
    unsigned long long* cnt;
    double* part;
  } w{p.ts_cnt, p.ts_part};
  SPAMM_CUDA_TRY(cudaMemsetAsync(w.part, 0, sizeof(double) * static_cast<size_t>(nch * 2 * p.BK + 1), s));
  // ave: mean norm product over all BM*BK*BN triples (reading R17) = sum_k sA[k] sB[k] / triples
  colsum_kernel<<<dim3(static_cast<unsigned>((p.BK + 127) / 128), static_cast<unsigned>(nch), 2), 128, 0, s>>>(
      p.nA, p.nBt, p.BM, p.BK, p.BN, w.part);
  const double triples = static_cast<double>(p.BM) * static_cast<double>(p.BK) * static_cast<double>(p.BN);
  double* d_ave = w.part + nch * 2 * p.BK;
  ave_kernel<<<1, 1024, 0, s>>>(w.part, nchA, nchB, p.BK, triples, d_ave);
  count_launch(2);
  SPAMM_CUDA_TRY(cudaGetLastError());
  double ave = 0.0;
  SPAMM_CUDA_TRY(cudaMemcpyAsync(&ave, d_ave, sizeof(double), cudaMemcpyDeviceToHost, s));
  SPAMM_CUDA_TRY(cudaStreamSynchronize(s));
  p.last_stream = s;
  // all-zero maps (e.g. a chain converged to 0) or non-finite norms: the search's bracket
  // [0, k*ave] is undefined
  if (!(std::isfinite(ave) && ave > 0.0))
    return fail(SPAMM_E_INVALID, "tau search needs finite norms with a positive mean product (ave = " +
                                     std::to_string(ave) + ")");

  auto vr_at = [&](double t, double* vr) -> spamm_status {
    int64_t kept = 0;
    SPAMM_TRY(count_on(p, t, w.cnt, s, &kept));
    *vr = static_cast<double>(kept) / triples;
    return SPAMM_OK;
  };
  // Sec. 3.5.2: tau = ave, bracket [0, k*ave], k = 1; bisection until |vr - target| < tol
  double tau = ave, lo = 0.0, hi = ave, vr = 0.0;
  int k = 1, it = 1;
  SPAMM_TRY(vr_at(tau, &vr));
  while (it < max_iter && !(std::fabs(vr - target) < tol)) {
    if (vr > target) {
      lo = tau;
      double vh = 0.0;
      SPAMM_TRY(vr_at(hi, &vh));
      // Sec. 3.5.2 grows k by one; after 64 steps k doubles so that the bracket reaches the largest
      // product (where vr = 0 <= target) in a bounded number of evaluations on heavy-tailed maps
      int widen = 0;
      while (vh > target) {
        k = widen < 64 ? k + 1 : 2 * k;
        ++widen;
        if (k > (1 << 30)) return fail(SPAMM_E_INVALID, "tau search bracket did not converge");
        hi = k * ave;
        SPAMM_TRY(vr_at(hi, &vh));
      }
    } else {
      hi = tau;
    }
    tau = 0.5 * (lo + hi);
    SPAMM_TRY(vr_at(tau, &vr));
    ++it;
  }
  *tau_out = tau;
  if (vr_out) *vr_out = vr;
  if (iters_out) *iters_out = it;
  p.tau = tau;
  p.skipmap_ready = false;
  p.last_stream = s;
  return SPAMM_OK;
}

}  // extern "C"
