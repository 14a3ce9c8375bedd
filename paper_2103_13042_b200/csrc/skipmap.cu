// skipmap.cu -- stage 2: the per-C-tile skip map (Alg. 2 lines 3-16, PAPER.md:152-172;
// valid-multiplication counts V, Sec. 3.5.1).
//
// keep(i,k,j)  <=>  !(nA[i][k] * nB[k][j] < tau)   in float64 (">= tau", PAPER.md:47/63/155;
// NaN kept, reading R2).
//
// B200 design: instead of one bitmap per CUDA block inside the multiply (the paper's
// map_offset compaction), the map is materialised once, globally, in two passes over
// the BM*BK*BN tests.  One warp owns one scheduling macro-tile (4 x MJ C tiles) and
// walks k in chunks of 32 (lane = k):
//   count : per-C-tile counts V, per-macro-tile union counts U, row work (atomics);
//   (CUB exclusive scans V -> leaf_ptr, U -> macro_ptr; CUB radix sort U -> LPT order)
//   emit  : ascending k lists per C tile (uint16) and (k, mask) lists per macro-tile.
// Both passes evaluate the identical predicate code, so the lists match the counts.
#include <cub/cub.cuh>

#include "internal.h"

namespace spamm {
namespace {

constexpr int kWarpsPerBlock = 8;

template <int MI, int MJ>
struct Chunk {
  uint32_t mask;   // bit li*MJ+lj set if (I*MI+li, k, J*MJ+lj) is kept
};

template <int MI, int MJ>
__device__ __forceinline__ uint32_t chunk_mask(const double* __restrict__ nA, const double* __restrict__ nBt,
                                               int64_t BM, int64_t BK, int64_t BN, double tau, int64_t I,
                                               int64_t J, int64_t k) {
  if (k >= BK) return 0u;
  double a[MI], b[MJ];
  bool va[MI], vb[MJ];
#pragma unroll
  for (int li = 0; li < MI; ++li) {
    const int64_t i = I * MI + li;
    va[li] = i < BM;
    a[li] = va[li] ? __ldg(nA + i * BK + k) : 0.0;
  }
#pragma unroll
  for (int lj = 0; lj < MJ; ++lj) {
    const int64_t j = J * MJ + lj;
    vb[lj] = j < BN;
    b[lj] = vb[lj] ? __ldg(nBt + j * BK + k) : 0.0;
  }
  uint32_t mask = 0u;
#pragma unroll
  for (int li = 0; li < MI; ++li)
#pragma unroll
    for (int lj = 0; lj < MJ; ++lj) {
      const double prod = __dmul_rn(a[li], b[lj]);
      const bool keep = va[li] && vb[lj] && !(prod < tau);
      mask |= static_cast<uint32_t>(keep) << (li * MJ + lj);
    }
  return mask;
}

template <int MI, int MJ>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    skip_count_kernel(const double* __restrict__ nA, const double* __restrict__ nBt, int64_t BM, int64_t BK,
                      int64_t BN, double tau, int64_t GN, int64_t gi0, int64_t n_macro, int64_t* __restrict__ V,
                      int64_t* __restrict__ U, unsigned long long* __restrict__ row_work) {
  const int lane = threadIdx.x & 31;
  const int64_t m = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
  if (m >= n_macro) return;
  const int64_t I = gi0 + m / GN, J = m % GN;
  uint32_t cnt[MI * MJ];
#pragma unroll
  for (int b = 0; b < MI * MJ; ++b) cnt[b] = 0u;
  uint32_t u = 0u;
  for (int64_t kc = 0; kc < BK; kc += 32) {
    const uint32_t mask = chunk_mask<MI, MJ>(nA, nBt, BM, BK, BN, tau, I, J, kc + lane);
#pragma unroll
    for (int b = 0; b < MI * MJ; ++b) cnt[b] += (mask >> b) & 1u;
    u += mask != 0u;
  }
#pragma unroll
  for (int b = 0; b < MI * MJ; ++b) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) cnt[b] += __shfl_xor_sync(0xffffffffu, cnt[b], o);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
  if (lane == 0) {
    U[I * GN + J] = u;
#pragma unroll
    for (int li = 0; li < MI; ++li) {
      const int64_t i = I * MI + li;
      if (i >= BM) continue;
      unsigned long long rw = 0;
#pragma unroll
      for (int lj = 0; lj < MJ; ++lj) {
        const int64_t j = J * MJ + lj;
        if (j < BN) {
          V[i * BN + j] = cnt[li * MJ + lj];
          rw += cnt[li * MJ + lj];
        }
      }
      if (rw) atomicAdd(row_work + i, rw);
    }
  }
}

template <int MI, int MJ>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    skip_emit_kernel(const double* __restrict__ nA, const double* __restrict__ nBt, int64_t BM, int64_t BK,
                     int64_t BN, double tau, int64_t GN, int64_t gi0, int64_t n_macro,
                     const int64_t* __restrict__ leaf_ptr, const int64_t* __restrict__ macro_ptr,
                     uint16_t* __restrict__ leaf_k, uint2* __restrict__ macro_ent) {
  const int lane = threadIdx.x & 31;
  const int64_t m = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
  if (m >= n_macro) return;
  const int64_t I = gi0 + m / GN, J = m % GN;
  // lane b keeps the running write offset of C tile b of the macro-tile
  int64_t lbase = 0;
  if (lane < MI * MJ) {
    const int64_t i = I * MI + lane / MJ, j = J * MJ + lane % MJ;
    if (i < BM && j < BN) lbase = leaf_ptr[i * BN + j];
  }
  int64_t mbase = macro_ptr[I * GN + J];
  const uint32_t lt = (1u << lane) - 1u;
  for (int64_t kc = 0; kc < BK; kc += 32) {
    const int64_t k = kc + lane;
    const uint32_t mask = chunk_mask<MI, MJ>(nA, nBt, BM, BK, BN, tau, I, J, k);
    const uint32_t any = __ballot_sync(0xffffffffu, mask != 0u);
    if (any == 0u) continue;
    if (mask) macro_ent[mbase + __popc(any & lt)] = make_uint2(static_cast<uint32_t>(k), mask);
    mbase += __popc(any);
#pragma unroll
    for (int b = 0; b < MI * MJ; ++b) {
      const bool bit = (mask >> b) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, bit);
      if (bal == 0u) continue;
      const int64_t base = __shfl_sync(0xffffffffu, lbase, b);
      if (bit) leaf_k[base + __popc(bal & lt)] = static_cast<uint16_t>(k);
      if (lane == b) lbase += __popc(bal);
    }
  }
}

__global__ void iota_kernel(int32_t* out, int64_t n, int64_t base) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) out[t] = static_cast<int32_t>(base + t);
}

template <int MJ>
spamm_status count_t(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s) {
  const int64_t n_macro = (gi1 - gi0) * p.GN;
  if (n_macro <= 0) return SPAMM_OK;
  const int64_t blocks = (n_macro + kWarpsPerBlock - 1) / kWarpsPerBlock;
  skip_count_kernel<kMacroI, MJ><<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, 0, s>>>(
      p.nA, p.nBt, p.BM, p.BK, p.BN, p.tau, p.GN, gi0, n_macro, p.V, p.U,
      reinterpret_cast<unsigned long long*>(p.row_work));
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

template <int MJ>
spamm_status emit_t(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s) {
  const int64_t n_macro = (gi1 - gi0) * p.GN;
  if (n_macro <= 0) return SPAMM_OK;
  const int64_t blocks = (n_macro + kWarpsPerBlock - 1) / kWarpsPerBlock;
  skip_emit_kernel<kMacroI, MJ><<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, 0, s>>>(
      p.nA, p.nBt, p.BM, p.BK, p.BN, p.tau, p.GN, gi0, n_macro, p.leaf_ptr, p.macro_ptr, p.leaf_k, p.macro_ent);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

}  // namespace

// count pass + scans + LPT sort for macro rows [gi0, gi1)
spamm_status launch_skipmap_count(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s) {
  const int64_t nleaf = p.BM * p.BN, nmac = p.GM * p.GN;
  SPAMM_CUDA_TRY(cudaMemsetAsync(p.V, 0, sizeof(int64_t) * (nleaf + 1), s));
  SPAMM_CUDA_TRY(cudaMemsetAsync(p.U, 0, sizeof(int64_t) * (nmac + 1), s));
  SPAMM_CUDA_TRY(cudaMemsetAsync(p.row_work, 0, sizeof(int64_t) * p.BM, s));
  if (p.MJ == kMacroJ_umma) {
    SPAMM_TRY(count_t<kMacroJ_umma>(p, gi0, gi1, s));
  } else {
    SPAMM_TRY(count_t<kMacroJ_simt>(p, gi0, gi1, s));
  }
  size_t bytes = p.cub_tmp_bytes;
  SPAMM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(p.cub_tmp, bytes, p.V, p.leaf_ptr, nleaf + 1, s));
  bytes = p.cub_tmp_bytes;
  SPAMM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(p.cub_tmp, bytes, p.U, p.macro_ptr, nmac + 1, s));
  // LPT schedule over the macro-tiles of the range: descending union length
  const int64_t n = (gi1 - gi0) * p.GN;
  if (n > 0) {
    iota_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(p.order_tmp, n, gi0 * p.GN);
    count_launch();
    bytes = p.cub_tmp_bytes;
    SPAMM_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(p.cub_tmp, bytes, p.U + gi0 * p.GN, p.keys_tmp,
                                                             p.order_tmp, p.order, static_cast<int>(n), 0,
                                                             32, s));
  }
  return SPAMM_OK;
}

spamm_status launch_skipmap_emit(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s) {
  if (p.MJ == kMacroJ_umma) return emit_t<kMacroJ_umma>(p, gi0, gi1, s);
  return emit_t<kMacroJ_simt>(p, gi0, gi1, s);
}

// CUB temp-storage requirement for the plan's sizes.
size_t skipmap_cub_bytes(int64_t nleaf, int64_t nmac) {
  size_t a = 0, b = 0, c = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, static_cast<int64_t*>(nullptr), static_cast<int64_t*>(nullptr),
                                nleaf + 1);
  cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<int64_t*>(nullptr), static_cast<int64_t*>(nullptr),
                                nmac + 1);
  cub::DeviceRadixSort::SortPairsDescending(nullptr, c, static_cast<int64_t*>(nullptr),
                                            static_cast<int64_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                            static_cast<int32_t*>(nullptr), static_cast<int>(nmac), 0, 32);
  size_t m = a > b ? a : b;
  return m > c ? m : c;
}

}  // namespace spamm
