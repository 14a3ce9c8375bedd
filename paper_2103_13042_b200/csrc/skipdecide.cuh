// skipdecide.cuh -- the keep predicate of one k-step of a macro-tile, shared by the skip-map
// kernel (skipmap.cu) and the fused skip + multiply kernel of small problems (multiply_x3.cu):
//   keep(i,k,j)  <=>  !(nA[i][k] * nB[k][j] < tau)   in float64 (PAPER.md:47/63/155; NaN kept, R2)
#pragma once
#include <cstdint>
#include <type_traits>

#include <cuda_runtime.h>

namespace spamm {

// keep bits of one k-step of a macro-tile: bit li*MJ+lj; 64-bit for 8 x 8 macro-tiles
template <int MI, int MJ>
using mask_t = typename std::conditional<(MI * MJ > 32), unsigned long long, uint32_t>::type;

template <int MI, int MJ>
struct ChunkVals {
  double a[MI], b[MJ];
};

// keep bits of one k: bit li*MJ+lj <=> !(a*b < tau), masked by the in-range tiles `valid`.
template <int MI, int MJ>
__device__ __forceinline__ mask_t<MI, MJ> chunk_mask(const ChunkVals<MI, MJ>& v, mask_t<MI, MJ> valid, double tau) {
  using M_ = mask_t<MI, MJ>;
  // Exact pre-filters (monotone rounding; NaN-propagating maxima keep NaN pairs):
  //   max(a) * max(b) < tau  =>  every a*b < tau;   min(a) * min(b) >= tau  =>  every a*b >= tau.
  double amax = 0.0, bmax = 0.0, amin = v.a[0], bmin = v.b[0];
#pragma unroll
  for (int li = 0; li < MI; ++li) {
    amax = (v.a[li] > amax || v.a[li] != v.a[li]) ? v.a[li] : amax;
    amin = fmin(amin, v.a[li]);
  }
#pragma unroll
  for (int lj = 0; lj < MJ; ++lj) {
    bmax = (v.b[lj] > bmax || v.b[lj] != v.b[lj]) ? v.b[lj] : bmax;
    bmin = fmin(bmin, v.b[lj]);
  }
  if (valid == 0u || __dmul_rn(amax, bmax) < tau) return 0u;
  if (__dmul_rn(amin, bmin) >= tau) return valid;
  M_ mask = 0u;
#pragma unroll
  for (int li = 0; li < MI; ++li) {
    uint32_t row = 0u;   // 32-bit row bits, merged into the (possibly 64-bit) mask once per row
#pragma unroll
    for (int lj = 0; lj < MJ; ++lj) {
      const double prod = __dmul_rn(v.a[li], v.b[lj]);
      row |= static_cast<uint32_t>(!(prod < tau)) << lj;
    }
    mask |= static_cast<M_>(row) << (li * MJ);
  }
  return mask & valid;
}

// bit li*MJ+lj set iff C tile (I*MI+li, J*MJ+lj) exists
template <int MI, int MJ>
__device__ __forceinline__ mask_t<MI, MJ> valid_bits(int64_t BM, int64_t BN, int64_t I, int64_t J) {
  using M_ = mask_t<MI, MJ>;
  const int64_t rr = BM - I * MI, cc = BN - J * MJ;   // C-tile rows / columns left in the grid
  const int rv = rr >= MI ? MI : (rr > 0 ? static_cast<int>(rr) : 0);
  const int cv = cc >= MJ ? MJ : (cc > 0 ? static_cast<int>(cc) : 0);
  const M_ row = (static_cast<M_>(1u) << cv) - 1u;    // MJ <= 8: one row's column bits
  M_ v = 0u;
#pragma unroll
  for (int li = 0; li < MI; ++li)
    if (li < rv) v |= row << (li * MJ);
  return v;
}

// Fused skip map (small problems, spamm_run): the producer warp decides its own macro-tile's
// (k, keep mask) list from the norm maps -- the same predicate and list format as the skip-map
// kernel (skipdecide.cuh, skipmap.cu) -- writes it with U, L, row work, totals and the identity
// claim order for the getters, then streams the kept k-steps (multiply_x3.cu, multiply_simt.cu).  No skip-map launch, no claim counter.
struct XFuse {
  const double* nA;    // [BM][BK]
  const double* nBt;   // [BN][BK]
  int64_t BM, BK, BN;
  double tau;
  int64_t* U;          // [GM*GN] k-steps per macro-tile (written)
  int64_t* L;          // [GM*GN] kept pairs per macro-tile (written)
  uint2* ment;         // [GM*GN][BK] (k, mask) entries (written)
  int32_t* order;      // [GM*GN] claim order (identity, written)
  unsigned long long* row_work;   // [BM] (zeroed by the norm kernel)
  unsigned long long* totals;     // [0] kept pairs [1] k-steps [2] macro-tiles without kept pairs (zeroed)
};

// kFuse: the skip map of macro-tile t (4 x 4 C tiles), decided by one warp in ascending k
// (lane = k) exactly as skip_pyr_kernel's no-pyramid branch decides it; returns U[t].
// With BK <= 32 (one chunk) the lane's entry stays in registers: *reg = (k, mask) of this lane's k,
// *any = the ballot of non-empty masks (entry q is held by the q-th set lane).
__device__ __forceinline__ int64_t fuse_tile_list(const XFuse& fz, int64_t t, int64_t GN, int lane, uint2* reg,
                                                  uint32_t* any_out) {
  const int64_t I = t / GN, J = t % GN;
  const uint32_t valid = valid_bits<4, 4>(fz.BM, fz.BN, I, J);
  const uint32_t lt = (1u << lane) - 1u;
  int64_t mbase = t * fz.BK;
  uint32_t rw[4] = {0u, 0u, 0u, 0u};
  for (int64_t k0 = 0; k0 < fz.BK; k0 += 32) {
    const int64_t k = k0 + lane;
    uint32_t mask = 0u;
    if (k < fz.BK && valid != 0u) {
      ChunkVals<4, 4> cv;
#pragma unroll
      for (int li = 0; li < 4; ++li) {
        const int64_t i = I * 4 + li;
        cv.a[li] = i < fz.BM ? __ldg(fz.nA + i * fz.BK + k) : 0.0;
      }
#pragma unroll
      for (int lj = 0; lj < 4; ++lj) {
        const int64_t j = J * 4 + lj;
        cv.b[lj] = j < fz.BN ? __ldg(fz.nBt + j * fz.BK + k) : 0.0;
      }
      mask = chunk_mask<4, 4>(cv, valid, fz.tau);
    }
#pragma unroll
    for (int li = 0; li < 4; ++li) rw[li] += static_cast<uint32_t>(__popc((mask >> (4 * li)) & 0xFu));
    const uint32_t any = __ballot_sync(0xffffffffu, mask != 0u);
    if (mask) fz.ment[mbase + __popc(any & lt)] = make_uint2(static_cast<uint32_t>(k), mask);
    mbase += __popc(any);
    *reg = make_uint2(static_cast<uint32_t>(k), mask);
    *any_out = any;
  }
  uint32_t lsum = 0;
#pragma unroll
  for (int li = 0; li < 4; ++li) {
    uint32_t v = rw[li];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    lsum += v;
    if (lane == li && I * 4 + li < fz.BM && v) atomicAdd(fz.row_work + I * 4 + li, static_cast<unsigned long long>(v));
  }
  const int64_t u = mbase - t * fz.BK;
  if (lane == 0) {
    fz.U[t] = u;
    fz.L[t] = lsum;
    fz.order[t] = static_cast<int32_t>(t);
    if (lsum) atomicAdd(fz.totals, static_cast<unsigned long long>(lsum));
    if (u) atomicAdd(fz.totals + 1, static_cast<unsigned long long>(u));
    else atomicAdd(fz.totals + 2, 1ull);
  }
  __syncwarp();   // BK > 32: the entries are read back by the whole warp
  return u;
}

}  // namespace spamm
