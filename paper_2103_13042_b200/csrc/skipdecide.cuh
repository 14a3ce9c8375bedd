// skipdecide.cuh -- the keep predicate of one k-step of a macro-tile, shared by the skip-map
// kernel (skipmap.cu) and the fused skip + multiply kernel of small problems (multiply_x3.cu):
//   keep(i,k,j)  <=>  !(nA[i][k] * nB[k][j] < tau)   in float64 (PAPER.md:47/63/155; NaN kept, R2)
#pragma once
#include <cstdint>
#include <type_traits>

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

}  // namespace spamm
