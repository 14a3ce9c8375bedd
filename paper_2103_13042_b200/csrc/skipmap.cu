// skipmap.cu -- stage 2: the per-C-tile skip map (Alg. 2 lines 3-16, PAPER.md:152-172;
// valid-multiplication counts V, Sec. 3.5.1).
//
// keep(i,k,j)  <=>  !(nA[i][k] * nB[k][j] < tau)   in float64 (">= tau", PAPER.md:47/63/155;
// NaN kept, reading R2).
//
// B200 design: instead of one bitmap per CUDA block inside the multiply (the paper's
// map_offset compaction), the map is materialised once, globally:
//   count : one CTA per scheduling macro-tile (4 x MJ C tiles), its 8 warps split k in
//           32-wide chunks (lane = k); per-C-tile counts V, the macro-tile's union count
//           U, row work (atomics) and a histogram of U (for the schedule);
//   scan  : one CTA (CUB for very many macro-tiles) -- exclusive scans over macro-tiles of
//           U (macro-list offsets) and L = kept pairs of the macro-tile (leaf-list
//           offsets; C-tile lists are stored macro-major), and of the U histogram in
//           descending order (bucket starts of the longest-processing-time-first schedule);
//   emit  : one CTA per macro-tile; warps count per chunk, scan the chunk counts in
//           shared memory, then write the ascending k list of every C tile (uint16), the
//           (k, keep-mask) list of the macro-tile and, for the tensor path, each k-step's
//           MMA runs (adjacent C-tile columns with equal row pattern) pre-decoded; the
//           macro-tile takes a slot in its U bucket: an LPT order without a sort.
// All passes evaluate the identical predicate code, so lists match counts exactly.
#include <cub/cub.cuh>

#include "internal.h"

namespace spamm {
namespace {

constexpr int kWarps = 8;
constexpr int kRoundChunks = 64;     // k-chunks (of 32) per emit round: 2048 k

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
  // Exact pre-filter: norms are >= 0 (or NaN), rounding is monotone, so
  // max(a) * max(b) < tau implies every a*b < tau.  NaN-propagating maxima keep NaN pairs.
  double amax = 0.0, bmax = 0.0;
#pragma unroll
  for (int li = 0; li < MI; ++li) amax = (a[li] > amax || a[li] != a[li]) ? a[li] : amax;
#pragma unroll
  for (int lj = 0; lj < MJ; ++lj) bmax = (b[lj] > bmax || b[lj] != b[lj]) ? b[lj] : bmax;
  if (__dmul_rn(amax, bmax) < tau) return 0u;
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
__global__ void __launch_bounds__(kWarps * 32)
    skip_count_kernel(const double* __restrict__ nA, const double* __restrict__ nBt, int64_t BM, int64_t BK,
                      int64_t BN, double tau, int64_t GN, int64_t gi0, int64_t* __restrict__ V,
                      int64_t* __restrict__ U, int64_t* __restrict__ Lm,
                      unsigned long long* __restrict__ row_work, unsigned long long* __restrict__ hist) {
  constexpr int NB = MI * MJ;
  __shared__ uint32_t red[kWarps][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = blockIdx.x;
  const int64_t I = gi0 + m / GN, J = m % GN;
  uint32_t my = 0, u = 0;   // lane b < NB: count of C tile b;  u: union count (warp-uniform)
  for (int64_t kc = static_cast<int64_t>(warp) * 32; kc < BK; kc += kWarps * 32) {
    const uint32_t mask = chunk_mask<MI, MJ>(nA, nBt, BM, BK, BN, tau, I, J, kc + lane);
    const uint32_t any = __ballot_sync(0xffffffffu, mask != 0u);
    if (any == 0u) continue;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const uint32_t bal = __ballot_sync(0xffffffffu, (mask >> b) & 1u);
      if (lane == b) my += __popc(bal);
    }
    u += __popc(any);
  }
  red[warp][lane] = my;
  if (lane == 0) red[warp][32] = u;
  __syncthreads();
  if (warp == 0) {
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) tot += red[w][lane];
    const int li = lane / MJ, lj = lane % MJ;
    const int64_t i = I * MI + li, j = J * MJ + lj;
    const bool valid = lane < NB && i < BM && j < BN;
    if (valid) V[i * BN + j] = tot;
    // row work: sum over the MJ lanes of each tile row
    uint32_t rs = valid ? tot : 0u;
#pragma unroll
    for (int o = 1; o < MJ; o <<= 1) {
      const uint32_t other = __shfl_down_sync(0xffffffffu, rs, o);
      if ((lj + o) < MJ) rs += other;
    }
    if (lane < NB && lj == 0 && i < BM && rs) atomicAdd(row_work + i, static_cast<unsigned long long>(rs));
    uint32_t lsum = valid ? tot : 0u;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    if (lane == 0) {
      Lm[I * GN + J] = lsum;
      uint32_t ut = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) ut += red[w][32];
      U[I * GN + J] = ut;
      atomicAdd(hist + ut, 1ull);
    }
  }
}

// Exclusive scan of n int64 values by one CTA of 1024 threads; out has n+1 entries, out[n] =
// total.  If reverse, out[u] = sum_{u' > u} in[u'] (descending buckets).
__device__ void block_scan_array(const int64_t* __restrict__ in, int64_t* __restrict__ out, int64_t n,
                                 bool reverse, int64_t* s_warp) {
  constexpr int kT = 1024, kItems = 8;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int64_t carry = 0;
  for (int64_t base = 0; base < n; base += kT * kItems) {
    int64_t v[kItems], sum = 0;
#pragma unroll
    for (int e = 0; e < kItems; ++e) {
      const int64_t x = base + static_cast<int64_t>(t) * kItems + e;
      v[e] = x < n ? in[reverse ? (n - 1 - x) : x] : 0;
      sum += v[e];
    }
    int64_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int64_t w = s_warp[lane], wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      s_warp[lane] = wi - w;          // exclusive warp offsets
      if (lane == 31) s_warp[32] = wi;  // chunk total
    }
    __syncthreads();
    int64_t run = carry + s_warp[warp] + (incl - sum);
#pragma unroll
    for (int e = 0; e < kItems; ++e) {
      const int64_t x = base + static_cast<int64_t>(t) * kItems + e;
      if (x < n) out[reverse ? (n - 1 - x) : x] = run;
      run += v[e];
    }
    carry += s_warp[32];
    __syncthreads();
  }
  if (t == 0) out[n] = carry;   // total
}

__global__ void __launch_bounds__(1024)
    skip_scan_kernel(const int64_t* __restrict__ U, int64_t* __restrict__ macro_ptr,
                     const int64_t* __restrict__ Lm, int64_t* __restrict__ leaf_base, int64_t nmac,
                     const int64_t* __restrict__ hist, int64_t* __restrict__ bucket_pos, int64_t nbucket) {
  __shared__ int64_t s_warp[33];
  if (nmac > 0) {
    block_scan_array(U, macro_ptr, nmac, false, s_warp);
    block_scan_array(Lm, leaf_base, nmac, false, s_warp);
  }
  // bucket_pos[u] = number of macro-tiles with union count > u (descending buckets)
  block_scan_array(hist, bucket_pos, nbucket, true, s_warp);
}

// Runs of a 4 x 8 keep mask for the tensor path: adjacent C-tile columns with the same
// non-zero 4-bit row pattern.  run = j0 | (len-1) << 3 | pat << 6  (10 bits, 3 per word).
__device__ __forceinline__ uint32_t col_pattern8(uint32_t mask, int lj) {
  return ((mask >> lj) & 1u) | (((mask >> (8 + lj)) & 1u) << 1) | (((mask >> (16 + lj)) & 1u) << 2) |
         (((mask >> (24 + lj)) & 1u) << 3);
}
__device__ __forceinline__ uint4 encode_runs(uint32_t k, uint32_t mask) {
  uint32_t words[3] = {0u, 0u, 0u};
  uint32_t nr = 0, cols = 0;
  int j = 0;
  while (j < 8) {
    const uint32_t pat = col_pattern8(mask, j);
    int j1 = j + 1;
    while (j1 < 8 && col_pattern8(mask, j1) == pat) ++j1;
    if (pat) {
      const uint32_t run = static_cast<uint32_t>(j) | (static_cast<uint32_t>(j1 - j - 1) << 3) | (pat << 6);
      words[nr / 3] |= run << (10 * (nr % 3));
      ++nr;
      cols |= ((1u << (j1 - j)) - 1u) << j;
    }
    j = j1;
  }
  return make_uint4(k | (nr << 16) | (cols << 24), words[0], words[1], words[2]);
}

template <int MI, int MJ>
__global__ void __launch_bounds__(kWarps * 32)
    skip_emit_kernel(const double* __restrict__ nA, const double* __restrict__ nBt, int64_t BM, int64_t BK,
                     int64_t BN, double tau, int64_t GN, int64_t gi0, const int64_t* __restrict__ V,
                     const int64_t* __restrict__ leaf_base, const int64_t* __restrict__ macro_ptr,
                     const int64_t* __restrict__ U, unsigned long long* __restrict__ bucket_pos,
                     int64_t* __restrict__ leaf_start, uint16_t* __restrict__ leaf_k,
                     uint2* __restrict__ macro_ent, uint4* __restrict__ macro_run, int32_t* __restrict__ order) {
  constexpr int NB = MI * MJ;
  __shared__ uint32_t ccnt[kRoundChunks][33];   // per chunk: per-C-tile counts, [32] = union count
  __shared__ int64_t base[33];                  // running write offsets: C tiles, [32] = macro list
  __shared__ uint32_t rtot[33];                 // round totals
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = blockIdx.x;
  const int64_t I = gi0 + m / GN, J = m % GN;
  const int64_t tile = I * GN + J;
  if (threadIdx.x < 32) {
    // C-tile lists are stored macro-major: start = leaf_base[tile] + counts of earlier C tiles
    const int64_t i = I * MI + lane / MJ, j = J * MJ + lane % MJ;
    const bool valid = lane < NB && i < BM && j < BN;
    const int64_t v = valid ? V[i * BN + j] : 0;
    int64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int64_t start = leaf_base[tile] + incl - v;
    if (valid) leaf_start[i * BN + j] = start;
    base[lane] = start;
    if (lane == 0) {
      base[32] = macro_ptr[tile];
      const unsigned long long slot = atomicAdd(bucket_pos + U[tile], 1ull);
      order[slot] = static_cast<int32_t>(tile);
    }
  }
  const uint32_t lt = (1u << lane) - 1u;
  const int64_t nchunks = (BK + 31) / 32;
  for (int64_t c0 = 0; c0 < nchunks; c0 += kRoundChunks) {
    const int nc = static_cast<int>(nchunks - c0 < kRoundChunks ? nchunks - c0 : kRoundChunks);
    // phase 1: per-chunk counts
    for (int c = warp; c < nc; c += kWarps) {
      const uint32_t mask = chunk_mask<MI, MJ>(nA, nBt, BM, BK, BN, tau, I, J, (c0 + c) * 32 + lane);
      const uint32_t any = __ballot_sync(0xffffffffu, mask != 0u);
      uint32_t my = 0;
      if (any != 0u) {
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const uint32_t bal = __ballot_sync(0xffffffffu, (mask >> b) & 1u);
          if (lane == b) my = __popc(bal);
        }
      }
      ccnt[c][lane] = my;
      if (lane == 0) ccnt[c][32] = __popc(any);
    }
    __syncthreads();
    // phase 2: exclusive scan over the round's chunks, one column per thread
    if (threadIdx.x < 33) {
      const int col = threadIdx.x;
      uint32_t run = 0;
      for (int c = 0; c < nc; ++c) {
        const uint32_t x = ccnt[c][col];
        ccnt[c][col] = run;
        run += x;
      }
      rtot[col] = run;
    }
    __syncthreads();
    // phase 3: write the lists (masks recomputed; identical predicate code)
    for (int c = warp; c < nc; c += kWarps) {
      const int64_t k = (c0 + c) * 32 + lane;
      const uint32_t mask = chunk_mask<MI, MJ>(nA, nBt, BM, BK, BN, tau, I, J, k);
      const uint32_t any = __ballot_sync(0xffffffffu, mask != 0u);
      if (any == 0u) continue;
      if (mask) {
        const int64_t e = base[32] + ccnt[c][32] + __popc(any & lt);
        macro_ent[e] = make_uint2(static_cast<uint32_t>(k), mask);
        if (MJ == 8 && macro_run != nullptr) macro_run[e] = encode_runs(static_cast<uint32_t>(k), mask);
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const bool bit = (mask >> b) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
        if (bit) leaf_k[base[b] + ccnt[c][b] + __popc(bal & lt)] = static_cast<uint16_t>(k);
      }
    }
    __syncthreads();
    if (threadIdx.x < 33) base[threadIdx.x] += rtot[threadIdx.x];
    __syncthreads();
  }
}

template <int MJ>
spamm_status count_t(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s) {
  const int64_t n_macro = (gi1 - gi0) * p.GN;
  if (n_macro <= 0) return SPAMM_OK;
  skip_count_kernel<kMacroI, MJ><<<static_cast<unsigned>(n_macro), kWarps * 32, 0, s>>>(
      p.nA, p.nBt, p.BM, p.BK, p.BN, p.tau, p.GN, gi0, p.V, p.U, p.L,
      reinterpret_cast<unsigned long long*>(p.row_work), reinterpret_cast<unsigned long long*>(p.hist));
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

template <int MJ>
spamm_status emit_t(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s) {
  const int64_t n_macro = (gi1 - gi0) * p.GN;
  if (n_macro <= 0) return SPAMM_OK;
  skip_emit_kernel<kMacroI, MJ><<<static_cast<unsigned>(n_macro), kWarps * 32, 0, s>>>(
      p.nA, p.nBt, p.BM, p.BK, p.BN, p.tau, p.GN, gi0, p.V, p.leaf_base, p.macro_ptr, p.U,
      reinterpret_cast<unsigned long long*>(p.bucket_pos), p.leaf_start, p.leaf_k, p.macro_ent, p.macro_run,
      p.order);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

constexpr int64_t kSmallScan = int64_t(1) << 15;   // macro-tile counts scanned by the single-CTA kernel

}  // namespace

// count pass + scans (macro-list and leaf-list offsets, LPT bucket starts) for macro rows [gi0, gi1)
spamm_status launch_skipmap_count(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s) {
  const int64_t nleaf = p.BM * p.BN, nmac = p.GM * p.GN;
  const bool partial = gi0 != 0 || gi1 != p.GM;
  if (partial) {
    SPAMM_CUDA_TRY(cudaMemsetAsync(p.V, 0, sizeof(int64_t) * (nleaf + 1), s));
    SPAMM_CUDA_TRY(cudaMemsetAsync(p.U, 0, sizeof(int64_t) * (nmac + 1), s));
    SPAMM_CUDA_TRY(cudaMemsetAsync(p.L, 0, sizeof(int64_t) * (nmac + 1), s));
  }
  SPAMM_CUDA_TRY(cudaMemsetAsync(p.row_work, 0, sizeof(int64_t) * p.BM, s));
  SPAMM_CUDA_TRY(cudaMemsetAsync(p.hist, 0, sizeof(int64_t) * (p.BK + 2), s));
  if (p.MJ == kMacroJ_umma) {
    SPAMM_TRY(count_t<kMacroJ_umma>(p, gi0, gi1, s));
  } else {
    SPAMM_TRY(count_t<kMacroJ_simt>(p, gi0, gi1, s));
  }
  // Out-of-range macro-tiles (multi-GPU shards) have U = L = 0 and are not in the histogram.
  const bool small = nmac <= kSmallScan;
  if (!small) {
    size_t bytes = p.cub_tmp_bytes;
    SPAMM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(p.cub_tmp, bytes, p.U, p.macro_ptr, nmac + 1, s));
    bytes = p.cub_tmp_bytes;
    SPAMM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(p.cub_tmp, bytes, p.L, p.leaf_base, nmac + 1, s));
  }
  skip_scan_kernel<<<1, 1024, 0, s>>>(p.U, p.macro_ptr, p.L, p.leaf_base, small ? nmac : 0, p.hist,
                                      p.bucket_pos, p.BK + 1);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

spamm_status launch_skipmap_emit(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s) {
  if (p.MJ == kMacroJ_umma) return emit_t<kMacroJ_umma>(p, gi0, gi1, s);
  return emit_t<kMacroJ_simt>(p, gi0, gi1, s);
}

// CUB temp-storage requirement for the plan's sizes (many-macro-tile scans only).
size_t skipmap_cub_bytes(int64_t nleaf, int64_t nmac) {
  size_t a = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, static_cast<int64_t*>(nullptr), static_cast<int64_t*>(nullptr),
                                nmac + 1);
  (void)nleaf;
  return a;
}

}  // namespace spamm
