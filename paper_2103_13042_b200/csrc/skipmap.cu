// skipmap.cu -- stage 2: the per-C-tile skip map (Alg. 2 lines 3-16, PAPER.md:152-172;
// valid-multiplication counts V, Sec. 3.5.1).
//
// keep(i,k,j)  <=>  !(nA[i][k] * nB[k][j] < tau)   in float64 (">= tau", PAPER.md:47/63/155;
// NaN kept, reading R2).
//
// B200 design: instead of one bitmap per CUDA block inside the multiply (the paper's
// map_offset compaction), the map is materialised once, globally:
//   count : one warp per scheduling macro-tile (4 x MJ C tiles) walks k in 32-wide chunks
//           (lane = k) with the next chunk's norm loads in flight; per-C-tile counts V,
//           the macro-tile's union count U, row work and a histogram of U; the last CTA
//           to finish (threadfence + ticket) performs the scans below;
//   scan  : one CTA (CUB for very many macro-tiles) -- exclusive scans over macro-tiles of
//           U (macro-list offsets) and L = kept pairs of the macro-tile (leaf-list
//           offsets; C-tile lists are stored macro-major), and of the U histogram in
//           descending order (bucket starts of the longest-processing-time-first schedule);
//   emit  : one warp per macro-tile walks k again (same predicate code, same prefetch),
//           skipping all-zero chunks, and writes the ascending k list of every C tile
//           (uint16), the (k, keep-mask) list of the macro-tile and, for the tensor path,
//           each k-step's MMA runs (adjacent C-tile columns with equal row pattern)
//           pre-decoded; the macro-tile takes a slot in its U bucket: an LPT order
//           without a sort.
// All passes evaluate the identical predicate code, so lists match counts exactly.
#include <cub/cub.cuh>

#include "internal.h"

namespace spamm {
namespace {

constexpr int kWarps = 8;

template <int MI, int MJ>
struct ChunkVals {
  double a[MI], b[MJ];
  bool kin;   // k < BK
};

// Norms of k-chunk column k for the MI rows of macro row I and the MJ columns of macro col J.
// Out-of-range entries load as 0 and are masked by index below.
template <int MI, int MJ>
__device__ __forceinline__ ChunkVals<MI, MJ> load_chunk(const double* __restrict__ nA, const double* __restrict__ nBt,
                                                        int64_t BM, int64_t BK, int64_t BN, int64_t I, int64_t J,
                                                        int64_t k) {
  ChunkVals<MI, MJ> v;
  const bool kin = k < BK;
  v.kin = kin;
#pragma unroll
  for (int li = 0; li < MI; ++li) {
    const int64_t i = I * MI + li;
    v.a[li] = (kin && i < BM) ? __ldg(nA + i * BK + k) : 0.0;
  }
#pragma unroll
  for (int lj = 0; lj < MJ; ++lj) {
    const int64_t j = J * MJ + lj;
    v.b[lj] = (kin && j < BN) ? __ldg(nBt + j * BK + k) : 0.0;
  }
  return v;
}

// keep bits of one chunk: bit li*MJ+lj <=> !(a*b < tau), for in-range (i, k, j) only.
template <int MI, int MJ>
__device__ __forceinline__ uint32_t chunk_mask(const ChunkVals<MI, MJ>& v, uint32_t valid, double tau) {
  // Exact pre-filter: norms are >= 0 (or NaN), rounding is monotone, so
  // max(a) * max(b) < tau implies every a*b < tau.  NaN-propagating maxima keep NaN pairs.
  double amax = 0.0, bmax = 0.0;
#pragma unroll
  for (int li = 0; li < MI; ++li) amax = (v.a[li] > amax || v.a[li] != v.a[li]) ? v.a[li] : amax;
#pragma unroll
  for (int lj = 0; lj < MJ; ++lj) bmax = (v.b[lj] > bmax || v.b[lj] != v.b[lj]) ? v.b[lj] : bmax;
  if (!v.kin || valid == 0u || __dmul_rn(amax, bmax) < tau) return 0u;
  uint32_t mask = 0u;
#pragma unroll
  for (int li = 0; li < MI; ++li)
#pragma unroll
    for (int lj = 0; lj < MJ; ++lj) {
      const double prod = __dmul_rn(v.a[li], v.b[lj]);
      mask |= static_cast<uint32_t>(!(prod < tau)) << (li * MJ + lj);
    }
  return mask & valid;
}

// bit li*MJ+lj set iff C tile (I*MI+li, J*MJ+lj) exists
template <int MI, int MJ>
__device__ __forceinline__ uint32_t valid_bits(int64_t BM, int64_t BN, int64_t I, int64_t J) {
  uint32_t v = 0u;
#pragma unroll
  for (int li = 0; li < MI; ++li)
#pragma unroll
    for (int lj = 0; lj < MJ; ++lj)
      if (I * MI + li < BM && J * MJ + lj < BN) v |= 1u << (li * MJ + lj);
  return v;
}

// Exclusive scan of n int64 values by one CTA; out has n+1 entries, out[n] = total.
// If reverse, out[u] = sum_{u' > u} in[u'] (descending buckets).
__device__ void block_scan_array(const int64_t* __restrict__ in, int64_t* __restrict__ out, int64_t n,
                                 bool reverse, int64_t* s_warp) {
  constexpr int kItems = 8;
  const int nt = blockDim.x, nw = nt >> 5;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int64_t carry = 0;
  for (int64_t base = 0; base < n; base += static_cast<int64_t>(nt) * kItems) {
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
      const int64_t w = lane < nw ? s_warp[lane] : 0;
      int64_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      if (lane < nw) s_warp[lane] = wi - w;   // exclusive warp offsets
      if (lane == 31) s_warp[32] = wi;        // chunk total
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
  if (t == 0) out[n] = carry;
}

struct ScanArgs {
  const int64_t* U;
  int64_t* macro_ptr;
  const int64_t* L;
  int64_t* leaf_base;
  int64_t nmac;        // 0: U/L scanned elsewhere (CUB)
  const int64_t* hist;
  int64_t* bucket_pos;
  int64_t nbucket;
  unsigned int* ticket;
};

__device__ void do_scans(const ScanArgs& sa, int64_t* s_warp) {
  if (sa.nmac > 0) {
    block_scan_array(sa.U, sa.macro_ptr, sa.nmac, false, s_warp);
    block_scan_array(sa.L, sa.leaf_base, sa.nmac, false, s_warp);
  }
  // bucket_pos[u] = number of macro-tiles with union count > u (descending buckets)
  block_scan_array(sa.hist, sa.bucket_pos, sa.nbucket, true, s_warp);
}

template <int MI, int MJ>
__global__ void __launch_bounds__(kWarps * 32)
    skip_count_kernel(const double* __restrict__ nA, const double* __restrict__ nBt, int64_t BM, int64_t BK,
                      int64_t BN, double tau, int64_t GN, int64_t gi0, int64_t n_macro, int64_t* __restrict__ V,
                      int64_t* __restrict__ U, int64_t* __restrict__ Lm, unsigned long long* __restrict__ row_work,
                      unsigned long long* __restrict__ hist, ScanArgs sa) {
  constexpr int NB = MI * MJ;
  __shared__ int64_t s_warp[33];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31;
  const int64_t m = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  if (m < n_macro) {
    const int64_t I = gi0 + m / GN, J = m % GN;
    const uint32_t valid = valid_bits<MI, MJ>(BM, BN, I, J);
    uint32_t my = 0, u = 0;   // lane b < NB: count of C tile b;  u: union count (warp-uniform)
    ChunkVals<MI, MJ> cur = load_chunk<MI, MJ>(nA, nBt, BM, BK, BN, I, J, lane);
    for (int64_t kc = 0; kc < BK; kc += 32) {
      ChunkVals<MI, MJ> nxt = cur;
      if (kc + 32 < BK) nxt = load_chunk<MI, MJ>(nA, nBt, BM, BK, BN, I, J, kc + 32 + lane);   // prefetch
      const uint32_t mask = chunk_mask<MI, MJ>(cur, valid, tau);
      const uint32_t any = __ballot_sync(0xffffffffu, mask != 0u);
      if (any != 0u) {
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const uint32_t bal = __ballot_sync(0xffffffffu, (mask >> b) & 1u);
          if (lane == b) my += __popc(bal);
        }
        u += __popc(any);
      }
      cur = nxt;
    }
    const int li = lane / MJ, lj = lane % MJ;
    const bool vl = lane < NB && ((valid >> lane) & 1u);
    if (vl) V[(I * MI + li) * BN + (J * MJ + lj)] = my;
    uint32_t rs = vl ? my : 0u;   // row work: sum over the MJ lanes of each tile row
#pragma unroll
    for (int o = 1; o < MJ; o <<= 1) {
      const uint32_t other = __shfl_down_sync(0xffffffffu, rs, o);
      if ((lj + o) < MJ) rs += other;
    }
    if (lane < NB && lj == 0 && I * MI + li < BM && rs) atomicAdd(row_work + I * MI + li, static_cast<unsigned long long>(rs));
    uint32_t lsum = vl ? my : 0u;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    if (lane == 0) {
      Lm[I * GN + J] = lsum;
      U[I * GN + J] = u;
      atomicAdd(hist + u, 1ull);
    }
  }
  // the last CTA to finish scans the per-macro-tile counts (no extra launch)
  if (sa.ticket == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int t = atomicAdd(sa.ticket, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  do_scans(sa, s_warp);
  if (threadIdx.x == 0) *sa.ticket = 0u;
}

__global__ void __launch_bounds__(1024) skip_scan_kernel(ScanArgs sa) {
  __shared__ int64_t s_warp[33];
  do_scans(sa, s_warp);
}

// Runs of a 4 x 8 keep mask for the tensor path: adjacent C-tile columns with the same
// non-zero 4-bit row pattern.  run = j0 | (len-1) << 3 | pat << 6  (10 bits, 3 per word).
__device__ __forceinline__ uint32_t col_pattern8(uint32_t mask, int lj) {
  return ((mask >> lj) & 1u) | (((mask >> (8 + lj)) & 1u) << 1) | (((mask >> (16 + lj)) & 1u) << 2) |
         (((mask >> (24 + lj)) & 1u) << 3);
}
// .w bit 31: width-2 entry (k-tiles k and k+1 share the mask; one 64-deep k-step)
__device__ __forceinline__ uint4 encode_runs(uint32_t k, uint32_t mask, uint32_t wide = 0u) {
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
  return make_uint4(k | (nr << 16) | (cols << 24), words[0], words[1], words[2] | (wide << 31));
}

template <int MI, int MJ>
__global__ void __launch_bounds__(kWarps * 32)
    skip_emit_kernel(const double* __restrict__ nA, const double* __restrict__ nBt, int64_t BM, int64_t BK,
                     int64_t BN, double tau, int64_t GN, int64_t gi0, int64_t n_macro, const int64_t* __restrict__ V,
                     const int64_t* __restrict__ leaf_base, const int64_t* __restrict__ macro_ptr,
                     const int64_t* __restrict__ U, unsigned long long* __restrict__ bucket_pos,
                     int64_t* __restrict__ leaf_start, uint16_t* __restrict__ leaf_k,
                     uint2* __restrict__ macro_ent, uint4* __restrict__ macro_run, int32_t* __restrict__ order) {
  constexpr int NB = MI * MJ;
  const int lane = threadIdx.x & 31;
  const int64_t m = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  if (m >= n_macro) return;
  const int64_t I = gi0 + m / GN, J = m % GN;
  const int64_t tile = I * GN + J;
  const uint32_t valid = valid_bits<MI, MJ>(BM, BN, I, J);
  // C-tile lists are stored macro-major: start = leaf_base[tile] + counts of earlier C tiles
  const int li = lane / MJ, lj = lane % MJ;
  const bool vl = lane < NB && ((valid >> lane) & 1u);
  const int64_t v = vl ? V[(I * MI + li) * BN + (J * MJ + lj)] : 0;
  int64_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int64_t lbase = leaf_base[tile] + incl - v;   // lane b: running write offset of C tile b
  if (vl) leaf_start[(I * MI + li) * BN + (J * MJ + lj)] = lbase;
  int64_t mbase = macro_ptr[tile];
  if (lane == 0) {
    const unsigned long long slot = atomicAdd(bucket_pos + U[tile], 1ull);
    order[slot] = static_cast<int32_t>(tile);
  }
  const uint32_t lt = (1u << lane) - 1u;
  ChunkVals<MI, MJ> cur = load_chunk<MI, MJ>(nA, nBt, BM, BK, BN, I, J, lane);
  for (int64_t kc = 0; kc < BK; kc += 32) {
    ChunkVals<MI, MJ> nxt = cur;
    if (kc + 32 < BK) nxt = load_chunk<MI, MJ>(nA, nBt, BM, BK, BN, I, J, kc + 32 + lane);   // prefetch
    const int64_t k = kc + lane;
    const uint32_t mask = chunk_mask<MI, MJ>(cur, valid, tau);
    cur = nxt;
    const uint32_t any = __ballot_sync(0xffffffffu, mask != 0u);
    if (any == 0u) continue;
    if (mask) {
      const int64_t e = mbase + __popc(any & lt);
      macro_ent[e] = make_uint2(static_cast<uint32_t>(k), mask);
      if (MJ == 8 && macro_run != nullptr) macro_run[e] = encode_runs(static_cast<uint32_t>(k), mask);
    }
    mbase += __popc(any);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const bool bit = (mask >> b) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, bit);
      if (bal == 0u) continue;
      const int64_t base = __shfl_sync(0xffffffffu, lbase, b);
      if (bit) leaf_k[base + __popc(bal & lt)] = static_cast<uint16_t>(k);
      if (lane == b) lbase += __popc(bal);
    }
  }
}


// ---------------------------------------------------------------------------
// Fixed-region mode (list storage reserved at the worst case): one pass.  Macro-tile t
// owns entries [t*BK, t*BK + U[t]) and C tile (i,j) owns k slots [(i*BN+j)*BK, .. + V),
// so no prefix sums are needed before writing.  The last CTA to finish builds the LPT
// order (U histogram -> descending bucket starts -> one slot per macro-tile) and totals.
struct LastArgs {
  const int64_t* hist;
  int64_t* bucket_pos;
  int64_t nbucket;
  const int64_t* U;
  const int64_t* L;
  int32_t* order;
  int64_t t0, t1;        // macro-tiles of the range [t0, t1)
  int64_t* totals;       // [0] kept pairs, [1] macro entries
  unsigned int* ticket;
};

__device__ void last_cta_order(const LastArgs& la, int64_t* s_warp) {
  block_scan_array(la.hist, la.bucket_pos, la.nbucket, true, s_warp);
  __syncthreads();
  int64_t kept = 0, ents = 0;
  for (int64_t t = la.t0 + threadIdx.x; t < la.t1; t += blockDim.x) {
    const int64_t u = la.U[t];
    const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(la.bucket_pos) + u, 1ull);
    la.order[slot] = static_cast<int32_t>(t);
    kept += la.L[t];
    ents += u;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    kept += __shfl_xor_sync(0xffffffffu, kept, o);
    ents += __shfl_xor_sync(0xffffffffu, ents, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(la.totals), static_cast<unsigned long long>(kept));
    atomicAdd(reinterpret_cast<unsigned long long*>(la.totals) + 1, static_cast<unsigned long long>(ents));
  }
}

template <int MI, int MJ>
__global__ void __launch_bounds__(kWarps * 32)
    skip_fused_kernel(const double* __restrict__ nA, const double* __restrict__ nBt, int64_t BM, int64_t BK,
                      int64_t BN, double tau, int64_t GN, int64_t gi0, int64_t n_macro, int64_t* __restrict__ V,
                      int64_t* __restrict__ U, int64_t* __restrict__ Lm, unsigned long long* __restrict__ row_work,
                      unsigned long long* __restrict__ hist, int64_t* __restrict__ leaf_start,
                      uint16_t* __restrict__ leaf_k, uint2* __restrict__ macro_ent, uint4* __restrict__ macro_run,
                      int64_t* __restrict__ Uw, int merge_ok, LastArgs la) {
  constexpr int NB = MI * MJ;
  __shared__ int64_t s_warp[33];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31;
  const int64_t m = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  if (m < n_macro) {
    const int64_t I = gi0 + m / GN, J = m % GN;
    const int64_t tile = I * GN + J;
    const uint32_t valid = valid_bits<MI, MJ>(BM, BN, I, J);
    const int li = lane / MJ, lj = lane % MJ;
    const bool vl = lane < NB && ((valid >> lane) & 1u);
    const int64_t leaf = (I * MI + li) * BN + (J * MJ + lj);
    const int64_t lstart = vl ? leaf * BK : 0;
    int64_t lbase = lstart;                 // lane b: running write offset of C tile b
    int64_t mbase = tile * BK;              // macro-tile region
    int64_t wbase = tile * BK;              // tensor-path entries (aligned equal-mask k pairs merged)
    const uint32_t lt = (1u << lane) - 1u;
    ChunkVals<MI, MJ> cur = load_chunk<MI, MJ>(nA, nBt, BM, BK, BN, I, J, lane);
    for (int64_t kc = 0; kc < BK; kc += 32) {
      ChunkVals<MI, MJ> nxt = cur;
      if (kc + 32 < BK) nxt = load_chunk<MI, MJ>(nA, nBt, BM, BK, BN, I, J, kc + 32 + lane);   // prefetch
      const int64_t k = kc + lane;
      const uint32_t mask = chunk_mask<MI, MJ>(cur, valid, tau);
      cur = nxt;
      const uint32_t any = __ballot_sync(0xffffffffu, mask != 0u);
      if (any == 0u) continue;
      if (mask) macro_ent[mbase + __popc(any & lt)] = make_uint2(static_cast<uint32_t>(k), mask);
      mbase += __popc(any);
      if (MJ == 8 && macro_run != nullptr) {
        // k-tiles 2p and 2p+1 with the same non-zero mask become one 64-deep k-step
        const uint32_t mnext = __shfl_down_sync(0xffffffffu, mask, 1);
        const uint32_t mprev = __shfl_up_sync(0xffffffffu, mask, 1);
        const bool even = (lane & 1) == 0;
        const bool wide = merge_ok && even && mask != 0u && mnext == mask;
        const bool absorbed = merge_ok && !even && mask != 0u && mprev == mask;
        const bool emit = mask != 0u && !absorbed;
        const uint32_t bal = __ballot_sync(0xffffffffu, emit);
        if (emit) macro_run[wbase + __popc(bal & lt)] = encode_runs(static_cast<uint32_t>(k), mask, wide ? 1u : 0u);
        wbase += __popc(bal);
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const bool bit = (mask >> b) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
        if (bal == 0u) continue;
        const int64_t base = __shfl_sync(0xffffffffu, lbase, b);
        if (bit) leaf_k[base + __popc(bal & lt)] = static_cast<uint16_t>(k);
        if (lane == b) lbase += __popc(bal);
      }
    }
    const uint32_t my = static_cast<uint32_t>(lbase - lstart);
    const uint32_t u = static_cast<uint32_t>(mbase - tile * BK);
    if (vl) {
      V[leaf] = my;
      leaf_start[leaf] = lstart;
    }
    uint32_t rs = vl ? my : 0u;   // row work: sum over the MJ lanes of each tile row
#pragma unroll
    for (int o = 1; o < MJ; o <<= 1) {
      const uint32_t other = __shfl_down_sync(0xffffffffu, rs, o);
      if ((lj + o) < MJ) rs += other;
    }
    if (lane < NB && lj == 0 && I * MI + li < BM && rs)
      atomicAdd(row_work + I * MI + li, static_cast<unsigned long long>(rs));
    uint32_t lsum = vl ? my : 0u;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    if (lane == 0) {
      Lm[tile] = lsum;
      U[tile] = u;
      if (Uw != nullptr) Uw[tile] = wbase - tile * BK;
      atomicAdd(hist + u, 1ull);
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(la.ticket, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  last_cta_order(la, s_warp);
  if (threadIdx.x == 0) *la.ticket = 0u;
}

template <int MJ>
spamm_status fused_t(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s) {
  const int64_t n_macro = (gi1 - gi0) * p.GN;
  const int64_t blocks = n_macro > 0 ? (n_macro + kWarps - 1) / kWarps : 1;
  LastArgs la{p.hist, p.bucket_pos, p.BK + 1, p.U, p.L, p.order, gi0 * p.GN, gi1 * p.GN, p.totals, p.ticket};
  skip_fused_kernel<kMacroI, MJ><<<static_cast<unsigned>(blocks), kWarps * 32, 0, s>>>(
      p.nA, p.nBt, p.BM, p.BK, p.BN, p.tau, p.GN, gi0, n_macro, p.V, p.U, p.L,
      reinterpret_cast<unsigned long long*>(p.row_work), reinterpret_cast<unsigned long long*>(p.hist),
      p.leaf_start, p.leaf_k, p.macro_ent, p.macro_run, p.Uw != p.U ? p.Uw : nullptr,
      static_cast<int>(p.Uw != p.U && p.N % 32 == 0), la);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

constexpr int64_t kSmallScan = int64_t(1) << 15;   // macro-tile counts scanned inside the count kernel

template <int MJ>
spamm_status count_t(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s, const ScanArgs& sa) {
  const int64_t n_macro = (gi1 - gi0) * p.GN;
  const int64_t blocks = n_macro > 0 ? (n_macro + kWarps - 1) / kWarps : 1;
  skip_count_kernel<kMacroI, MJ><<<static_cast<unsigned>(blocks), kWarps * 32, 0, s>>>(
      p.nA, p.nBt, p.BM, p.BK, p.BN, p.tau, p.GN, gi0, n_macro, p.V, p.U, p.L,
      reinterpret_cast<unsigned long long*>(p.row_work), reinterpret_cast<unsigned long long*>(p.hist), sa);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

template <int MJ>
spamm_status emit_t(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s) {
  const int64_t n_macro = (gi1 - gi0) * p.GN;
  if (n_macro <= 0) return SPAMM_OK;
  const int64_t blocks = (n_macro + kWarps - 1) / kWarps;
  skip_emit_kernel<kMacroI, MJ><<<static_cast<unsigned>(blocks), kWarps * 32, 0, s>>>(
      p.nA, p.nBt, p.BM, p.BK, p.BN, p.tau, p.GN, gi0, n_macro, p.V, p.leaf_base, p.macro_ptr, p.U,
      reinterpret_cast<unsigned long long*>(p.bucket_pos), p.leaf_start, p.leaf_k, p.macro_ent, p.macro_run,
      p.order);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

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
  // row_work [BM], hist [BK+2] and totals [2] are contiguous in one allocation (see api.cu)
  SPAMM_CUDA_TRY(cudaMemsetAsync(p.row_work, 0, sizeof(int64_t) * (p.BM + p.BK + 4), s));
  // Out-of-range macro-tiles (multi-GPU shards) have U = L = 0 and are not in the histogram.
  const bool small = nmac <= kSmallScan;
  ScanArgs sa{p.U, p.macro_ptr, p.L, p.leaf_base, small ? nmac : 0, p.hist, p.bucket_pos, p.BK + 1,
              small ? p.ticket : nullptr};
  if (p.MJ == kMacroJ_umma) {
    SPAMM_TRY(count_t<kMacroJ_umma>(p, gi0, gi1, s, sa));
  } else {
    SPAMM_TRY(count_t<kMacroJ_simt>(p, gi0, gi1, s, sa));
  }
  if (!small) {
    size_t bytes = p.cub_tmp_bytes;
    SPAMM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(p.cub_tmp, bytes, p.U, p.macro_ptr, nmac + 1, s));
    bytes = p.cub_tmp_bytes;
    SPAMM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(p.cub_tmp, bytes, p.L, p.leaf_base, nmac + 1, s));
    sa.ticket = nullptr;
    skip_scan_kernel<<<1, 1024, 0, s>>>(sa);
    count_launch();
    SPAMM_CUDA_TRY(cudaGetLastError());
  }
  SPAMM_CUDA_TRY(cudaMemcpyAsync(p.totals, p.leaf_base + nmac, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  SPAMM_CUDA_TRY(cudaMemcpyAsync(p.totals + 1, p.macro_ptr + nmac, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  return SPAMM_OK;
}

// fixed-region single pass (requires worst-case list storage, p.fixed_regions)
spamm_status launch_skipmap_fused(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s) {
  const int64_t nleaf = p.BM * p.BN, nmac = p.GM * p.GN;
  const bool partial = gi0 != 0 || gi1 != p.GM;
  if (partial) {
    SPAMM_CUDA_TRY(cudaMemsetAsync(p.V, 0, sizeof(int64_t) * (nleaf + 1), s));
    SPAMM_CUDA_TRY(cudaMemsetAsync(p.U, 0, sizeof(int64_t) * (nmac + 1), s));
    SPAMM_CUDA_TRY(cudaMemsetAsync(p.L, 0, sizeof(int64_t) * (nmac + 1), s));
  }
  // row_work [BM], hist [BK+2] and totals [2] are contiguous in one allocation (see api.cu)
  SPAMM_CUDA_TRY(cudaMemsetAsync(p.row_work, 0, sizeof(int64_t) * (p.BM + p.BK + 4), s));
  if (p.MJ == kMacroJ_umma) return fused_t<kMacroJ_umma>(p, gi0, gi1, s);
  return fused_t<kMacroJ_simt>(p, gi0, gi1, s);
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
