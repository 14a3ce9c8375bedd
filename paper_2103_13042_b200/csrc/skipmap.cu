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

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

#include "internal.h"

namespace spamm {
namespace {

constexpr int kWarps = 8;

// keep bits of one k-step of a macro-tile: bit li*MJ+lj; 64-bit for 8 x 8 macro-tiles
template <int MI, int MJ>
using mask_t = typename std::conditional<(MI * MJ > 32), unsigned long long, uint32_t>::type;

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
__device__ __forceinline__ mask_t<MI, MJ> chunk_mask(const ChunkVals<MI, MJ>& v, mask_t<MI, MJ> valid, double tau) {
  using M_ = mask_t<MI, MJ>;
  // Exact pre-filters: norms are >= 0 (or NaN) and rounding is monotone, so
  //   max(a) * max(b) < tau   =>  every a*b < tau   (NaN-propagating maxima keep NaN pairs);
  //   min(a) * min(b) >= tau  =>  every a*b >= tau  (NaN pairs are kept either way).
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
  if (!v.kin || valid == 0u || __dmul_rn(amax, bmax) < tau) return 0u;
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
  if (mask == 0xFFFFFFFFu)   // all 4 x 8 pairs kept: one run j0 = 0, len = 8, pattern 1111
    return make_uint4(k | (1u << 16) | (0xFFu << 24), 0u | (7u << 3) | (15u << 6), 0u, wide << 31);
  // bit lj of bnd: column lj's 4-bit pattern differs from column lj+1's (any row byte differs);
  // bit lj of nz: column lj has a kept pair.  Runs = maximal segments between boundaries
  // whose columns are non-zero (same result as walking the columns, a fraction of the ops).
  const uint32_t d = (mask ^ (mask >> 1)) & 0x7F7F7F7Fu;
  const uint32_t bnd = (d | (d >> 8) | (d >> 16) | (d >> 24)) & 0x7Fu;
  const uint32_t nz = (mask | (mask >> 8) | (mask >> 16) | (mask >> 24)) & 0xFFu;
  // runs 0-2 -> w0, 3-5 -> w1, 6-7 -> w2, 10 bits each (explicit registers: a dynamically indexed
  // array would live in local memory)
  uint32_t w0 = 0u, w1 = 0u, w2 = 0u;
  uint32_t nr = 0, cols = 0, sh = 0;
  uint32_t j = 0;
  while (j < 8) {
    const uint32_t b = bnd >> j;
    const uint32_t j1 = b ? j + static_cast<uint32_t>(__ffs(b)) : 8u;
    if ((nz >> j) & 1u) {
      const uint32_t pat = col_pattern8(mask, static_cast<int>(j));
      const uint32_t run = (j | ((j1 - j - 1) << 3) | (pat << 6)) << sh;
      if (nr < 3) w0 |= run;
      else if (nr < 6) w1 |= run;
      else w2 |= run;
      ++nr;
      sh = sh == 20u ? 0u : sh + 10u;
      cols |= ((1u << (j1 - j)) - 1u) << j;
    }
    j = j1;
  }
  return make_uint4(k | (nr << 16) | (cols << 24), w0, w1, w2 | (wide << 31));
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
  unsigned long long* tstamp;   // debug (SPAMM_DEBUG_SKIP_PROF): [0] first CTA start, [1] last CTA enter, [2] exit
  unsigned int* sched;          // the multiply's claim counters [4], zeroed by the last CTA
};
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long g;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
  return g;
}

// Bucket starts live in shared memory when they fit (atomics there are ~10x cheaper than
// global ones, and this loop is the serial tail of the launch).
constexpr int kSmemBuckets = 2048;
__device__ void last_cta_order(const LastArgs& la, int64_t* s_warp, unsigned long long* s_pos) {
  block_scan_array(la.hist, la.bucket_pos, la.nbucket, true, s_warp);
  __syncthreads();
  const bool in_smem = la.nbucket <= kSmemBuckets;
  unsigned long long* pos = in_smem ? s_pos : reinterpret_cast<unsigned long long*>(la.bucket_pos);
  if (in_smem)
    for (int64_t b = threadIdx.x; b < la.nbucket; b += blockDim.x) s_pos[b] = static_cast<unsigned long long>(la.bucket_pos[b]);
  __syncthreads();
  constexpr int R = 8;   // independent loads / atomics in flight per thread
  int64_t kept = 0, ents = 0;
  for (int64_t base = la.t0; base < la.t1; base += static_cast<int64_t>(blockDim.x) * R) {
    int64_t u[R], l[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t t = base + static_cast<int64_t>(r) * blockDim.x + threadIdx.x;
      u[r] = t < la.t1 ? la.U[t] : -1;
      l[r] = t < la.t1 ? la.L[t] : 0;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (u[r] < 0) continue;
      const int64_t t = base + static_cast<int64_t>(r) * blockDim.x + threadIdx.x;
      const unsigned long long slot = atomicAdd(pos + u[r], 1ull);
      la.order[slot] = static_cast<int32_t>(t);
      kept += l[r];
      ents += u[r];
    }
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

// One CTA per macro-tile: warp w evaluates k = kb + 32 w + lane of each 256-wide k block,
// so a macro-tile's MI x MJ x 256 keep bits are decided by 256 threads at once.  Per-warp
// counts (k-steps, tensor-path entries) are scanned across the 8 warps in shared memory,
// then every warp writes its part of the ascending macro lists.  Only the macro-level
// lists -- (k, keep mask) per k-step, which hold every keep bit -- are written here; the
// per-C-tile k lists are expanded from them on request (leaf_expand_kernel).  Row work
// and kept-pair counts are popcounts of the masks.
constexpr int kFusedWarps = 8;
constexpr int kKB = 32 * kFusedWarps;   // k per block: thread (w, lane) owns k = kb + 32 w + lane
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <int MI, int MJ>
__global__ void __launch_bounds__(kFusedWarps * 32, (MI + MJ > 12) ? 3 : 4)
    skip_fused_kernel(const double* __restrict__ nA, const double* __restrict__ nBt, int64_t BM, int64_t BK,
                      int64_t BN, double tau, int64_t GN, int64_t gi0, int64_t n_macro, int64_t* __restrict__ U,
                      int64_t* __restrict__ Lm, unsigned long long* __restrict__ row_work,
                      unsigned long long* __restrict__ hist, void* __restrict__ macro_ent_v,
                      uint4* __restrict__ macro_run, int64_t* __restrict__ Uw, int merge_ok, LastArgs la) {
  using M_ = mask_t<MI, MJ>;
  constexpr bool kMask64 = MI * MJ > 32;  // 8 x 8 tiles: 64-bit masks, (k, mask_lo, mask_hi, 0) entries
  constexpr int kRunStride = kMask64 ? 2 : 1;   // tensor-path region per macro-tile: kRunStride * BK entries
  constexpr int W = kFusedWarps;
  constexpr int R = MI + MJ;              // norm rows per macro-tile: MI of A, MJ of B^T
  __shared__ uint32_t s_cm[W], s_cr[W], s_rw[W][MI];
  __shared__ int64_t s_warp[33];
  __shared__ int s_last;
  // dynamic: each thread's own norm column, double-buffered [2][R][kKB]; reused by the
  // last CTA for the bucket positions (kSmemBuckets <= 2 * R * kKB)
  extern __shared__ double s_dyn[];
  double(*s_val)[R][kKB] = reinterpret_cast<double(*)[R][kKB]>(s_dyn);
  unsigned long long* s_pos = reinterpret_cast<unsigned long long*>(s_dyn);
  static_assert(kSmemBuckets <= 2 * R * kKB, "bucket array must fit the staging buffer");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = threadIdx.x;
  if (la.tstamp && threadIdx.x == 0) atomicMin(la.tstamp, gtimer());
  // stage the norms of unit (macro-tile mm, k block kk) for this thread's column
  auto stage = [&](int64_t mm, int64_t kk, int buf) {
    if (mm < n_macro) {
      const int64_t I = gi0 + mm / GN, J = mm % GN;
      const int64_t k = kk + col;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const bool isA = r < MI;
        const int64_t row = isA ? I * MI + r : J * MJ + (r - MI);
        const bool ok = k < BK && row < (isA ? BM : BN);
        if (ok)
          cp_async8(&s_val[buf][r][col], (isA ? nA : nBt) + row * BK + k);
        else
          s_val[buf][r][col] = 0.0;   // out of range loads as 0 and is masked by index
      }
    }
    cp_async_commit();
  };
  // Persistent CTAs walk (macro-tile, k block) units; the next unit's norms are in flight
  // while the current one is decided.
  int64_t m = blockIdx.x, kb = 0;
  int buf = 0;
  stage(m, kb, 0);
  int64_t mbase = 0, wbase = 0;
  uint32_t rw[MI];
  const uint32_t lt = (1u << lane) - 1u;
  while (m < n_macro) {
    int64_t nm = m, nk = kb + kKB;
    if (nk >= BK) {
      nm = m + gridDim.x;
      nk = 0;
    }
    const long long c0 = clock64();
    stage(nm, nk, buf ^ 1);
    cp_async_wait1();
    const long long c1 = clock64();
    const int64_t I = gi0 + m / GN, J = m % GN;
    const int64_t tile = I * GN + J;
    const M_ valid = valid_bits<MI, MJ>(BM, BN, I, J);
    if (kb == 0) {
      mbase = tile * BK;                    // macro-tile region
      wbase = tile * BK * kRunStride;       // tensor-path entries
#pragma unroll
      for (int li = 0; li < MI; ++li) rw[li] = 0u;
    }
    const int64_t k = kb + col;
    ChunkVals<MI, MJ> cv;
    cv.kin = k < BK;
#pragma unroll
    for (int li = 0; li < MI; ++li) cv.a[li] = s_val[buf][li][col];
#pragma unroll
    for (int lj = 0; lj < MJ; ++lj) cv.b[lj] = s_val[buf][MI + lj][col];
    const M_ mask = chunk_mask<MI, MJ>(cv, valid, tau);
#pragma unroll
    for (int li = 0; li < MI; ++li)
      rw[li] += static_cast<uint32_t>(__popcll(static_cast<unsigned long long>(mask >> (li * MJ)) & ((1ull << MJ) - 1ull)));
    const uint32_t any = __ballot_sync(0xffffffffu, mask != 0u);
    // tensor-path entries: k-tiles 2p and 2p+1 with the same non-zero mask become one
    // 64-deep k-step
    bool wide = false;
    uint32_t ne = 0;
    if (MJ == 8 && macro_run != nullptr) {
      const M_ mnext = __shfl_down_sync(0xffffffffu, mask, 1);
      const M_ mprev = __shfl_up_sync(0xffffffffu, mask, 1);
      const bool even = (lane & 1) == 0;
      wide = merge_ok && even && mask != 0u && mnext == mask;
      const bool absorbed = merge_ok && !even && mask != 0u && mprev == mask;
      if (mask != 0u && !absorbed) {
        ne = 1u;
      }
    }
    uint32_t ie = ne;   // inclusive warp scan of entry counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, ie, o);
      if (lane >= o) ie += y;
    }
    if (lane == 0) s_cm[warp] = __popc(any);
    if (lane == 31) s_cr[warp] = ie;
    __syncthreads();
    uint32_t om = 0, orr = 0, tm = 0, tr = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t cm = s_cm[w], cr = s_cr[w];
      if (w < warp) {
        om += cm;
        orr += cr;
      }
      tm += cm;
      tr += cr;
    }
    if (mask) {
      if constexpr (kMask64)
        reinterpret_cast<uint4*>(macro_ent_v)[mbase + om + __popc(any & lt)] =
            make_uint4(static_cast<uint32_t>(k), static_cast<uint32_t>(mask), static_cast<uint32_t>(mask >> 32), 0u);
      else
        reinterpret_cast<uint2*>(macro_ent_v)[mbase + om + __popc(any & lt)] =
            make_uint2(static_cast<uint32_t>(k), static_cast<uint32_t>(mask));
    }
    for (uint32_t q = 0; q < ne; ++q) {
      const int64_t at = wbase + orr + (ie - ne) + q;
      if constexpr (kMask64) {   // 256 x 256 two-issuer path: the 4 x 8 runs of each half, entries 2 * at, +1
        const int64_t at2 = wbase + 2 * (orr + (ie - ne) + q);
        macro_run[at2] = encode_runs(static_cast<uint32_t>(k), static_cast<uint32_t>(mask), wide ? 1u : 0u);
        macro_run[at2 + 1] = encode_runs(static_cast<uint32_t>(k), static_cast<uint32_t>(mask >> 32), wide ? 1u : 0u);
      } else
        macro_run[at] = encode_runs(static_cast<uint32_t>(k), static_cast<uint32_t>(mask), wide ? 1u : 0u);
    }
    mbase += tm;
    wbase += kMask64 ? 2 * tr : tr;
    if (kb + kKB >= BK) {   // last k block of the macro-tile: counts
#pragma unroll
      for (int li = 0; li < MI; ++li) {
        uint32_t v = rw[li];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) s_rw[warp][li] = v;
      }
      __syncthreads();
      if (warp == 0) {
        uint32_t r = 0;   // lane li < MI: kept pairs of tile row I*MI + li
        if (lane < MI)
#pragma unroll
          for (int w = 0; w < W; ++w) r += s_rw[w][lane];
        if (lane < MI && I * MI + lane < BM && r)
          atomicAdd(row_work + I * MI + lane, static_cast<unsigned long long>(r));
        uint32_t lsum = r;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        if (lane == 0) {
          const uint32_t u = static_cast<uint32_t>(mbase - tile * BK);
          Lm[tile] = lsum;
          U[tile] = u;
          if (Uw != nullptr) Uw[tile] = wbase - tile * BK * kRunStride;
          atomicAdd(hist + u, 1ull);
        }
      }
    }
    __syncthreads();   // s_cm / s_cr / s_rw and this buffer are rewritten next
    if (la.tstamp && threadIdx.x == 0) {
      atomicAdd(la.tstamp + 3, static_cast<unsigned long long>(c1 - c0));
      atomicAdd(la.tstamp + 4, static_cast<unsigned long long>(clock64() - c1));
      atomicAdd(la.tstamp + 5, 1ull);
    }
    m = nm;
    kb = nk;
    buf ^= 1;
  }
  const long long cf0 = clock64();
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(la.ticket, 1u);
    s_last = (t == gridDim.x - 1);
    if (la.tstamp) {
      atomicAdd(la.tstamp + 6, static_cast<unsigned long long>(clock64() - cf0));
      atomicMax(la.tstamp + 7, gtimer());
    }
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  asm volatile("cp.async.wait_all;" ::: "memory");   // the staging buffer becomes s_pos
  __syncthreads();
  if (la.tstamp && threadIdx.x == 0) la.tstamp[1] = gtimer();
  last_cta_order(la, s_warp, s_pos);
  if (threadIdx.x == 0) *la.ticket = 0u;
  if (threadIdx.x < 4 && la.sched) la.sched[threadIdx.x] = 0u;
  if (la.tstamp) {
    __syncthreads();
    if (threadIdx.x == 0) la.tstamp[2] = gtimer();
  }
}

// Per-C-tile k lists (fixed regions: C tile (i,j) owns slots [(i*BN+j)*BK, +V)) expanded
// from the macro lists: one warp per macro-tile, lane b appends the k-steps whose mask has
// bit b -- ascending k, exactly the skip map the fused pass decided.
template <int MI, int MJ>
__global__ void __launch_bounds__(kWarps * 32)
    leaf_expand_kernel(int64_t BM, int64_t BK, int64_t BN, int64_t GN, int64_t gi0, int64_t n_macro,
                       const int64_t* __restrict__ U, const void* __restrict__ macro_ent_v, int64_t* __restrict__ V,
                       int64_t* __restrict__ leaf_start, uint16_t* __restrict__ leaf_k) {
  constexpr int NB = MI * MJ;
  constexpr int NL = (NB + 31) / 32;   // leaves per lane
  using M_ = mask_t<MI, MJ>;
  const int lane = threadIdx.x & 31;
  const int64_t m = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  if (m >= n_macro) return;
  const int64_t I = gi0 + m / GN, J = m % GN;
  const int64_t tile = I * GN + J;
  const M_ valid = valid_bits<MI, MJ>(BM, BN, I, J);
  int64_t n[NL], lstart[NL], leaf[NL];
  bool vl[NL];
#pragma unroll
  for (int h = 0; h < NL; ++h) {
    const int b = lane + 32 * h;
    vl[h] = b < NB && ((valid >> b) & 1u);
    leaf[h] = (I * MI + b / MJ) * BN + (J * MJ + b % MJ);
    lstart[h] = leaf[h] * BK;
    n[h] = 0;
  }
  const int64_t u = U[tile];
  for (int64_t e0 = 0; e0 < u; e0 += 32) {
    const int64_t e = tile * BK + e0 + lane;
    uint32_t mk = 0u;
    M_ mm = 0u;
    if (e0 + lane < u) {
      if constexpr (NB > 32) {
        const uint4 x = reinterpret_cast<const uint4*>(macro_ent_v)[e];
        mk = x.x;
        mm = static_cast<M_>(x.y) | (static_cast<M_>(x.z) << 32);
      } else {
        const uint2 x = reinterpret_cast<const uint2*>(macro_ent_v)[e];
        mk = x.x;
        mm = x.y;
      }
    }
    const int cnt = static_cast<int>(u - e0 < 32 ? u - e0 : 32);
    for (int q = 0; q < cnt; ++q) {
      const uint32_t k = __shfl_sync(0xffffffffu, mk, q);
      const M_ mask = __shfl_sync(0xffffffffu, mm, q);
#pragma unroll
      for (int h = 0; h < NL; ++h)
        if (vl[h] && ((mask >> (lane + 32 * h)) & 1u)) leaf_k[lstart[h] + n[h]++] = static_cast<uint16_t>(k);
    }
  }
#pragma unroll
  for (int h = 0; h < NL; ++h)
    if (vl[h]) {
      V[leaf[h]] = n[h];
      leaf_start[leaf[h]] = lstart[h];
    }
}

template <int MI, int MJ>
spamm_status fused_t(Plan& p, int64_t gi0, int64_t gi1, cudaStream_t s) {
  const int64_t n_macro = (gi1 - gi0) * p.GN;
  // resident CTAs per SM: the staging buffer is 2 x (MI + MJ) x 256 doubles (48 KB for 4 x 8, 64 KB for 8 x 8)
  constexpr int kPerSm = (MI + MJ > 12) ? 3 : 4;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(n_macro, static_cast<int64_t>(p.num_sms) * kPerSm));
  static unsigned long long* tst = nullptr;
  if (getenv("SPAMM_DEBUG_SKIP_PROF") && !tst) cudaMalloc(&tst, 128);
  if (tst) {
    const unsigned long long init[12] = {~0ull, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyAsync(tst, init, sizeof(init), cudaMemcpyHostToDevice, s);
  }
  LastArgs la{p.hist, p.bucket_pos, p.BK + 1, p.U, p.L, p.order, gi0 * p.GN, gi1 * p.GN, p.totals, p.ticket, tst, p.sched};
  constexpr int dyn = 2 * (MI + MJ) * kKB * static_cast<int>(sizeof(double));
  static bool attr = false;
  if (!attr) {
    SPAMM_CUDA_TRY(cudaFuncSetAttribute(skip_fused_kernel<MI, MJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    attr = true;
  }
  skip_fused_kernel<MI, MJ><<<static_cast<unsigned>(blocks), kFusedWarps * 32, dyn, s>>>(
      p.nA, p.nBt, p.BM, p.BK, p.BN, p.tau, p.GN, gi0, n_macro, p.U, p.L,
      reinterpret_cast<unsigned long long*>(p.row_work), reinterpret_cast<unsigned long long*>(p.hist),
      p.macro_ent, p.macro_run, p.Uw != p.U ? p.Uw : nullptr, static_cast<int>(p.Uw != p.U && p.N % 32 == 0), la);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  if (tst) {
    unsigned long long h[12];
    cudaMemcpyAsync(h, tst, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "[skip prof] main part %.2f us, last-CTA order pass %.2f us; per unit: wait %.0f cyc, work %.0f cyc "
            "(%llu units); per CTA fence+ticket %.0f cyc; last ticket at +%.2f us\n", (h[1] - h[0]) * 1e-3,
            (h[2] - h[1]) * 1e-3, double(h[3]) / h[5], double(h[4]) / h[5], h[5], double(h[6]) / blocks,
            (h[7] - h[0]) * 1e-3);
  }
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
  if (!p.ws_zeroed) SPAMM_CUDA_TRY(cudaMemsetAsync(p.row_work, 0, sizeof(int64_t) * (p.BM + p.BK + 4), s));
  p.ws_zeroed = false;
  p.sched_zeroed = true;   // the last CTA zeroes the multiply's claim counters
  if (p.MI == kMacroI_dual) return fused_t<kMacroI_dual, kMacroJ_umma>(p, gi0, gi1, s);
  if (p.MJ == kMacroJ_umma) return fused_t<kMacroI, kMacroJ_umma>(p, gi0, gi1, s);
  return fused_t<kMacroI, kMacroJ_simt>(p, gi0, gi1, s);
}

spamm_status launch_leaf_expand(Plan& p, cudaStream_t s) {
  const int64_t gi0 = p.row_begin_macro, gi1 = p.row_end_macro;
  const int64_t nleaf = p.BM * p.BN;
  if (gi0 != 0 || gi1 != p.GM) SPAMM_CUDA_TRY(cudaMemsetAsync(p.V, 0, sizeof(int64_t) * (nleaf + 1), s));
  const int64_t n_macro = (gi1 - gi0) * p.GN;
  if (n_macro <= 0) return SPAMM_OK;
  const int64_t blocks = (n_macro + kWarps - 1) / kWarps;
  if (p.MI == kMacroI_dual)
    leaf_expand_kernel<kMacroI_dual, kMacroJ_umma><<<static_cast<unsigned>(blocks), kWarps * 32, 0, s>>>(
        p.BM, p.BK, p.BN, p.GN, gi0, n_macro, p.U, p.macro_ent, p.V, p.leaf_start, p.leaf_k);
  else if (p.MJ == kMacroJ_umma)
    leaf_expand_kernel<kMacroI, kMacroJ_umma><<<static_cast<unsigned>(blocks), kWarps * 32, 0, s>>>(
        p.BM, p.BK, p.BN, p.GN, gi0, n_macro, p.U, p.macro_ent, p.V, p.leaf_start, p.leaf_k);
  else
    leaf_expand_kernel<kMacroI, kMacroJ_simt><<<static_cast<unsigned>(blocks), kWarps * 32, 0, s>>>(
        p.BM, p.BK, p.BN, p.GN, gi0, n_macro, p.U, p.macro_ent, p.V, p.leaf_start, p.leaf_k);
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
