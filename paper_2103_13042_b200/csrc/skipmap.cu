// skipmap.cu -- stage 2: the per-C-tile skip map (Alg. 2 lines 3-16, PAPER.md:152-172;
// valid-multiplication counts V, Sec. 3.5.1).
//
// keep(i,k,j)  <=>  !(nA[i][k] * nB[k][j] < tau)   in float64 (">= tau", PAPER.md:47/63/155;
// NaN kept, reading R2).
//
// B200 design: the map is materialised once, globally, as macro-level lists (the paper builds a
// bitmap + map_offset per CUDA block inside the multiply):
//   pyramid : per macro row I (MI tile rows) and k chunk c (32 k-tiles) the max and min of nA over
//             the MI x 32 tiles, and the same per macro column J over nB -- one level of Eq. 1's
//             quadtree above the leaves, aligned with the schedule's macro-tiles;
//   skip map: per macro-tile (I, J) the chunks are classified from the pyramid alone, exactly:
//               max_A * max_B <  tau  =>  every pair of the chunk skipped (rounding is monotone;
//                                         NaN maxima never skip)
//               min_A * min_B >= tau  =>  every pair kept (NaN pairs are kept anyway)
//             and only the remaining "mixed" chunks load their MI + MJ norms per k and test the
//             MI x MJ products.  The work is output-sensitive: a banded product touches a band
//             of chunks instead of all BM x BK x BN triples.  One warp decides one chunk
//             (lane = k); the 8 warps of a CTA take 8 surviving chunks at a time in ascending k
//             and write, at offsets scanned across the warps, the macro-tile's (k, keep mask)
//             list and, for the tensor path, each k-step's MMA runs pre-decoded per 128-row half;
//   order   : the main loop appends every macro-tile to a work or an empty list and counts two
//             histograms (LPT key BK - U; super-block); a grid-wide scatter kernel places the
//             work list by bucket (a bucket sort, no comparison sort) and appends the empty tiles:
//             the multiply's claim order, plus the totals (kept pairs, k-steps).
// Row work (Sec. 3.5.1's V summed over a row) and kept counts are popcounts of the masks.
// The per-C-tile k lists are expanded from the macro lists only on request (leaf_expand).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <type_traits>

#include "internal.h"
#include "skipdecide.cuh"
#include "sm100.cuh"

namespace spamm {
namespace {

constexpr int kWarps = 8;

// Runs of a 4 x 8 keep mask for the tensor path: adjacent C-tile columns with the same
// non-zero 4-bit row pattern.  run = j0 | (len-1) << 3 | pat << 6  (10 bits, 3 per word).
__device__ __forceinline__ uint32_t col_pattern8(uint32_t mask, int lj) {
  return ((mask >> lj) & 1u) | (((mask >> (8 + lj)) & 1u) << 1) | (((mask >> (16 + lj)) & 1u) << 2) |
         (((mask >> (24 + lj)) & 1u) << 3);
}
// x = k | #runs << 16 | needed columns << 24; runs in y, z, w (bits 0-19 of w; the multiply
// keeps its stage flags in w's top bits)
__device__ __forceinline__ uint4 encode_runs(uint32_t k, uint32_t mask) {
  if (mask == 0xFFFFFFFFu)   // all 4 x 8 pairs kept: one run j0 = 0, len = 8, pattern 1111
    return make_uint4(k | (1u << 16) | (0xFFu << 24), 0u | (7u << 3) | (15u << 6), 0u, 0u);
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
  return make_uint4(k | (nr << 16) | (cols << 24), w0, w1, w2);
}

// NaN-propagating max (any NaN -> NaN) and NaN-ignoring min, the pyramid's reductions
__device__ __forceinline__ double max_nan(double a, double b) { return (a != a || b != b) ? (a + b) : fmax(a, b); }

// ------------------------------------------------------------------ norm pyramid
// One warp per (group g, chunk c): groups 0..GM-1 are macro rows of nA (MI rows each), groups
// GM..GM+GN-1 macro columns of nB^T (MJ rows each); lane = k offset in the chunk.  Tiles past
// BM / BN / BK do not exist and are left out of both reductions.
template <int MI, int MJ>
__global__ void __launch_bounds__(256)
    pyramid_kernel(const double* __restrict__ nA, const double* __restrict__ nBt, int64_t BM, int64_t BK, int64_t BN,
                   int64_t GM, int64_t GN, int64_t NC, double* __restrict__ pyr) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  sm100::pdl_wait();
  sm100::pdl_trigger();
  if (w >= (GM + GN) * NC) return;
  const int64_t g = w / NC, c = w % NC;
  const bool isA = g < GM;
  const int R = isA ? MI : MJ;
  const int64_t row0 = (isA ? g : g - GM) * R, nrows = isA ? BM : BN;
  const double* __restrict__ src = isA ? nA : nBt;
  const int64_t k = c * kChunk + lane;
  double mx = 0.0, mn = INFINITY;
  for (int r = 0; r < R; ++r) {
    const int64_t row = row0 + r;
    if (row < nrows && k < BK) {
      const double v = __ldg(src + row * BK + k);
      mx = max_nan(mx, v);
      mn = fmin(mn, v);
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    mx = max_nan(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  if (lane == 0) {
    double* base = isA ? pyr + g * NC : pyr + 2 * GM * NC + (g - GM) * NC;
    const int64_t half = isA ? GM * NC : GN * NC;
    base[c] = mx;
    base[half + c] = mn;
  }
}

// Exclusive scan of n int64 values by one CTA; out has n+1 entries, out[n] = total.
// If reverse, out[u] = sum_{u' > u} in[u'] (descending buckets).  in / out may alias.
__device__ void block_scan_array(const int64_t* in, int64_t* out, int64_t n, bool reverse, int64_t* s_warp) {
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
  __syncthreads();
}

struct OrderArgs {
  int64_t* hist;         // [BK + 2] LPT bucket counts (key BK - U)
  int64_t* hist_sb;      // [NSB] super-block bucket counts
  int64_t* bucket_cnt;   // [max(BK + 2, NSB + 1)] slots taken per bucket (zeroed with the workspace)
  int64_t* bucket_pos;   // [max(BK + 2, NSB + 1)] bucket starts (only when they exceed shared memory)
  unsigned long long* sb_bits;   // [NSB][kSbWords] working tiles of each super-block (row-major bit)
  int64_t nsb;
  const int64_t* U;
  const int64_t* L;
  int64_t BK, GN;
  int num_sms;
  int32_t* work;         // [GM*GN] macro-tiles with kept pairs
  int32_t* empty;        // [GM*GN] macro-tiles without kept pairs
  unsigned int* cnt;     // [0] work-list length, [1] empty-list length, [2] skip-map tile claims
  int32_t* order;
  int64_t* totals;       // [0] kept pairs, [1] macro entries, [2] macro-tiles without kept pairs
  unsigned int* sched;   // the multiply's claim counters [4]
  const int64_t* d_range;   // multi-GPU: range [d_range[0], d_range[1]) of macro rows, else t0 / t1
  int64_t t0, t1;
};
constexpr int kSmemBuckets = 4096;
constexpr int64_t kInlineOrderTiles = 4096;   // ranges up to this many macro-tiles: order by the last CTA
constexpr uint32_t kOrdR = SPAMM_ORD_R, kOrdC = SPAMM_ORD_C;   // super-block of kOrdR x kOrdC macro-tiles
constexpr int64_t kSbWords = (kOrdR * kOrdC + 63) / 64;        // 64-bit words of a super-block's tile mask

// warp-aggregated atomicAdd of 1 per lane on cnt[key]: lanes with equal keys share one atomic;
// returns each lane's old value + its rank among the equal lanes
template <typename T>
__device__ __forceinline__ T agg_inc(T* cnt, int64_t key, bool active) {
  const unsigned act = __ballot_sync(0xffffffffu, active);
  if (!active) return 0;
  const unsigned peers = __match_any_sync(act, static_cast<unsigned long long>(key));
  const int leader = __ffs(peers) - 1;
  const int lane = threadIdx.x & 31;
  T base = 0;
  if (lane == leader) base = atomicAdd(cnt + key, static_cast<T>(__popc(peers)));
  base = __shfl_sync(peers, base, leader);
  return base + static_cast<T>(__popc(peers & ((1u << lane) - 1u)));
}

// super-block of macro-tile t in the range starting at tile t0 (32-bit arithmetic: tile ids < 2^31)
__device__ __forceinline__ int64_t sb_of(int64_t t, int64_t t0, int64_t GN) {
  const uint32_t gn = static_cast<uint32_t>(GN), nsbc = (gn + kOrdC - 1) / kOrdC;
  const uint32_t rel = static_cast<uint32_t>(t - t0), row0 = static_cast<uint32_t>(t0) / gn;
  const uint32_t li = rel / gn, lj = (static_cast<uint32_t>(t) - row0 * gn - li * gn);
  return static_cast<int64_t>((li / kOrdR) * nsbc + lj / kOrdC);
}

// bit of macro-tile t inside its super-block (row-major position)
__device__ __forceinline__ uint32_t sb_pos(int64_t t, int64_t t0, int64_t GN) {
  const uint32_t gn = static_cast<uint32_t>(GN);
  const uint32_t li = static_cast<uint32_t>(t - t0) / gn, lj = static_cast<uint32_t>(t % GN);
  return (li % kOrdR) * kOrdC + lj % kOrdC;
}
__device__ __forceinline__ void mark_working(const OrderArgs& oa, int64_t t, int64_t t0) {
  const uint32_t b = sb_pos(t, t0, oa.GN);
  atomicOr(oa.sb_bits + sb_of(t, t0, oa.GN) * kSbWords + b / 64, 1ull << (b % 64));
}

__device__ __forceinline__ void order_range(const OrderArgs& oa, int64_t& t0, int64_t& t1) {
  t0 = oa.t0;
  t1 = oa.t1;
  if (oa.d_range) {
    t0 = oa.d_range[0] * oa.GN;
    t1 = oa.d_range[1] * oa.GN;
  }
}

// The multiply's claim order of the macro-tiles of the range (a parallel bucket sort):
//   * few tiles per CTA (n_work < 16 per SM): longest processing time first -- key BK - U, so the
//     long tiles start first and the short ones fill the tail (Sec. 3.5.1's balance goal);
//   * many tiles per CTA (balance is free): by super-block of kOrdR x kOrdC macro-tiles, row-major,
//     default bands of 6 macro rows walked column by column: the tiles claimed together share a B
//     column strip and start their k-lists within a few k-steps of each other (on a band, the first
//     kept k moves by 4 k-tiles per macro row), so their operand loads hit in L2.  Measured at
//     N = 65536 (DRAM reads of the multiply / its time): 12 x 12 blocks 266 GB / 66 ms, 8 x 8 170 GB,
//     6 x 6 115 GB / 60 ms, 6 x 1 58 ms; ordering by the first kept k instead put tiles of one
//     anti-diagonal -- no shared strips -- in flight together: 645 GB / 103 ms;
//   * macro-tiles without kept pairs last (zero-filled by the multiply).
// The skip map's main loop appends the tiles to a work or an empty list and counts both
// histograms; order_lists_kernel does that from U instead on the multi-GPU final pass (part of the
// range was decided by the provisional launch).  order_scatter_kernel: every CTA scans the chosen
// histogram into shared memory and places its share of the work list with one atomic per bucket
// and lane group (global per-bucket counters).  Ties (same bucket) are in arbitrary order.
__global__ void __launch_bounds__(256) order_lists_kernel(const OrderArgs oa) {
  sm100::pdl_wait();
  sm100::pdl_trigger();
  int64_t t0, t1;
  order_range(oa, t0, t1);
  int64_t kept = 0, ents = 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t base = t0 + static_cast<int64_t>(blockIdx.x) * blockDim.x; base < t1; base += stride) {
    const int64_t t = base + threadIdx.x;
    const int64_t u = t < t1 ? oa.U[t] : -1;
    if (t < t1) {
      kept += oa.L[t];
      ents += u;
    }
    const bool isw = u > 0, ise = u == 0;   // every lane calls every agg_inc (warp-synchronous)
    const unsigned w = agg_inc<unsigned>(oa.cnt, 0, isw);
    const unsigned e = agg_inc<unsigned>(oa.cnt + 1, 0, ise);
    agg_inc<unsigned long long>(reinterpret_cast<unsigned long long*>(oa.hist), isw ? oa.BK - u : 0, isw);
    agg_inc<unsigned long long>(reinterpret_cast<unsigned long long*>(oa.hist_sb), isw ? sb_of(t, t0, oa.GN) : 0, isw);
    if (isw) {
      oa.work[w] = static_cast<int32_t>(t);
      mark_working(oa, t, t0);
    }
    if (ise) oa.empty[e] = static_cast<int32_t>(t);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    kept += __shfl_xor_sync(0xffffffffu, kept, o);
    ents += __shfl_xor_sync(0xffffffffu, ents, o);
  }
  if ((threadIdx.x & 31) == 0 && (kept || ents)) {
    atomicAdd(reinterpret_cast<unsigned long long*>(oa.totals), static_cast<unsigned long long>(kept));
    atomicAdd(reinterpret_cast<unsigned long long*>(oa.totals) + 1, static_cast<unsigned long long>(ents));
  }
}

__global__ void __launch_bounds__(1024) order_scan_kernel(const OrderArgs oa) {   // > kSmemBuckets buckets only
  __shared__ int64_t s_warp[33];
  sm100::pdl_wait();
  sm100::pdl_trigger();
  const int64_t n_work = oa.cnt[0];
  const bool blocked = n_work >= 16 * static_cast<int64_t>(oa.num_sms);
  block_scan_array(blocked ? oa.hist_sb : oa.hist, oa.bucket_pos, blocked ? oa.nsb : oa.BK + 1, false, s_warp);
}

// Place the work list into the claim order and append the empty tiles.  CTA `cta` of `ncta` (the
// scatter kernel: one per SM; the skip map's last CTA for small ranges: 1 of 1); s_pos = shared
// memory of kSmemBuckets + 1 words.
__device__ void order_place(const OrderArgs& oa, int64_t t0, int64_t t1, int cta, int ncta, int64_t* s_pos,
                            int64_t* s_warp) {
  const int64_t n_work = oa.cnt[0], n_empty = oa.cnt[1];
  const bool blocked = n_work >= 16 * static_cast<int64_t>(oa.num_sms);
  const int64_t nbucket = blocked ? oa.nsb : oa.BK + 1;
  const int64_t* base = oa.bucket_pos;
  if (nbucket <= kSmemBuckets) {   // every CTA scans the (small) histogram itself
    block_scan_array(blocked ? oa.hist_sb : oa.hist, s_pos, nbucket, false, s_warp);
    base = s_pos;
  }
  const int64_t stride = static_cast<int64_t>(ncta) * blockDim.x;
  if (blocked) {   // slot = super-block start + rank of the tile among its block's working tiles (row-major)
    for (int64_t i = static_cast<int64_t>(cta) * blockDim.x + threadIdx.x; i < n_work; i += stride) {
      const int64_t t = oa.work[i];
      const int64_t sb = sb_of(t, t0, oa.GN);
      const uint32_t b = sb_pos(t, t0, oa.GN);
      const unsigned long long* w = oa.sb_bits + sb * kSbWords;
      int64_t rank = 0;
      for (uint32_t q = 0; q < b / 64; ++q) rank += __popcll(w[q]);
      rank += __popcll(w[b / 64] & ((1ull << (b % 64)) - 1ull));
      oa.order[base[sb] + rank] = static_cast<int32_t>(t);
    }
  } else if (cta == 0) {
    // LPT: one CTA walks the range in tile order, one window at a time, so equal keys (Toeplitz
    // bands have many equal U) keep row-major order -- neighbouring tiles run together
    unsigned long long* pos = nbucket <= kSmemBuckets ? reinterpret_cast<unsigned long long*>(s_pos)
                                                      : reinterpret_cast<unsigned long long*>(oa.bucket_cnt);
    for (int64_t c0 = t0; c0 < t1; c0 += blockDim.x) {
      const int64_t t = c0 + threadIdx.x;
      const int64_t u = t < t1 ? oa.U[t] : 0;
      const int64_t key = u > 0 ? oa.BK - u : 0;
      const unsigned long long slot = agg_inc<unsigned long long>(pos, key, u > 0);
      if (u > 0) oa.order[nbucket <= kSmemBuckets ? static_cast<int64_t>(slot) : base[key] + static_cast<int64_t>(slot)] =
          static_cast<int32_t>(t);
      __syncthreads();
    }
  }
  for (int64_t i = static_cast<int64_t>(cta) * blockDim.x + threadIdx.x; i < n_empty; i += stride)
    oa.order[n_work + i] = oa.empty[i];
  if (cta == 0 && threadIdx.x == 0) oa.totals[2] = n_empty;
  if (cta == 0 && threadIdx.x < 4 && oa.sched) oa.sched[threadIdx.x] = 0u;
}

__global__ void __launch_bounds__(1024) order_scatter_kernel(const OrderArgs oa) {
  __shared__ int64_t s_warp[33];
  __shared__ int64_t s_pos[kSmemBuckets + 1];
  sm100::pdl_wait();
  sm100::pdl_trigger();
  int64_t t0, t1;
  order_range(oa, t0, t1);
  order_place(oa, t0, t1, blockIdx.x, gridDim.x, s_pos, s_warp);
}

struct SkipArgs {
  const double* nA;
  const double* nBt;
  const double* pyr;
  int64_t BM, BK, BN, GM, GN, NC;
  double tau;
  int64_t gi0, gi1, ex0, ex1;   // macro rows [gi0, gi1) minus [ex0, ex1)
  const int64_t* d_range;       // overrides gi0..ex1 when non-null (multi-GPU)
  int64_t* U;
  int64_t* L;
  unsigned long long* row_work; // nullptr: not accumulated (second multi-GPU pass)
  void* macro_ent;
  uint4* macro_run;             // nullptr: FP32 paths
  unsigned int* claim;          // tile-claim counter (zeroed with the workspace; a second launch on the
                                // same workspace -- the multi-GPU final pass -- uses its own)
};

// One WARP per macro-tile (32 macro-tiles in flight per SM, no block-level barriers): warps claim
// macro-tiles from a counter (a banded product's tiles differ widely in work); lane c classifies
// k chunk c from the pyramid, then the surviving chunks are decided one at a time in ascending k
// (lane = k), each writing its entries at warp-scanned offsets.
template <int MI, int MJ>
__global__ void __launch_bounds__(kWarps * 32) skip_pyr_kernel(const SkipArgs a, const OrderArgs oa, int lists,
                                                               int inline_order) {
  __shared__ int64_t s_warp[33];
  __shared__ int s_last;
  extern __shared__ int64_t s_dyn[];   // inline order: kSmemBuckets + 1 bucket starts
  using M_ = mask_t<MI, MJ>;
  constexpr bool kMask64 = MI * MJ > 32;          // 8 x 8 tiles: (k, mask_lo, mask_hi, 0) entries
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  sm100::pdl_wait();
  sm100::pdl_trigger();
  int64_t gi0 = a.gi0, gi1 = a.gi1, ex0 = a.ex0, ex1 = a.ex1;
  if (a.d_range) {
    gi0 = a.d_range[0];
    gi1 = a.d_range[1];
    ex0 = a.d_range[2];
    ex1 = a.d_range[3];
  }
  ex0 = ex0 < gi0 ? gi0 : (ex0 > gi1 ? gi1 : ex0);
  ex1 = ex1 < ex0 ? ex0 : (ex1 > gi1 ? gi1 : ex1);
  const int64_t n_lo = (ex0 - gi0) * a.GN;
  const int64_t n_macro = n_lo + (gi1 - ex1) * a.GN;
  const double* __restrict__ paMax = a.pyr;
  const double* __restrict__ paMin = a.pyr + a.GM * a.NC;
  const double* __restrict__ pbMax = a.pyr + 2 * a.GM * a.NC;
  const double* __restrict__ pbMin = pbMax + a.GN * a.NC;
  const double tau = a.tau;
  int64_t w_kept = 0, w_ents = 0;   // this warp's totals (lane 0)

  for (;;) {
    unsigned int mc = 0;
    if (lane == 0) mc = atomicAdd(a.claim, 1u);
    const int64_t m = __shfl_sync(0xffffffffu, mc, 0);
    if (m >= n_macro) break;
    const int64_t tile = m < n_lo ? gi0 * a.GN + m : ex1 * a.GN + (m - n_lo);
    const int64_t I = tile / a.GN, J = tile % a.GN;
    const M_ valid = valid_bits<MI, MJ>(a.BM, a.BN, I, J);
    int64_t mbase = tile * a.BK;   // macro-tile region (entry e: 2e, 2e+1 in macro_run)
    uint32_t rw[MI];
#pragma unroll
    for (int li = 0; li < MI; ++li) rw[li] = 0u;
    for (int64_t c0 = 0; c0 < a.NC; c0 += 32) {
      // lane = chunk c0 + lane: 0 skipped, 1 mixed, 2 all kept (from the pyramid, exactly; R20)
      const int64_t c = c0 + lane;
      uint32_t cls = 0;
      if (c < a.NC && valid != 0u) {
        if (a.pyr == nullptr) {   // small K: no pyramid, every chunk tests its pairs
          cls = 1u;
        } else {
          const double amax = paMax[I * a.NC + c], bmax = pbMax[J * a.NC + c];
          if (!(__dmul_rn(amax, bmax) < tau))
            cls = __dmul_rn(paMin[I * a.NC + c], pbMin[J * a.NC + c]) >= tau ? 2u : 1u;
        }
      }
      uint32_t surv = __ballot_sync(0xffffffffu, cls != 0u);
      const uint32_t full = __ballot_sync(0xffffffffu, cls == 2u);
      while (surv) {
        const int cc = __ffs(surv) - 1;
        surv &= surv - 1u;
        const int64_t k = (c0 + cc) * kChunk + lane;
        M_ mask = 0u;
        if (k < a.BK) {
          if ((full >> cc) & 1u) {
            mask = valid;                 // all pairs of the chunk kept: no norm loads
          } else {
            ChunkVals<MI, MJ> cv;
#pragma unroll
            for (int li = 0; li < MI; ++li) {
              const int64_t i = I * MI + li;
              cv.a[li] = i < a.BM ? __ldg(a.nA + i * a.BK + k) : 0.0;
            }
#pragma unroll
            for (int lj = 0; lj < MJ; ++lj) {
              const int64_t j = J * MJ + lj;
              cv.b[lj] = j < a.BN ? __ldg(a.nBt + j * a.BK + k) : 0.0;
            }
            mask = chunk_mask<MI, MJ>(cv, valid, tau);
          }
        }
#pragma unroll
        for (int li = 0; li < MI; ++li)
          rw[li] += static_cast<uint32_t>(__popcll(static_cast<unsigned long long>(mask >> (li * MJ)) & ((1ull << MJ) - 1ull)));
        const uint32_t any = __ballot_sync(0xffffffffu, mask != 0u);
        if (mask) {
          const int64_t e = mbase + __popc(any & lt);
          if constexpr (kMask64) {
            reinterpret_cast<uint4*>(a.macro_ent)[e] =
                make_uint4(static_cast<uint32_t>(k), static_cast<uint32_t>(mask), static_cast<uint32_t>(mask >> 32), 0u);
            if (a.macro_run != nullptr) {   // 256 x 256 two-issuer path: the 4 x 8 runs of each half
              a.macro_run[2 * e] = encode_runs(static_cast<uint32_t>(k), static_cast<uint32_t>(mask));
              a.macro_run[2 * e + 1] = encode_runs(static_cast<uint32_t>(k), static_cast<uint32_t>(mask >> 32));
            }
          } else {
            reinterpret_cast<uint2*>(a.macro_ent)[e] = make_uint2(static_cast<uint32_t>(k), static_cast<uint32_t>(mask));
          }
        }
        mbase += __popc(any);
      }
    }
    // ---- per-macro-tile counts: union length U, kept pairs L, row work; the order's lists
    uint32_t lsum = 0;
#pragma unroll
    for (int li = 0; li < MI; ++li) {
      uint32_t v = rw[li];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      lsum += v;
      if (a.row_work && lane == li && I * MI + li < a.BM && v) atomicAdd(a.row_work + I * MI + li, static_cast<unsigned long long>(v));
    }
    if (lane == 0) {
      const int64_t u = mbase - tile * a.BK;
      a.U[tile] = u;
      a.L[tile] = lsum;
      w_kept += lsum;
      w_ents += u;
      if (lists) {
        if (u > 0) {
          oa.work[atomicAdd(oa.cnt, 1u)] = static_cast<int32_t>(tile);
          atomicAdd(reinterpret_cast<unsigned long long*>(oa.hist) + (a.BK - u), 1ull);
          atomicAdd(reinterpret_cast<unsigned long long*>(oa.hist_sb) + sb_of(tile, gi0 * a.GN, a.GN), 1ull);
          mark_working(oa, tile, gi0 * a.GN);
        } else {
          oa.empty[atomicAdd(oa.cnt + 1, 1u)] = static_cast<int32_t>(tile);
        }
      }
    }
  }
  if (lane == 0 && lists && (w_kept || w_ents)) {
    atomicAdd(reinterpret_cast<unsigned long long*>(oa.totals), static_cast<unsigned long long>(w_kept));
    atomicAdd(reinterpret_cast<unsigned long long*>(oa.totals) + 1, static_cast<unsigned long long>(w_ents));
  }
  if (!inline_order) return;
  // small ranges: the last CTA to finish places the claim order itself (saves a launch)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(oa.cnt + 3, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  order_place(oa, gi0 * a.GN, gi1 * a.GN, 0, 1, s_dyn, s_warp);
  if (threadIdx.x == 0) oa.cnt[3] = 0u;
}

// Per-C-tile k lists (C tile (i,j) owns slots [(i*BN+j)*BK, +V)) expanded from the macro lists:
// one warp per macro-tile, lane b appends the k-steps whose mask has bit b -- ascending k,
// exactly the skip map the fused pass decided.
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

// Multi-GPU partition on the device (spamm_partition_rows' rule over macro rows, integer
// arithmetic so host and device cut identically): macro-row work from the all-reduced row
// work, then cut r = first macro row g whose exclusive prefix pre satisfies
// 2 n pre + n w_g >= 2 r total.  Writes the range block (api: internal.h kRangeWords).
__global__ void __launch_bounds__(1024)
    partition_kernel(const int64_t* __restrict__ row_work, int64_t BM, int MI, int64_t GM, int rank, int nranks,
                     int64_t* __restrict__ rng) {
  extern __shared__ int64_t s_mw[];   // [GM]
  for (int64_t g = threadIdx.x; g < GM; g += blockDim.x) {
    int64_t s = 0;
    for (int r = 0; r < MI; ++r) {
      const int64_t i = g * MI + r;
      if (i < BM) s += row_work[i];
    }
    s_mw[g] = s;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int64_t total = 0;
  for (int64_t g = 0; g < GM; ++g) total += s_mw[g];
  int64_t* cut = rng + 6;
  cut[0] = 0;
  int64_t pre = 0, g = 0;
  const int64_t n = nranks;
  for (int r = 1; r < nranks; ++r) {
    while (g < GM && 2 * n * pre + n * s_mw[g] < 2 * static_cast<int64_t>(r) * total) {
      pre += s_mw[g];
      ++g;
    }
    cut[r] = g > cut[r - 1] ? g : cut[r - 1];
  }
  cut[nranks] = GM;
  rng[0] = cut[rank];
  rng[1] = cut[rank + 1];
  rng[2] = GM * rank / nranks;           // the provisional (even) range whose skip map is built
  rng[3] = GM * (rank + 1) / nranks;
  rng[4] = nranks;
  rng[5] = rank;
}

template <int MI, int MJ>
spamm_status skip_t(Plan& p, int64_t gi0, int64_t gi1, bool on_device, bool order, bool row_work, cudaStream_t s) {
  const int64_t n_macro = on_device ? p.GM * p.GN : (gi1 - gi0) * p.GN;
  constexpr int kPerSm = 4;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n_macro + kWarps - 1) / kWarps,
                                                                static_cast<int64_t>(p.num_sms) * kPerSm));
  SkipArgs a{p.nA, p.nBt, p.pyr_ready ? p.pyr : nullptr, p.BM, p.BK, p.BN, p.GM, p.GN, p.NC, p.tau, gi0, gi1, 0, 0,
             on_device ? p.d_range : nullptr, p.U, p.L,
             row_work ? reinterpret_cast<unsigned long long*>(p.row_work) : nullptr, p.macro_ent, p.macro_run,
             p.ws_cnt + (on_device ? 3 : 2)};
  OrderArgs oa{p.hist, p.hist_sb, p.bucket_cnt, p.bucket_pos, p.sb_bits, p.NSB, p.U, p.L, p.BK, p.GN, p.num_sms, p.tile_lists,
               p.tile_lists + p.GM * p.GN, p.ws_cnt, p.order, p.totals, p.sched, on_device ? p.d_range : nullptr,
               gi0 * p.GN, gi1 * p.GN};
  // the main loop builds the order's lists unless part of the range came from another launch; small
  // ranges get their order from the skip kernel's last CTA (no scatter launch)
  const int lists = order && !on_device ? 1 : 0;
  const bool inl = lists && n_macro <= kInlineOrderTiles && std::max<int64_t>(p.BK + 1, p.NSB) <= kSmemBuckets;
  const int dyn = inl ? static_cast<int>((kSmemBuckets + 1) * sizeof(int64_t)) : 0;
  auto kern = skip_pyr_kernel<MI, MJ>;
  SPAMM_SET_SMEM(kern, static_cast<int>((kSmemBuckets + 1) * sizeof(int64_t)), p.device);
  SPAMM_CUDA_TRY(launch_pdl(kern, dim3(static_cast<unsigned>(blocks)), dim3(kWarps * 32), dyn, s, a, oa, lists,
                            inl ? 1 : 0));
  count_launch();
  if (order && !inl) {
    // one CTA per 1024 macro-tiles of the range, at most one per SM
    const unsigned g = static_cast<unsigned>(
        std::max<int64_t>(1, std::min<int64_t>(p.num_sms, ((on_device ? p.GM : gi1 - gi0) * p.GN + 1023) / 1024)));
    if (on_device) {
      SPAMM_CUDA_TRY(launch_pdl(order_lists_kernel, dim3(g), dim3(256), 0, s, oa));
      count_launch();
    }
    if (std::max<int64_t>(p.BK + 1, p.NSB) > kSmemBuckets) {
      SPAMM_CUDA_TRY(launch_pdl(order_scan_kernel, dim3(1), dim3(1024), 0, s, oa));
      count_launch();
    }
    SPAMM_CUDA_TRY(launch_pdl(order_scatter_kernel, dim3(g), dim3(1024), 0, s, oa));
    count_launch();
  }
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

}  // namespace

spamm_status launch_pyramid(Plan& p, cudaStream_t s) {
  const int64_t warps = (p.GM + p.GN) * p.NC;
  const unsigned blocks = static_cast<unsigned>((warps + 7) / 8);
  auto kern = p.MI == kMacroTC ? pyramid_kernel<kMacroTC, kMacroTC> : pyramid_kernel<kMacroF32, kMacroF32>;
  SPAMM_CUDA_TRY(launch_pdl(kern, dim3(blocks), dim3(256), 0, s, static_cast<const double*>(p.nA),
                            static_cast<const double*>(p.nBt), p.BM, p.BK, p.BN, p.GM, p.GN, p.NC, p.pyr));
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  p.pyr_ready = true;
  return SPAMM_OK;
}

spamm_status launch_skipmap(Plan& p, int64_t gi0, int64_t gi1, bool on_device, bool order, bool row_work,
                            cudaStream_t s) {
  if (p.MI == kMacroTC) return skip_t<kMacroTC, kMacroTC>(p, gi0, gi1, on_device, order, row_work, s);
  return skip_t<kMacroF32, kMacroF32>(p, gi0, gi1, on_device, order, row_work, s);
}

spamm_status launch_partition(Plan& p, int rank, int nranks, cudaStream_t s) {
  const int smem = static_cast<int>(p.GM * sizeof(int64_t));
  if (smem > 200 * 1024) return fail(SPAMM_E_UNSUPPORTED, "too many macro rows for the device partition");
  SPAMM_SET_SMEM(partition_kernel, 200 * 1024, p.device);
  partition_kernel<<<1, 1024, smem, s>>>(p.row_work, p.BM, p.MI, p.GM, rank, nranks, p.d_range);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

spamm_status launch_leaf_expand(Plan& p, cudaStream_t s) {
  const int64_t gi0 = p.row_begin_macro, gi1 = p.row_end_macro;
  const int64_t nleaf = p.BM * p.BN;
  if (gi0 != 0 || gi1 != p.GM) SPAMM_CUDA_TRY(cudaMemsetAsync(p.V, 0, sizeof(int64_t) * nleaf, s));
  const int64_t n_macro = (gi1 - gi0) * p.GN;
  if (n_macro <= 0) return SPAMM_OK;
  const int64_t blocks = (n_macro + kWarps - 1) / kWarps;
  if (p.MI == kMacroTC)
    leaf_expand_kernel<kMacroTC, kMacroTC><<<static_cast<unsigned>(blocks), kWarps * 32, 0, s>>>(
        p.BM, p.BK, p.BN, p.GN, gi0, n_macro, p.U, p.macro_ent, p.V, p.leaf_start, p.leaf_k);
  else
    leaf_expand_kernel<kMacroF32, kMacroF32><<<static_cast<unsigned>(blocks), kWarps * 32, 0, s>>>(
        p.BM, p.BK, p.BN, p.GN, gi0, n_macro, p.U, p.macro_ent, p.V, p.leaf_start, p.leaf_k);
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

}  // namespace spamm
