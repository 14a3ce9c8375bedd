// norms.cu -- stage 1: tile Frobenius norms (Eq. 2; get-norm kernel Sec. 3.2,
// PAPER.md:105-123).
//
// B200 design (not the paper's one-block-per-tile shared-memory tree): the matrices are
// read exactly once by TMA.  A CTA owns one 32-row tile strip and a range of 512-byte-wide
// column boxes ([32 rows x 512 B] = 8 FP32 tiles or 4... see kColsPerBox); one thread issues
// the bulk tensor loads into a 4-deep shared-memory ring (mbarrier completion), the 4
// warps each reduce 8 rows of a box: every lane squares 16 contiguous bytes per row in
// float64, the lanes of one tile combine with an xor butterfly and the warps' partials
// are summed in warp order.  The operation sequence per tile does not depend on the
// tile's position, so equal tiles give bit-identical norms (Toeplitz inputs).  TMA's
// out-of-bounds zero fill implements the zero padding of PAPER.md:99.  A and B are
// normed by one launch.
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "internal.h"
#include "sm100.cuh"

namespace spamm {
namespace {

using namespace sm100;

constexpr int kWarps = 8;              // warps per CTA, each reducing 32 / kWarps rows of a box
constexpr int kRowsPerWarp = 32 / kWarps;
constexpr int kThreads = kWarps * 32;
constexpr int kBoxBytesRow = 512;      // bytes per box row (256 BF16 / 128 FP32 columns)
constexpr int kBoxBytes = 32 * kBoxBytesRow;   // 16 KB
constexpr int kBoxesPerCta = 16;       // max column boxes walked by one CTA
constexpr int kStages = 2;             // TMA ring depth (33 KB per CTA: 6 CTAs per SM)
template <int S>
constexpr size_t smem_bytes() { return 128 + static_cast<size_t>(S) * kBoxBytes + 1024; }

template <typename T>
__device__ __forceinline__ double sq16(const uint4& raw);
template <>
__device__ __forceinline__ double sq16<float>(const uint4& raw) {
  double s = 0.0;
  const float* f = reinterpret_cast<const float*>(&raw);
#pragma unroll
  for (int e = 0; e < 4; ++e) s = fma(static_cast<double>(f[e]), static_cast<double>(f[e]), s);
  return s;
}
template <>
__device__ __forceinline__ double sq16<__nv_bfloat16>(const uint4& raw) {
  double s = 0.0;
  const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const double x = static_cast<double>(__bfloat162float(h[e]));
    s = fma(x, x, s);
  }
  return s;
}
template <>
__device__ __forceinline__ double sq16<__half>(const uint4& raw) {
  double s = 0.0;
  const __half* h = reinterpret_cast<const __half*>(&raw);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const double x = static_cast<double>(__half2float(h[e]));
    s = fma(x, x, s);
  }
  return s;
}

struct NormJob {
  int64_t rows, cols;          // matrix extent (elements)
  double* out;                 // output map
  int64_t out_rs, out_cs;      // out[it*rs + kt*cs]
  int64_t r0, nrow;            // tile rows [r0, r0+nrow)
  int64_t ncb;                 // CTAs along the columns
  int bpc;                     // column boxes per CTA (<= kBoxesPerCta; fewer for small grids)
  double* out2;                // optional second map (A == B: nB^T from A's tiles), or nullptr
  int64_t out2_rs, out2_cs;
  uint16_t* planes;            // SPAMM_FP32X3: 3 bfloat16 split planes [3][rows][pld] of this matrix, or nullptr
  int64_t pld, pcol0;          // plane leading dimension; column offset of this job's strip in the planes
};

// a = a0 + a1 + a2 in bfloat16, each the RNE of the remaining residual (the residuals are
// exact in float).  Non-finite a: a0 carries it, a1 = a2 = 0 (products stay Inf/NaN like GEMM).
__device__ __forceinline__ void split3(float a, uint16_t& h0, uint16_t& h1, uint16_t& h2) {
  const __nv_bfloat16 b0 = __float2bfloat16_rn(a);
  const float r1 = a - __bfloat162float(b0);
  const __nv_bfloat16 b1 = __float2bfloat16_rn(r1);
  const float r2 = r1 - __bfloat162float(b1);
  const __nv_bfloat16 b2 = __float2bfloat16_rn(r2);
  const bool fin = isfinite(__bfloat162float(b0));
  h0 = __bfloat16_as_ushort(b0);
  h1 = fin ? __bfloat16_as_ushort(b1) : static_cast<uint16_t>(0);
  h2 = fin ? __bfloat16_as_ushort(b2) : static_cast<uint16_t>(0);
}
template <typename T>
__device__ __forceinline__ void write_planes(const NormJob&, const uint4&, int64_t, int64_t) {}
template <>
__device__ __forceinline__ void write_planes<float>(const NormJob& j, const uint4& raw, int64_t row, int64_t col) {
  const float* f = reinterpret_cast<const float*>(&raw);
  uint16_t h[3][4];
#pragma unroll
  for (int e = 0; e < 4; ++e) split3(f[e], h[0][e], h[1][e], h[2][e]);
  const int64_t plane = j.rows * j.pld;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const uint2 v = make_uint2(static_cast<uint32_t>(h[q][0]) | (static_cast<uint32_t>(h[q][1]) << 16),
                               static_cast<uint32_t>(h[q][2]) | (static_cast<uint32_t>(h[q][3]) << 16));
    *reinterpret_cast<uint2*>(j.planes + q * plane + row * j.pld + j.pcol0 + col) = v;
  }
}

// grid = (max ncb, nrowA + nrowB); blockIdx.y < nrowA -> job A else job B.
template <typename T>
__global__ void __launch_bounds__(kThreads) tile_norms_kernel(const __grid_constant__ CUtensorMap tmA,
                                                              const __grid_constant__ CUtensorMap tmB, NormJob ja,
                                                              NormJob jb, int64_t* __restrict__ zws, int zn) {
  constexpr int V = 16 / sizeof(T);              // elements per 16-byte lane load
  constexpr int kCols = kBoxBytesRow / sizeof(T);  // columns per box
  constexpr int LPT = 32 / V;                    // lanes per 32-column tile
  constexpr int TPB = kCols / 32;                // tiles per box
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint8_t* ring = smem;
  __shared__ uint64_t full[kStages];
  __shared__ double part[kWarps][kBoxesPerCta * TPB];

  pdl_wait();      // predecessors may write A (chained products) or read the counters zeroed below
  pdl_trigger();
  if (zws != nullptr && blockIdx.x == 0 && blockIdx.y == 0)   // the skip map's counters (spamm_run)
    for (int i = threadIdx.x; i < zn; i += blockDim.x) zws[i] = 0;
  const bool isA = blockIdx.y < ja.nrow;
  const NormJob& j = isA ? ja : jb;
  const CUtensorMap* tm = isA ? &tmA : &tmB;
  const int64_t it = j.r0 + (isA ? blockIdx.y : blockIdx.y - ja.nrow);
  if (static_cast<int64_t>(blockIdx.x) >= j.ncb) return;
  const int64_t box0 = static_cast<int64_t>(blockIdx.x) * j.bpc;
  const int64_t nbox_total = (j.cols + kCols - 1) / kCols;
  const int nbox = static_cast<int>(nbox_total - box0 < j.bpc ? nbox_total - box0 : j.bpc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    tma_prefetch_desc(tm);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int b = 0; b < nbox && b < kStages; ++b) {
      mbar_arrive_expect_tx(&full[b], kBoxBytes);
      tma_load_2d(ring + b * kBoxBytes, tm, &full[b], static_cast<int32_t>((box0 + b) * kCols),
                  static_cast<int32_t>(it * 32));
    }
  }
  for (int b = 0; b < nbox; ++b) {
    const int s = b % kStages;
    mbar_wait(&full[s], static_cast<uint32_t>((b / kStages) & 1));
    const uint8_t* box = ring + s * kBoxBytes;
    double acc = 0.0;                            // this lane's 16 bytes in the warp's 8 rows
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) {
      const uint4 raw = *reinterpret_cast<const uint4*>(box + (warp * kRowsPerWarp + r) * kBoxBytesRow + lane * 16);
      acc += sq16<T>(raw);
      if (j.planes != nullptr) {   // FP32X3: the element's bfloat16 split (rows/cols of the padded planes)
        const int64_t row = it * 32 + warp * kRowsPerWarp + r, col = (box0 + b) * kCols + lane * (16 / sizeof(T));
        if (row < j.rows && col < j.pld - j.pcol0) write_planes<T>(j, raw, row, col);
      }
    }
#pragma unroll
    for (int o = LPT / 2; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((lane % LPT) == 0) part[warp][b * TPB + lane / LPT] = acc;
    __syncthreads();                             // everyone is done with stage s
    if (threadIdx.x == 0 && b + kStages < nbox) {
      mbar_arrive_expect_tx(&full[s], kBoxBytes);
      tma_load_2d(ring + s * kBoxBytes, tm, &full[s], static_cast<int32_t>((box0 + b + kStages) * kCols),
                  static_cast<int32_t>(it * 32));
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nbox * TPB; t += kThreads) {
    double tot = part[0][t];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) tot += part[w][t];   // warp order: position independent
    const int64_t kt = box0 * TPB + t;
    if (kt * 32 < j.cols) {
      const double nrm = sqrt(tot);
      j.out[it * j.out_rs + kt * j.out_cs] = nrm;
      if (j.out2) j.out2[it * j.out2_rs + kt * j.out2_cs] = nrm;
    }
  }
}

template <typename T>
spamm_status launch_t(Plan& p, const void* A, int64_t lda, int64_t ar0, int64_t ar1, const void* B, int64_t ldb,
                      int64_t bj0, int64_t bj1, cudaStream_t s, CUtensorMapDataType dt) {
  constexpr int kCols = kBoxBytesRow / sizeof(T);
  CUtensorMap tA{}, tB{};
  NormJob ja{p.M, p.K, p.nA, p.BK, 1, ar0, ar1 - ar0, 0, 8, nullptr, 0, 0, nullptr, 0, 0};
  if (p.prec == SPAMM_FP32X3 && p.planes) {
    ja.planes = p.planes;
    ja.pld = p.ldpa;
  }
  // B column strip [bj0*32, bj1*32): treated as a (K x cols) matrix; tile row k, tile col j -> nBt[j*BK + k]
  const int64_t bcols = std::min<int64_t>(p.N, bj1 * kTile) - bj0 * kTile;
  NormJob jb{p.K, bcols > 0 ? bcols : 0, p.nBt + bj0 * p.BK, 1, p.BK, 0, bj1 > bj0 ? p.BK : 0, 0, 8, nullptr, 0, 0,
             nullptr, 0, 0};
  if (p.prec == SPAMM_FP32X3 && p.planes) {
    jb.planes = p.planes + 3 * p.M * p.ldpa;
    jb.pld = p.ldpb;
    jb.pcol0 = bj0 * kTile;
  }
  // B is A (same square matrix, same layout, full ranges): read it once.  Tile (r, c) of A is
  // tile (k = r, j = c) of B, so its norm is also nB^T[c*BK + r] (C = A*A, e.g. matrix powers).
  p.b_is_a = false;
  if (A == B && lda == ldb && p.M == p.K && p.K == p.N && ar0 == 0 && ar1 == p.BM && bj0 == 0 && bj1 == p.BN) {
    p.b_is_a = true;   // FP32X3: A's planes serve as B's
    ja.out2 = p.nBt;
    ja.out2_rs = 1;
    ja.out2_cs = p.BK;
    jb.nrow = 0;
  }
  // boxes per CTA: 8 (128 KB streamed per CTA) unless that leaves fewer than ~4 CTAs per SM,
  // then fewer so that small problems are not latency-bound on a handful of CTAs.  Ring depth 2
  // (33 KB per CTA, 6 CTAs per SM: the N = 8192 grid runs in about one wave; 29.3 vs 31.1 us with
  // 4 stages, r01f)
  int bpc = 8;
  auto ncb_of = [&](const NormJob& jj, int b) -> int64_t {
    const int64_t per_cta = static_cast<int64_t>(b) * kCols;
    return jj.nrow > 0 ? (jj.cols + per_cta - 1) / per_cta : 0;
  };
  while (bpc > 1 && ncb_of(ja, bpc) * ja.nrow + ncb_of(jb, bpc) * jb.nrow < 4 * static_cast<int64_t>(p.num_sms))
    bpc >>= 1;
  ja.bpc = jb.bpc = bpc;
  ja.ncb = ncb_of(ja, bpc);
  jb.ncb = ncb_of(jb, bpc);
  if (ja.nrow > 0)
    SPAMM_TRY(encode_tmap_2d(&tA, dt, sizeof(T), A, p.K, p.M, lda, kCols, 32, CU_TENSOR_MAP_SWIZZLE_NONE));
  if (jb.nrow > 0) {
    const void* Bs = static_cast<const char*>(B) + static_cast<size_t>(bj0) * kTile * sizeof(T);
    SPAMM_TRY(encode_tmap_2d(&tB, dt, sizeof(T), Bs, bcols, p.K, ldb, kCols, 32, CU_TENSOR_MAP_SWIZZLE_NONE));
  }
  SPAMM_SET_SMEM(tile_norms_kernel<T>, static_cast<int>(smem_bytes<kStages>()), p.device);
  int64_t* zws = p.zero_ws_next ? p.row_work : nullptr;
  const int zn = static_cast<int>(ws_words(p));
  const int64_t gx = std::max(ja.ncb, jb.ncb);
  const int64_t gy = ja.nrow + jb.nrow;
  if (gx <= 0 || gy <= 0) return SPAMM_OK;
  if (gy > 65535) return fail(SPAMM_E_UNSUPPORTED, "more than 65535 tile rows in one norm launch");
  dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
  SPAMM_CUDA_TRY(launch_pdl(tile_norms_kernel<T>, grid, dim3(kThreads), smem_bytes<kStages>(), s, tA, tB, ja, jb, zws, zn));
  count_launch();
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

}  // namespace

spamm_status launch_norms2(Plan& p, const void* A, int64_t lda, int64_t ar0, int64_t ar1, const void* B,
                           int64_t ldb, int64_t bj0, int64_t bj1, cudaStream_t s) {
  switch (p.prec) {
    case SPAMM_FP32:
    case SPAMM_FP32X3:
      return launch_t<float>(p, A, lda, ar0, ar1, B, ldb, bj0, bj1, s, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
    case SPAMM_BF16:
      return launch_t<__nv_bfloat16>(p, A, lda, ar0, ar1, B, ldb, bj0, bj1, s, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
    case SPAMM_FP16:
      return launch_t<__half>(p, A, lda, ar0, ar1, B, ldb, bj0, bj1, s, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  }
  return fail(SPAMM_E_UNSUPPORTED, "precision");
}

}  // namespace spamm
