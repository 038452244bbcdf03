// format_kernels.cuh — the V:N:M compressor and decompressor for sm_100a (HBM-bound kernels).
//
// venom_compress implements PAPER.md:187-189 (§3, Fig 2 ④): per V×M block pick the four most
// significant columns, then per row the two largest weights among them; PAPER.md:192-195 (Fig 3)
// fixes the three output arrays. The readings DESIGN.md lists (#1 L1 over the block's rows in fp64,
// ascending rows; #3 two-stage greedy; #5/#6 ties -> lower index; #7 ascending storage; #8 nibble
// packing) are what make the output byte-identical to the CPU oracle.
#pragma once
#include <cuda.h>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ptx_sm100.cuh"

namespace venom {

constexpr int kStatusNonFinite = 6;
constexpr int kStatusCorruptMetadata = 7;

template <bool kBF16>
__device__ __forceinline__ float bits_to_float(uint16_t b) {
  if constexpr (kBF16) {
    return __uint_as_float(static_cast<uint32_t>(b) << 16);
  } else {
    return __half2float(__ushort_as_half(b));
  }
}
template <bool kBF16>
__device__ __forceinline__ bool bits_non_finite(uint16_t b) {
  return kBF16 ? ((b & 0x7F80u) == 0x7F80u) : ((b & 0x7C00u) == 0x7C00u);
}

// Compression. grid = (ceil(G / gpc), R / V), block = 256 threads.
// One CTA owns one row-block rb and a chunk of `gpc` consecutive groups (gpc even, so metadata
// bytes — two groups each — are never shared between CTAs).
//   phase 1: column L1 mass over the block's V rows in fp64. Each thread sums VEC adjacent
//            columns (16-byte loads when VEC = 8) over a contiguous range of rows, ascending.
//            fp16: |a| are multiples of 2^-24 below 2^16, so fp64 partial sums over row ranges
//            are exact and their (fixed-order) total is bit-identical to the oracle's sequential
//            sum; the rows are split over the idle threads. bf16: one range (sequential, same
//            order as the oracle: exactness is not guaranteed, order is).
//   phase 2: thread per group: top-4 columns by (s desc, index asc), sorted ascending
//   phase 3: thread per (row, pair of groups): top-2 of the 4 by (|a| desc, position asc),
//            raw-bit value copy, nibble packing — one metadata byte and 8 value bytes per thread.
template <bool kBF16, int VEC>
__global__ void __launch_bounds__(256) vnm_compress_kernel(
    const uint16_t* __restrict__ A, int64_t R, int64_t K, int64_t lda, int V, int M, int64_t G,
    int gpc, uint16_t* __restrict__ values, uint8_t* __restrict__ metadata,
    uint8_t* __restrict__ column_idx, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int64_t rb = blockIdx.y;
  const int64_t g0 = static_cast<int64_t>(blockIdx.x) * gpc;
  const int ng = static_cast<int>((G - g0) < gpc ? (G - g0) : gpc);  // groups in this chunk
  const int ncols = ng * M;
  const int wmax = gpc * M;
  const int ncv = (ncols + VEC - 1) / VEC;                 // column vectors in this chunk
  const int ncv_max = (wmax + VEC - 1) / VEC;
  const int nsplit_max = kBF16 ? 1 : (static_cast<int>(blockDim.x) / ncv_max > 0 ? static_cast<int>(blockDim.x) / ncv_max : 1);
  double* s_part = reinterpret_cast<double*>(smem_raw);                      // nsplit_max × wmax
  double* s_score = s_part;                                                  // reused: row 0
  uint8_t* s_sel = smem_raw + sizeof(double) * static_cast<size_t>(nsplit_max) * wmax;  // gpc × 4
  const int64_t k0 = g0 * M;
  const int64_t row0 = rb * V;
  const int64_t meta_row = (G + 1) / 2;
  const int nsplit = nsplit_max < V ? nsplit_max : V;  // row ranges (fp16 only; smem-sized)

  // ---- phase 1: column L1 mass, fp64, ascending rows within each range
  bool bad = false;
  for (int t = threadIdx.x; t < ncv * nsplit; t += blockDim.x) {
    const int cv = t % ncv, sp = t / ncv;
    const int rbeg = static_cast<int>((static_cast<int64_t>(V) * sp) / nsplit);
    const int rend = static_cast<int>((static_cast<int64_t>(V) * (sp + 1)) / nsplit);
    const int c0 = cv * VEC;
    const uint16_t* col = A + row0 * lda + k0 + c0;
    double acc[VEC];
#pragma unroll
    for (int u = 0; u < VEC; ++u) acc[u] = 0.0;
    const bool full = (VEC == 1) || (c0 + VEC <= ncols);
    int i = rbeg;
    if (VEC == 8 && full) {
      for (; i + 4 <= rend; i += 4) {
        uint4 w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = __ldg(reinterpret_cast<const uint4*>(col + static_cast<int64_t>(i + q) * lda));
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t ww[4] = {w[q].x, w[q].y, w[q].z, w[q].w};
#pragma unroll
          for (int u = 0; u < VEC; ++u) {
            const uint16_t b = static_cast<uint16_t>((ww[u >> 1] >> (16 * (u & 1))) & 0xFFFFu);
            bad |= bits_non_finite<kBF16>(b);
            acc[u] = __dadd_rn(acc[u], static_cast<double>(fabsf(bits_to_float<kBF16>(b))));
          }
        }
      }
    }
    for (; i < rend; ++i) {
#pragma unroll
      for (int u = 0; u < VEC; ++u) {
        if (c0 + u < ncols) {
          const uint16_t b = __ldg(col + static_cast<int64_t>(i) * lda + u);
          bad |= bits_non_finite<kBF16>(b);
          acc[u] = __dadd_rn(acc[u], static_cast<double>(fabsf(bits_to_float<kBF16>(b))));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < VEC; ++u)
      if (c0 + u < ncols) s_part[sp * wmax + c0 + u] = acc[u];
  }
  if (bad && status != nullptr) atomicMax(status, kStatusNonFinite);
  __syncthreads();
  if (nsplit > 1) {
    // fixed-order total of the exact fp16 partial sums
    for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
      double sum = s_part[c];
      for (int sp = 1; sp < nsplit; ++sp) sum = __dadd_rn(sum, s_part[sp * wmax + c]);
      s_part[c] = sum;  // s_score aliases row 0: each thread only touches its own column
    }
    __syncthreads();
  }

  // ---- phase 2: the four most significant columns of each block
  for (int q = threadIdx.x; q < ng; q += blockDim.x) {
    const double* s = s_score + q * M;
    int c[4];
    // selection by repeated maximum: a strictly larger score displaces a lower index
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      int best = -1;
      double bs = 0.0;
      for (int j = 0; j < M; ++j) {
        bool taken = false;
#pragma unroll
        for (int u = 0; u < t; ++u) taken |= (c[u] == j);
        if (taken) continue;
        if (best < 0 || s[j] > bs) {
          best = j;
          bs = s[j];
        }
      }
      c[t] = best;
    }
    // sort ascending (4-element network)
#define VENOM_CSWAP(x, y) \
  if (c[x] > c[y]) {      \
    int t_ = c[x];        \
    c[x] = c[y];          \
    c[y] = t_;            \
  }
    VENOM_CSWAP(0, 1) VENOM_CSWAP(2, 3) VENOM_CSWAP(0, 2) VENOM_CSWAP(1, 3) VENOM_CSWAP(1, 2)
#undef VENOM_CSWAP
    uint32_t word = static_cast<uint32_t>(c[0]) | (static_cast<uint32_t>(c[1]) << 8) |
                    (static_cast<uint32_t>(c[2]) << 16) | (static_cast<uint32_t>(c[3]) << 24);
    reinterpret_cast<uint32_t*>(column_idx)[rb * G + g0 + q] = word;
    reinterpret_cast<uint32_t*>(s_sel)[q] = word;
  }
  __syncthreads();

  // ---- phase 3: per row, two largest |w| among the selected columns (2:4)
  const int npairs = (ng + 1) / 2;
  const int work = V * npairs;
  for (int w = threadIdx.x; w < work; w += blockDim.x) {
    const int i = w / npairs;
    const int pp = w - i * npairs;
    const int64_t row = row0 + i;
    uint8_t byte = 0;
    uint16_t out[4] = {0, 0, 0, 0};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = 2 * pp + h;
      if (q >= ng) break;
      const uint8_t* cs = s_sel + 4 * q;
      const uint16_t* arow = A + row * lda + k0 + static_cast<int64_t>(q) * M;
      uint16_t v[4];
      uint32_t mag[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        v[t] = __ldg(arow + cs[t]);
        mag[t] = v[t] & 0x7FFFu;  // |w| order for finite sign-magnitude formats; ±0 tie
      }
      int p0 = 0;
#pragma unroll
      for (int t = 1; t < 4; ++t)
        if (mag[t] > mag[p0]) p0 = t;
      int p1 = -1;
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (t != p0 && (p1 < 0 || mag[t] > mag[p1])) p1 = t;
      const int lo = min(p0, p1), hi = max(p0, p1);
      out[2 * h + 0] = v[lo];
      out[2 * h + 1] = v[hi];
      byte |= static_cast<uint8_t>((lo | (hi << 2)) << (4 * h));
    }
    const int64_t g = g0 + 2 * pp;
    uint16_t* vdst = values + (row * G + g) * 2;
    const uint32_t w0 = static_cast<uint32_t>(out[0]) | (static_cast<uint32_t>(out[1]) << 16);
    const uint32_t w1 = static_cast<uint32_t>(out[2]) | (static_cast<uint32_t>(out[3]) << 16);
    if (2 * pp + 1 < ng) {
      if (((row * G + g) & 1) == 0) {
        *reinterpret_cast<uint2*>(vdst) = make_uint2(w0, w1);  // 8-byte aligned
      } else {
        reinterpret_cast<uint32_t*>(vdst)[0] = w0;  // odd G: only 4-byte aligned
        reinterpret_cast<uint32_t*>(vdst)[1] = w1;
      }
    } else {
      *reinterpret_cast<uint32_t*>(vdst) = w0;
    }
    metadata[row * meta_row + g / 2] = byte;
  }
}

// Shared-memory layout of vnm_compress_tile_kernel (host and device agree on it): the V × W tile
// (16-bit), NS row-slice partial column sums (fp32), the column scores (fp64), per group the
// selected-column word, the 4th / 5th largest score and a flag, a per-column "selected" byte, and
// with kExpand the re-encoding's nibbles [V][W/8].
struct CompressTileLayout {
  static constexpr int NS = 8;  // row slices of the approximate column sums
  size_t tile, tile_bytes, part, score, sel, th, rank, m2, total;
  // swz: the tile as ceil(W / 64) boxes of V rows × 128 B with the 128-byte TMA swizzle (each box
  // 1 KB aligned); else rows of W + 8 elements (a 16-byte pad per row). Either way the 8 rows a
  // column-wise access touches fall in 8 different bank groups (a dense 256-byte pitch put them
  // all in the same banks: 8-way conflicts in phase 3).
  __host__ __device__ CompressTileLayout(int V, int W, int gpc, bool expand, int ntiles = 1, bool swz = false) {
    tile = 0;
    tile_bytes = swz ? static_cast<size_t>((W + 63) / 64) * ((static_cast<size_t>(V) * 128 + 1023) & ~size_t(1023))
                     : ((static_cast<size_t>(V) * (W + 8) * 2 + 1023) & ~size_t(1023));
    part = tile_bytes * ntiles;
    score = part + static_cast<size_t>(NS) * W * 4;
    sel = score + static_cast<size_t>(W) * 8;
    th = sel + ((static_cast<size_t>(gpc) * 4 + 15) & ~size_t(15));
    rank = th + static_cast<size_t>(gpc) * 16;
    m2 = rank + ((static_cast<size_t>(W) + 15) & ~size_t(15));
    total = m2 + (expand ? static_cast<size_t>(V) * (W / 8) : 0) + 16 + 1024;  // + 1 KB base alignment
  }
};

// Element addressing of a compressor tile in shared memory (see CompressTileLayout).
struct TileView {
  const uint16_t* base;
  int pitch;      // padded: row pitch in elements (W + 8)
  int box;        // swizzled: elements per 64-column box (V·64 rounded to 1 KB)
  bool swz;
  __device__ __forceinline__ int idx(int i, int c) const {
    return swz ? (c >> 6) * box + i * 64 + (((((c >> 3) & 7) ^ (i & 7))) << 3) + (c & 7) : i * pitch + c;
  }
  __device__ __forceinline__ uint16_t at(int i, int c) const { return base[idx(i, c)]; }
  // the 8 columns 8·cv .. 8·cv + 7 of row i (16-byte aligned)
  __device__ __forceinline__ uint4 vec(int i, int cv) const {
    return *reinterpret_cast<const uint4*>(base + idx(i, 8 * cv));
  }
};

// Compression, shared-memory tile variant (the default when the V × W tile fits): the CTA's V × W
// block of A (W = gpc·M columns) is read from HBM once with 16-byte loads, all in flight together,
// then:
//   phase 1: column L1 mass. The oracle's score is the fp64 sum of |a| over the V rows in ascending
//            order (reading #2). Computing that for every column costs ~13 instructions per element
//            (the compressor was instruction-bound at 1.2 TB/s), so the kernel first sums in fp32
//            (|a| of fp16 / bf16 is exact in fp32; NS row slices, then the slices in order) and
//            only decides from those where they cannot be wrong: an fp32 sum of n non-negative terms
//            is within n·2^-24 (relative) of the exact sum, so when the 4th and 5th largest
//            approximate scores of a group differ by more than twice that bound, the exact top-4
//            set — which is all the format stores (reading #7: ascending) — is the approximate one.
//            Groups that fail the margin test (near-ties, all-zero blocks, fp32 overflow) get the
//            exact scores: fp16 as integer sums of |a| in units of 2^-24 (exact, so equal to the
//            oracle's fp64 sum in any order), bf16 as the oracle's sequential fp64 sum.
//   phase 2: rank of each column in its group by (score desc, index asc); rank < 4 is selected.
//   phase 3: thread per (row, group): top-2 of the 4 by (|a| desc, position asc), raw-bit value
//            copy, nibble packing (+ the V:2:4 re-encoding with kExpand).
// Phases 1-4 of the compressor on one V × W tile already in shared memory (`tile`, pitch W); the
// scratch arrays live at `smem_raw` + CompressTileLayout offsets. Called by the tile kernel (after
// its own loads) and by the persistent TMA kernel (once per tile of its pipeline).
// MC / GPC / NTHR: compile-time M, groups per tile and block size (0 = runtime). With all three
// fixed and G % GPC == 0 (every tile full), the per-tile index arithmetic has no divisions — round 2
// measured the per-tile setup at a third of the compressor's instructions, mostly divisions by
// runtime M and group counts.
template <bool kBF16, bool kExpand, int MC = 0, int GPC = 0, int NTHR = 0>
__device__ __forceinline__ void compress_tile_process(
    const TileView tile_in, uint8_t* smem_in, int64_t R, int64_t K, int V, int M_in, int64_t G,
    int gpc_in, int64_t rb, int64_t g0, uint16_t* __restrict__ values, uint8_t* __restrict__ metadata,
    uint8_t* __restrict__ column_idx, int32_t* __restrict__ status, uint32_t* __restrict__ values2,
    uint32_t* __restrict__ meta_tc, int dbg, int nbuf) {
  // the tile and scratch pointers re-derived from the dynamic shared-memory symbol: the compiler
  // then emits shared-space accesses (LDS / STS, 32-bit addresses) instead of generic ones (ncu
  // showed LD.E / ST.E with 64-bit address arithmetic when they arrived as plain pointers)
  extern __shared__ __align__(16) uint8_t smem_dyn[];
  uint8_t* smem_raw = smem_dyn + (smem_in - smem_dyn);
  TileView tile = tile_in;
  tile.base = reinterpret_cast<const uint16_t*>(smem_dyn + (reinterpret_cast<const uint8_t*>(tile_in.base) - smem_dyn));
  const int M = MC ? MC : M_in;
  const int gpc = GPC ? GPC : gpc_in;
  const int ng = GPC ? GPC : static_cast<int>((G - g0) < gpc ? (G - g0) : gpc);  // groups in this chunk
  const int W = gpc * M;                 // tile pitch (elements)
  const int ncols = ng * M;
  const int64_t row0 = rb * V;
  const int64_t meta_row = (G + 1) / 2;
  const int tid = threadIdx.x, nthr = NTHR ? NTHR : static_cast<int>(blockDim.x);

  constexpr int NS = CompressTileLayout::NS;
  const CompressTileLayout lay(V, W, gpc, kExpand, nbuf, tile.swz);  // scratch after the nbuf tile buffers
  float* s_part = reinterpret_cast<float*>(smem_raw + lay.part);       // [NS][W]
  double* s_score = reinterpret_cast<double*>(smem_raw + lay.score);   // [W]
  uint32_t* s_sel = reinterpret_cast<uint32_t*>(smem_raw + lay.sel);   // [gpc]
  double* s_th = reinterpret_cast<double*>(smem_raw + lay.th);         // [gpc][2]: 4th, 5th score
  uint8_t* s_rank = smem_raw + lay.rank;                               // [W]: selected?
  // kExpand: the V:2:4 re-encoding's nibbles of this tile, [V][W/8] bytes (subgroups 2j, 2j+1)
  uint8_t* s_m2 = smem_raw + lay.m2;
  (void)K;

  // ---- phase 1a: approximate column sums: thread per (8-column vector, row slice), fp32
  const int nv8 = (ncols + 7) / 8;
  const int ns = (nthr / nv8) < NS ? ((nthr / nv8) > 0 ? nthr / nv8 : 1) : NS;
  for (int t = tid; t < nv8 * ns; t += nthr) {
    const int cv = t % nv8, sl = t / nv8;
    const int r0 = (sl * V) / ns, r1 = ((sl + 1) * V) / ns;
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (!(dbg & 2))
      for (int i = r0; i < r1; ++i) {
        const uint4 w = tile.vec(i, cv);
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          a[2 * h] += fabsf(bits_to_float<kBF16>(static_cast<uint16_t>(ww[h] & 0xFFFFu)));
          a[2 * h + 1] += fabsf(bits_to_float<kBF16>(static_cast<uint16_t>(ww[h] >> 16)));
        }
      }
#pragma unroll
    for (int e = 0; e < 8; ++e) s_part[sl * W + 8 * cv + e] = a[e];
  }
  __syncthreads();
  bool bad = false;
  for (int c = tid; c < ncols; c += nthr) {
    float sum = s_part[c];
    for (int sl = 1; sl < ns; ++sl) sum += s_part[sl * W + c];
    s_score[c] = static_cast<double>(sum);
    if (!isfinite(sum)) {
      // an inf / nan input makes the sum non-finite; bf16 sums of finite values can also overflow
      // fp32, so the column itself is checked
      if constexpr (kBF16) {
        for (int i = 0; i < V; ++i) bad |= bits_non_finite<true>(tile.at(i, c));
      } else {
        bad = true;  // fp16: |a| <= 65504, so a finite column sums to < 2^40 (finite)
      }
    }
  }
  if (bad && status != nullptr) atomicMax(status, kStatusNonFinite);
  __syncthreads();

  // ---- phase 2a: rank of column j in its group by (score desc, index asc) = its place in the
  // order the format selects by (reading #5); the 4th and 5th scores of each group are kept
  // the margin test of phase 1b on a group's 4th and 5th fp32 scores (below)
  const double tol = 2.1 * static_cast<double>(V + NS) * 0x1p-24;
  auto decided = [&](int q) -> bool {
    if (M <= 4) return true;
    const double s4 = s_th[2 * q], s5 = s_th[2 * q + 1];
    return (s4 - s5) > tol * s4 && s4 < 1e30;  // false for NaN / overflow (inf - inf)
  };
  auto rank_pass = [&](bool only_flagged) {
    for (int t = tid; t < ncols; t += nthr) {
      const int q = t / M, j = t - q * M;
      if (only_flagged && decided(q)) continue;  // exact pass: flagged groups only
      const double* sc = s_score + q * M;
      const double sj = sc[j];
      int rank = 0;
      for (int i = 0; i < M; ++i) rank += (sc[i] > sj) || (sc[i] == sj && i < j);
      s_rank[t] = static_cast<uint8_t>(rank < 4 ? 1 : 0);
      if (!only_flagged) {
        if (rank == 3) s_th[2 * q] = sj;
        if (rank == 4) s_th[2 * q + 1] = sj;
      }
    }
  };
  rank_pass(false);
  __syncthreads();
  // ---- phase 1b: the margin test (evaluated by every thread that needs it, from the 4th and 5th
  // scores — no separate phase and barrier), and exact scores for the groups that fail it
  bool any_exact = false;
  for (int t = tid; t < ncols; t += nthr) {
    const int q = t / M;
    if (decided(q)) continue;
    any_exact = true;
    if constexpr (!kBF16) {
      // fp16: every |a| is k·2^-24 with an integer k < 2^40 (k = m for subnormals, (1024 + m) <<
      // (e - 1) for normals) and a column's sum stays < 2^53, so the oracle's fp64 sum is exact and
      // equals the integer sum in any order; compared in units of 2^-24 (one scale per group)
      uint64_t acc = 0;
      for (int i = 0; i < V; ++i) {
        const uint32_t hb = tile.at(i, t) & 0x7FFFu;
        const uint32_t e = hb >> 10, m = hb & 0x3FFu;
        acc += e ? (static_cast<uint64_t>(0x400u | m) << (e - 1)) : static_cast<uint64_t>(m);
      }
      s_score[t] = static_cast<double>(acc);
    } else {
      // bf16: the oracle's order (ascending rows, fp64)
      double acc = 0.0;
      for (int i = 0; i < V; ++i) acc = __dadd_rn(acc, static_cast<double>(fabsf(bits_to_float<true>(tile.at(i, t)))));
      s_score[t] = acc;
    }
  }
  if (__syncthreads_or(any_exact)) {
    rank_pass(true);
    __syncthreads();
  }
  // ---- phase 2b: the four selected columns of each group, ascending (reading #7). For M dividing
  // 32 a warp ballot of the selection flags gives every group's mask at once and the group's first
  // lane extracts the 4 set positions (the serial scan by one thread per group kept every other
  // warp waiting at the barrier below); otherwise one thread scans its group.
  if (M <= 32 && (32 % M) == 0 && ncols <= nthr) {
    const bool sel = tid < ncols && s_rank[tid] != 0;
    const uint32_t mask = __ballot_sync(0xFFFFFFFFu, sel);
    if (tid < ncols && (tid % M) == 0) {
      uint32_t m = (mask >> (tid & 31)) & (M == 32 ? 0xFFFFFFFFu : ((1u << M) - 1u));
      uint32_t word = 0;
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        word |= static_cast<uint32_t>(__ffs(m) - 1) << (8 * n);
        m &= m - 1;
      }
      const int q = tid / M;
      reinterpret_cast<uint32_t*>(column_idx)[rb * G + g0 + q] = word;
      s_sel[q] = word;
    }
  } else {
    for (int q = tid; q < ng; q += nthr) {
      uint32_t word = 0;
      int n = 0;
      for (int j = 0; j < M && n < 4; ++j)
        if (s_rank[q * M + j]) word |= static_cast<uint32_t>(j) << (8 * n++);
      reinterpret_cast<uint32_t*>(column_idx)[rb * G + g0 + q] = word;
      s_sel[q] = word;
    }
  }
  __syncthreads();

  // ---- phase 3 (plain compression): thread per (pair of groups, row) — the pair fills one
  // metadata byte and 8 value bytes; a thread keeps its pair's 8 selected column offsets in
  // registers and steps over rows (pointer increments only)
  if constexpr (!kExpand) {
    const int npr = (ng + 1) / 2;  // group pairs per row
    if (!(dbg & 4) && nthr % npr == 0) {
      const int pp = tid % npr, rs = nthr / npr;
      const int qa = 2 * pp, qb = 2 * pp + 1;
      const bool has_b = qb < ng;
      const uint32_t wa = s_sel[qa], wb = has_b ? s_sel[qb] : 0x03020100u;
      int ca[4], cb[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        ca[t] = qa * M + static_cast<int>((wa >> (8 * t)) & 0xFFu);
        cb[t] = qb * M + static_cast<int>((wb >> (8 * t)) & 0xFFu);
      }
      auto top2 = [](const uint16_t (&v)[4], uint32_t& word, uint32_t& nib) {
        // top-2 by (|a| desc, position asc): keys (|a| << 2) | (3 - t) are distinct and order the
        // candidates exactly so (|w| order for finite sign-magnitude values; ±0 tie); the two
        // largest of four keys with six min/max operations, no branches
        uint32_t k[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) k[t] = ((v[t] & 0x7FFFu) << 2) | static_cast<uint32_t>(3 - t);
        const uint32_t a = max(k[0], k[1]), b = min(k[0], k[1]), c = max(k[2], k[3]), d = min(k[2], k[3]);
        const uint32_t first = max(a, c), second = max(min(a, c), max(b, d));
        const uint32_t pa = 3u - (first & 3u), pb = 3u - (second & 3u);
        const uint32_t lo = min(pa, pb), hi = max(pa, pb);
        const uint64_t vv = static_cast<uint64_t>(v[0]) | (static_cast<uint64_t>(v[1]) << 16) |
                            (static_cast<uint64_t>(v[2]) << 32) | (static_cast<uint64_t>(v[3]) << 48);
        word = static_cast<uint32_t>((vv >> (16 * lo)) & 0xFFFFu) | (static_cast<uint32_t>((vv >> (16 * hi)) & 0xFFFFu) << 16);
        nib = lo | (hi << 2);
      };
      const int i0 = tid / npr;
      uint32_t* vrow = reinterpret_cast<uint32_t*>(values) + (row0 + i0) * G + g0 + qa;
      uint8_t* mrow = metadata + (row0 + i0) * meta_row + (g0 + qa) / 2;
      const int64_t vstep = static_cast<int64_t>(rs) * G, mstep = static_cast<int64_t>(rs) * meta_row;
      // the 8 selected columns' element offsets for row i0; a row step of rs moves every one of them
      // by the same amount when the swizzle pattern (row % 8) repeats (rs % 8 == 0)
      const bool inc = !tile.swz || (rs & 7) == 0;
      int oa[4], ob[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        oa[t] = tile.idx(i0, ca[t]);
        ob[t] = tile.idx(i0, cb[t]);
      }
      const int ostep = tile.swz ? rs * 64 : rs * tile.pitch;
      const uint16_t* tb = tile.base;
      // an odd G makes (row·G + g) odd on alternate rows: 8-byte stores only when aligned
      for (int i = i0; i < V; i += rs, vrow += vstep, mrow += mstep, tb += ostep) {
        uint16_t va[4], vb[4];
        if (inc) {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            va[t] = tb[oa[t]];
            vb[t] = tb[ob[t]];
          }
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            va[t] = tile.at(i, ca[t]);
            vb[t] = tile.at(i, cb[t]);
          }
        }
        uint32_t w0, w1, n0, n1;
        top2(va, w0, n0);
        top2(vb, w1, n1);
        if (has_b) {
          if ((reinterpret_cast<uintptr_t>(vrow) & 7) == 0) {
            *reinterpret_cast<uint2*>(vrow) = make_uint2(w0, w1);
          } else {
            vrow[0] = w0;
            vrow[1] = w1;
          }
          *mrow = static_cast<uint8_t>(n0 | (n1 << 4));
        } else {
          vrow[0] = w0;
          *mrow = static_cast<uint8_t>(n0);
        }
      }
      return;
    }
  }

  // ---- phase 3: thread per (row, group): the two largest |w| among the selected columns (2:4);
  // consecutive threads take consecutive groups of a row (coalesced value stores), the two
  // nibbles of a metadata byte are joined with a lane shuffle. When the block size is a multiple
  // of the row length a thread keeps one group and steps over rows (no divisions per item).
  const int per_row = ng + (ng & 1);  // even: lane pairs (2j, 2j+1) share a metadata byte
  const int work3 = (dbg & 4) ? 0 : V * per_row;
  const bool fixed_q = (nthr % per_row) == 0;
  for (int w0 = 0; w0 < work3; w0 += nthr) {
    const int w = w0 + tid;
    const bool act = w < work3;
    const int i = !act ? 0 : (fixed_q ? (w0 / per_row) + tid / per_row : w / per_row);
    const int q = !act ? 0 : (fixed_q ? tid % per_row : w - i * per_row);
    const bool live = act && q < ng;
    const int64_t row = row0 + i;
    uint32_t nibble = 0;
    if (live) {
      const uint32_t cw = s_sel[q];

      uint16_t v[4];
      uint32_t mag[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        v[t] = tile.at(i, q * M + static_cast<int>((cw >> (8 * t)) & 0xFFu));
        mag[t] = v[t] & 0x7FFFu;  // |w| order for finite sign-magnitude formats; ±0 tie
      }
      // top-2 by (|a| desc, position asc) with register-only selects (no local-memory indexing)
      int p0 = 0;
      uint32_t m0 = mag[0];
#pragma unroll
      for (int t = 1; t < 4; ++t)
        if (mag[t] > m0) { p0 = t; m0 = mag[t]; }
      int p1 = -1;
      uint32_t m1 = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (t != p0 && (p1 < 0 || mag[t] > m1)) { p1 = t; m1 = mag[t]; }
      const int lo = min(p0, p1), hi = max(p0, p1);
      uint16_t vlo = v[0], vhi = v[0];
#pragma unroll
      for (int t = 1; t < 4; ++t) {
        if (t == lo) vlo = v[t];
        if (t == hi) vhi = v[t];
      }
      nibble = static_cast<uint32_t>(lo | (hi << 2));
      reinterpret_cast<uint32_t*>(values)[row * G + g0 + q] =
          static_cast<uint32_t>(vlo) | (static_cast<uint32_t>(vhi) << 16);
      if constexpr (kExpand) {
        // the same matrix as V:2:4 over the original K (reading #18): per 4-column
        // subgroup the kept values (inserted zeros +0.0) and one nibble; M % 8 == 0, so the
        // group's subgroups fill whole bytes of s_m2
        const int ca = static_cast<int>((cw >> (8 * lo)) & 0xFFu), cb = static_cast<int>((cw >> (8 * hi)) & 0xFFu);
        const uint32_t va = vlo, vb = vhi;
        const int sub = M / 4;
        uint32_t* v2 = values2 + row * (K / 4) + (g0 + q) * sub;
        uint32_t nbits = 0;
        for (int u = 0; u < sub; ++u) {
          const int j0 = 4 * u;
          const bool in0 = (ca >= j0 && ca < j0 + 4), in1 = (cb >= j0 && cb < j0 + 4);
          uint32_t wv, nb;
          if (in0 && in1) {
            wv = va | (vb << 16);
            nb = static_cast<uint32_t>(ca - j0) | (static_cast<uint32_t>(cb - j0) << 2);
          } else if (in0 || in1) {
            const uint32_t x = in0 ? va : vb;
            const uint32_t ii = static_cast<uint32_t>((in0 ? ca : cb) - j0);
            wv = (ii == 0u) ? x : (x << 16);
            nb = (ii == 0u) ? 0x4u : (ii << 2);
          } else {
            wv = 0u;
            nb = 0x4u;
          }
          v2[u] = wv;
          nbits |= nb << (4 * (u & 1));
          if (u & 1) {
            s_m2[i * (W / 8) + (q * sub + u) / 2] = static_cast<uint8_t>(nbits);
            nbits = 0;
          }
        }
      }
    }
    // join the nibbles of groups (2j, 2j+1): per_row is even, so partners are adjacent lanes
    const uint32_t other = __shfl_down_sync(0xFFFFFFFFu, nibble, 1);
    if (live && (q & 1) == 0) {
      const uint32_t byte = nibble | ((q + 1 < ng ? other : 0u) << 4);
      metadata[row * meta_row + (g0 + q) / 2] = static_cast<uint8_t>(byte);
    }
  }

  if constexpr (kExpand) {
    // ---- phase 4: tensor-core order of the re-encoded metadata (venom_order_metadata's layout)
    // for the 128-row-tile lanes whose rows this CTA owns, over its k-stages of 32 subgroups
    // (W % 128 == 0 and g0·M % 128 == 0: the CTA owns whole k-stages). Rows >= R of the last
    // row tile and subgroups >= K/4 read as 0x4 nibbles.
    __syncthreads();
    const int64_t G2 = K / 4;
    const int64_t num_ks2 = (G2 + 31) / 32;
    const int64_t ks0 = (g0 * M / 4) / 32;
    const int nks = W / 128;
    const int64_t r1 = (row0 + V == R) ? ((R + 127) / 128) * 128 : row0 + V;  // rows covered
    const int nrows16 = static_cast<int>((r1 - row0) / 16);                    // 16-row bands
    // one work item = (k-stage, 16-row band, lane-in-band b in [0,8) x {k1}, kb): the band's 16 lanes
    const int items = nks * nrows16 * 16 * 4;
    for (int t = threadIdx.x; t < ((dbg & 8) ? 0 : items); t += blockDim.x) {
      const int kb = t & 3;
      const int l16 = (t >> 2) & 15;  // lane within the band: L & 15 = (L & 7) | (k1 << 3)
      const int rest = t >> 6;
      const int band = rest % nrows16;
      const int ksl = rest / nrows16;
      const int64_t ks = ks0 + ksl;
      if (ks >= num_ks2) continue;
      const int64_t ra = row0 + 16 * band + (l16 & 7);
      const int k1 = l16 >> 3;
      const int64_t mt = ra / 128;
      const int L = static_cast<int>(((ra % 128) / 16) * 16) + l16;
      const int e0 = ksl * 32 + kb * 8 + 4 * k1;  // first subgroup (tile-relative)
      uint32_t lo = 0x4444u, hi = 0x4444u;
      if (ks * 32 + kb * 8 + 4 * k1 < G2) {
        const int ia = static_cast<int>(ra - row0);
        if (ra < R) lo = s_m2[ia * (W / 8) + e0 / 2] | (static_cast<uint32_t>(s_m2[ia * (W / 8) + e0 / 2 + 1]) << 8);
        if (ra + 8 < R) hi = s_m2[(ia + 8) * (W / 8) + e0 / 2] | (static_cast<uint32_t>(s_m2[(ia + 8) * (W / 8) + e0 / 2 + 1]) << 8);
      }
      meta_tc[((mt * num_ks2 + ks) * 128 + L) * 4 + kb] = lo | (hi << 16);
    }
  }
}

template <bool kBF16, bool kExpand>
__global__ void __launch_bounds__(512) vnm_compress_tile_kernel(
    const uint16_t* __restrict__ A, int64_t R, int64_t K, int64_t lda, int V, int M, int64_t G,
    int gpc, uint16_t* __restrict__ values, uint8_t* __restrict__ metadata,
    uint8_t* __restrict__ column_idx, int32_t* __restrict__ status,
    uint32_t* __restrict__ values2, uint32_t* __restrict__ meta_tc, int dbg) {
  extern __shared__ __align__(16) uint8_t smem_dyn[];
  uint8_t* smem_raw = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  const int64_t rb = blockIdx.y;
  const int64_t g0 = static_cast<int64_t>(blockIdx.x) * gpc;
  const int ng = static_cast<int>((G - g0) < gpc ? (G - g0) : gpc);  // groups in this chunk
  const int W = gpc * M;                 // tile pitch (elements)
  const int ncols = ng * M;
  const int64_t k0 = g0 * M;
  const int64_t row0 = rb * V;
  const int64_t meta_row = (G + 1) / 2;
  const int tid = threadIdx.x, nthr = blockDim.x;
  constexpr int NS = CompressTileLayout::NS;
  const CompressTileLayout lay(V, W, gpc, kExpand);
  const int P = W + 8;                                                // padded row pitch
  uint16_t* tile = reinterpret_cast<uint16_t*>(smem_raw + lay.tile);  // [V][W + 8]
  float* s_part = reinterpret_cast<float*>(smem_raw + lay.part);       // [NS][W]
  double* s_score = reinterpret_cast<double*>(smem_raw + lay.score);   // [W]
  uint32_t* s_sel = reinterpret_cast<uint32_t*>(smem_raw + lay.sel);   // [gpc]
  double* s_th = reinterpret_cast<double*>(smem_raw + lay.th);         // [gpc][2]: 4th, 5th score
  uint8_t* s_rank = smem_raw + lay.rank;                               // [W]: selected?
  // kExpand: the V:2:4 re-encoding's nibbles of this tile, [V][W/8] bytes (subgroups 2j, 2j+1)
  uint8_t* s_m2 = smem_raw + lay.m2;

  // ---- phase 0: the block tile, 16-byte loads (8 columns) where aligned, else element-wise. With
  // a fixed (column vector, row) mapping per thread and 32-bit offsets from one base pointer, the
  // whole tile is in flight at once for a handful of instructions per load. Non-finite inputs are
  // detected from the column sums in phase 1 (an inf / nan makes its column's sum non-finite).
  const int nvec = ncols / 8;  // full 8-column vectors of a row (W % 8 == 0 by construction)
  const bool vec_ok = ((lda & 7) == 0) && ((k0 & 7) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  if (vec_ok && nvec > 0 && !(dbg & 1)) {
    if (nthr % nvec == 0 && static_cast<int64_t>(V) * (lda / 8) < (int64_t(1) << 31)) {
      constexpr int U = 8;
      const int cv = tid % nvec, rstep = nthr / nvec, i0 = tid / nvec;
      const uint32_t step = static_cast<uint32_t>(rstep * (lda / 8));  // uint4 per row step
      const uint4* src = reinterpret_cast<const uint4*>(A + (row0 + i0) * lda + k0) + cv;
      uint16_t* dst = tile + i0 * P + 8 * cv;
      const int nload = i0 < V ? (V - i0 + rstep - 1) / rstep : 0;  // rows of this thread
      for (int k = 0; k < nload; k += U) {
        uint4 w[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (k + u < nload) w[u] = __ldcs(src + static_cast<uint32_t>(k + u) * step);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (k + u < nload) *reinterpret_cast<uint4*>(dst + (k + u) * rstep * P) = w[u];
      }
    } else {
      constexpr int U = 4;
      const int nv = V * nvec;
      for (int t0 = tid; t0 < nv; t0 += U * nthr) {
        uint4 w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int t = t0 + u * nthr;
          if (t < nv) {
            const int i = t / nvec, cv = t - i * nvec;
            w[u] = __ldcs(reinterpret_cast<const uint4*>(A + (row0 + i) * lda + k0) + cv);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int t = t0 + u * nthr;
          if (t < nv) {
            const int i = t / nvec, cv = t - i * nvec;
            *reinterpret_cast<uint4*>(tile + i * P + 8 * cv) = w[u];
          }
        }
      }
    }
  }
  const int cstart = vec_ok ? 8 * nvec : 0;
  const int ntail = ncols - cstart;
  if (ntail > 0) {
    for (int t = tid; t < V * ntail; t += nthr) {
      const int i = t / ntail, c = cstart + (t - i * ntail);
      tile[i * P + c] = __ldg(A + (row0 + i) * lda + k0 + c);
    }
  }
  __syncthreads();

  compress_tile_process<kBF16, kExpand>(TileView{tile, P, 0, false}, smem_raw, R, K, V, M, G, gpc, rb, g0, values,
                                          metadata, column_idx, status, values2, meta_tc, dbg, 1);
}

// Compression, persistent TMA variant (the default when A is 16-byte aligned with a 16-byte row
// pitch, V <= 256 and W % 64 == 0): one CTA per SM slot walks the (row block, column chunk) tiles in row-major
// order; the V × W tile of the next two tiles is in flight (W / 64 TMA boxes of 64 columns with the
// 128-byte swizzle each, double-buffered,
// mbarrier-completed) while phases 1-4 run on the current one, so HBM streams continuously and
// the per-CTA prologue is paid once (the one-tile-per-CTA kernel spent its time in load latency,
// prologue and barriers: 0.61 ms for the GPT-3 FFN weight).
template <bool kBF16, bool kExpand, int MC = 0, int GPC = 0>
__global__ void __launch_bounds__(256) vnm_compress_tma_kernel(
    const __grid_constant__ CUtensorMap tm_a, int64_t R, int64_t K, int V, int M, int64_t G, int gpc,
    int64_t nchunks, int64_t ntiles, uint16_t* __restrict__ values, uint8_t* __restrict__ metadata,
    uint8_t* __restrict__ column_idx, int32_t* __restrict__ status, uint32_t* __restrict__ values2,
    uint32_t* __restrict__ meta_tc, int dbg) {
  using namespace ptx;
  extern __shared__ __align__(16) uint8_t smem_dyn[];
  uint8_t* smem_raw = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[2];
  const int W = gpc * M;
  const CompressTileLayout lay(V, W, gpc, kExpand, 2, true);
  const int nbox = (W + 63) / 64;
  const uint32_t box_stride = static_cast<uint32_t>((V * 128 + 1023) & ~1023);  // bytes per 64-column box
  const uint32_t tile_bytes = static_cast<uint32_t>(nbox) * V * 128;           // bytes the TMA delivers
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&full[0]), 1);
    mbar_init(smem_u32(&full[1]), 1);
    fence_mbar_init();
    prefetch_tmap(&tm_a);
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  auto issue = [&](int64_t rb, int64_t cc, int b) {  // thread 0: tile (rb, cc) -> buffer b
    mbar_arrive_expect_tx(smem_u32(&full[b]), tile_bytes);
    for (int x = 0; x < nbox; ++x)
      tma_load_2d(smem_u32(smem_raw + b * lay.tile_bytes + x * box_stride), &tm_a, smem_u32(&full[b]),
                  static_cast<int32_t>(cc * W + 64 * x), static_cast<int32_t>(rb * V), pol);
  };
  int64_t t = blockIdx.x;
  if (threadIdx.x == 0) {
    if (t < ntiles) issue(t / nchunks, t % nchunks, 0);
    const int64_t t1 = t + gridDim.x;
    if (t1 < ntiles) issue(t1 / nchunks, t1 % nchunks, 1);
  }
  // (row block, column chunk) of tile t, advanced by the grid stride without a division per tile
  const int64_t drb = static_cast<int64_t>(gridDim.x) / nchunks, dcc = static_cast<int64_t>(gridDim.x) - drb * nchunks;
  int64_t rb = t / nchunks, cc = t - rb * nchunks;
  for (int it = 0; t < ntiles; t += gridDim.x, ++it, rb += drb, cc += dcc) {
    if (cc >= nchunks) {
      cc -= nchunks;
      ++rb;
    }
    const int b = it & 1;
    mbar_wait(smem_u32(&full[b]), (it >> 1) & 1);
    compress_tile_process<kBF16, kExpand, MC, GPC, (MC && GPC) ? 256 : 0>(
        TileView{reinterpret_cast<const uint16_t*>(smem_raw + b * lay.tile_bytes), 0,
                                                   static_cast<int>(box_stride / 2), true}, smem_raw,
                                          R, K, V, M, G, gpc, rb, cc * gpc, values, metadata, column_idx, status,
                                          values2, meta_tc, dbg, 2);
    __syncthreads();  // every thread is done with buffer b (and the scratch) before it is refilled
    if (threadIdx.x == 0 && t + 2 * static_cast<int64_t>(gridDim.x) < ntiles) {
      int64_t rb2 = rb + 2 * drb, cc2 = cc + 2 * dcc;  // tile t + 2·grid, no division
      while (cc2 >= nchunks) {
        cc2 -= nchunks;
        ++rb2;
      }
      issue(rb2, cc2, b);
    }
  }
}

// Decompression: grid (column chunks, rows); thread per (row, kVec consecutive output elements).
// Output +0.0 except the kept positions. Validates metadata when `status` is non-null. 32-bit
// index arithmetic inside a row (K < 2^31), group/position advanced incrementally.
template <int kVec>
__global__ void __launch_bounds__(256) vnm_decompress_kernel(
    const uint16_t* __restrict__ values, const uint8_t* __restrict__ metadata,
    const uint8_t* __restrict__ column_idx, int64_t R, int64_t K, int V, int M, int64_t G,
    uint16_t* __restrict__ out, int64_t lda, int32_t* __restrict__ status) {
  const int64_t meta_row = (G + 1) / 2;
  const int kk = static_cast<int>(K);
  const int chunks = static_cast<int>((K + kVec - 1) / kVec);
  const int total = static_cast<int>(R * chunks);  // host guarantees < 2^31
  bool bad = false;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int rowi = idx / chunks;
    const int64_t row = rowi;
    const int k0 = (idx - rowi * chunks) * kVec;
    const int64_t rb = row / V;
    const uint32_t* cw_row = reinterpret_cast<const uint32_t*>(column_idx) + rb * G;
    const uint32_t* v_row = reinterpret_cast<const uint32_t*>(values) + row * G;
    const uint8_t* m_row = metadata + row * meta_row;
    int g = k0 / M;
    int j = k0 - g * M;
    uint16_t o[kVec];
    int c0 = -1, c1 = -1;
    uint16_t v0 = 0, v1 = 0;
    int cur_g = -1;
#pragma unroll
    for (int u = 0; u < kVec; ++u) {
      o[u] = 0;
      if (k0 + u < kk) {
        if (g != cur_g) {
          cur_g = g;
          const uint32_t cw = __ldg(cw_row + g);
          const uint32_t nib = (__ldg(m_row + (g >> 1)) >> (4 * (g & 1))) & 0xFu;
          const uint32_t p0 = nib & 3u, p1 = nib >> 2;
          const uint32_t ca = cw & 0xFFu, cb = (cw >> 8) & 0xFFu, cc = (cw >> 16) & 0xFFu, cd = cw >> 24;
          bad |= !(ca < cb && cb < cc && cc < cd && cd < static_cast<uint32_t>(M)) || !(p0 < p1);
          c0 = static_cast<int>((cw >> (8 * p0)) & 0xFFu);
          c1 = static_cast<int>((cw >> (8 * p1)) & 0xFFu);
          const uint32_t vv = __ldg(v_row + g);
          v0 = static_cast<uint16_t>(vv & 0xFFFFu);
          v1 = static_cast<uint16_t>(vv >> 16);
        }
        o[u] = (j == c0) ? v0 : ((j == c1) ? v1 : static_cast<uint16_t>(0));
      }
      if (++j == M) {
        j = 0;
        ++g;
      }
    }
    uint16_t* dst = out + row * lda + k0;
    if (kVec == 8 && k0 + 8 <= kk) {
      uint4 w;
      w.x = o[0] | (uint32_t(o[1]) << 16);
      w.y = o[2] | (uint32_t(o[3]) << 16);
      w.z = o[4] | (uint32_t(o[5]) << 16);
      w.w = o[6] | (uint32_t(o[7]) << 16);
      *reinterpret_cast<uint4*>(dst) = w;
    } else {
#pragma unroll
      for (int u = 0; u < kVec; ++u)
        if (k0 + u < kk) dst[u] = o[u];
    }
  }
  if (bad && status != nullptr) atomicMax(status, kStatusCorruptMetadata);
}

// Decompression fast path for M % 8 == 0 (16-byte output vectors never straddle a group):
// grid (chunk blocks, row slots); thread per (8 outputs of a row) for ROWS rows at a time, all of
// their loads issued before any store (the loads of one row alone leave HBM idle: 1.9 TB/s at the
// GPT-3 size). The two kept positions are placed with shifts, no per-element branches; the
// streamed output is written with evict-first stores (it is not re-read by the step). CPG = M / 8
// when it is a compile-time 1, 2 or 4, else 0 (runtime M).
template <int CPG, int ROWS>
__global__ void __launch_bounds__(256) vnm_decompress_m8_kernel(
    const uint32_t* __restrict__ values, const uint8_t* __restrict__ metadata,
    const uint32_t* __restrict__ column_idx, int R, int K, int V, int M, int G,
    uint16_t* __restrict__ out, int64_t lda, int32_t* __restrict__ status) {
  // thread per (group, ROWS rows) when CPG is a compile-time 1 / 2 / 4: one set of loads (value
  // pair, nibble, column word) per row fills the group's whole M outputs (CPG 16-byte stores);
  // CPG = 0 (runtime M): thread per 8-output chunk
  constexpr int NCH = CPG ? CPG : 1;
  const int cpg = CPG ? CPG : M / 8;  // 8-output chunks per group
  const int unit = blockIdx.x * blockDim.x + threadIdx.x;  // group (CPG) or chunk (runtime M)
  const int g = CPG ? unit : unit / cpg;
  if (CPG ? (unit >= G) : (unit >= K / 8)) return;
  const int jbase = CPG ? 0 : (unit - g * cpg) * 8;  // first column of this thread's chunk(s) in the group
  const int meta_row = (G + 1) / 2;
  const bool same_block = (V % ROWS) == 0;  // the ROWS rows of a slot share column_idx
  const bool check = status != nullptr;
  bool bad = false;
  for (int row0 = blockIdx.y * ROWS; row0 < R; row0 += gridDim.y * ROWS) {
    uint32_t cw[ROWS], nb[ROWS], vv[ROWS];
    const int rb0 = row0 / V;
#pragma unroll
    for (int u = 0; u < ROWS; ++u) {
      const int row = row0 + u;
      cw[u] = 0x03020100u;
      nb[u] = 0x4u;
      vv[u] = 0u;
      if (row < R) {
        cw[u] = __ldg(column_idx + static_cast<int64_t>(same_block ? rb0 : row / V) * G + g);
        nb[u] = __ldg(metadata + static_cast<int64_t>(row) * meta_row + (g >> 1));
        vv[u] = __ldcs(values + static_cast<int64_t>(row) * G + g);
      }
    }
#pragma unroll
    for (int u = 0; u < ROWS; ++u) {
      const int row = row0 + u;
      if (row >= R) break;
      const uint32_t c = cw[u];
      const uint32_t nib = (nb[u] >> (4 * (g & 1))) & 0xFu;
      const uint32_t p0 = nib & 3u, p1 = nib >> 2;
      if (check)
        bad |= !((c & 0xFFu) < ((c >> 8) & 0xFFu) && ((c >> 8) & 0xFFu) < ((c >> 16) & 0xFFu) &&
                 ((c >> 16) & 0xFFu) < (c >> 24) && (c >> 24) < static_cast<uint32_t>(M)) ||
               !(p0 < p1);
      const uint32_t c0 = (c >> (8 * p0)) & 0xFFu, c1 = (c >> (8 * p1)) & 0xFFu;  // kept columns in the group
      const uint64_t x0 = vv[u] & 0xFFFFu, x1 = vv[u] >> 16;
      uint4* dst = reinterpret_cast<uint4*>(out + static_cast<int64_t>(row) * lda + static_cast<int64_t>(g) * M + jbase);
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        // offsets of the two kept columns inside chunk k (outside [0, 8): not in it); each lands
        // in the low or high 64-bit half by a shift — no per-position branches
        const uint32_t d0 = c0 - static_cast<uint32_t>(jbase + 8 * k), d1 = c1 - static_cast<uint32_t>(jbase + 8 * k);
        uint64_t lo = 0, hi = 0;
        lo |= (d0 < 4u) ? (x0 << (16 * d0)) : 0ull;
        hi |= (d0 - 4u < 4u) ? (x0 << (16 * (d0 - 4u))) : 0ull;
        lo |= (d1 < 4u) ? (x1 << (16 * d1)) : 0ull;
        hi |= (d1 - 4u < 4u) ? (x1 << (16 * (d1 - 4u))) : 0ull;
        __stcs(dst + k, make_uint4(static_cast<uint32_t>(lo), static_cast<uint32_t>(lo >> 32), static_cast<uint32_t>(hi),
                                   static_cast<uint32_t>(hi >> 32)));
      }
    }
  }
  if (bad) atomicMax(status, kStatusCorruptMetadata);
}

// Re-encoding V:N:M (M % 4 == 0) -> V:2:4 over the original K (reading #18; the oracle's
// oracle_expand_2to4 states the rules). grid (pairs of groups, rows); thread per (row, 2 groups):
// the kept positions of each group are resolved through column_idx and the m-indices, and every
// 4-column subgroup is written as two values + one nibble. The output column_idx is the identity.
__global__ void __launch_bounds__(256) vnm_expand_2to4_kernel(
    const uint32_t* __restrict__ values, const uint8_t* __restrict__ metadata,
    const uint32_t* __restrict__ column_idx, int64_t R, int V, int M, int64_t G,
    uint32_t* __restrict__ values2, uint8_t* __restrict__ metadata2,
    uint32_t* __restrict__ column_idx2, int32_t* __restrict__ status) {
  const int npairs = static_cast<int>((G + 1) / 2);
  const int total = static_cast<int>(R * npairs);  // host guarantees < 2^31
  const int sub = M / 4;                       // subgroups per group
  const int64_t G2 = G * sub, meta_row = (G + 1) / 2, meta_row2 = (G2 + 1) / 2;
  bool bad = false;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int rowi = idx / npairs;
    const int64_t row = rowi;
    const int64_t pp = idx - rowi * npairs;
    const int64_t rb = rowi / V;
    uint32_t acc = 0;   // pending nibbles of the current output byte
    for (int h = 0; h < 2; ++h) {
      const int64_t g = 2 * pp + h;
      if (g >= G) break;
      const uint32_t cw = __ldg(column_idx + rb * G + g);
      const uint32_t nib = (__ldg(metadata + row * meta_row + (g >> 1)) >> (4 * (g & 1))) & 0xFu;
      const uint32_t p0 = nib & 3u, p1 = nib >> 2;
      // the same validity rule as vnm_decompress_kernel: m-indices ascending, column_idx strictly
      // ascending and < M
      bad |= !(p0 < p1) || !((cw & 0xFFu) < ((cw >> 8) & 0xFFu) && ((cw >> 8) & 0xFFu) < ((cw >> 16) & 0xFFu) &&
                             ((cw >> 16) & 0xFFu) < (cw >> 24) && (cw >> 24) < static_cast<uint32_t>(M));
      const int c0 = static_cast<int>((cw >> (8 * p0)) & 0xFFu);
      const int c1 = static_cast<int>((cw >> (8 * p1)) & 0xFFu);
      const uint32_t v = __ldg(values + row * G + g);
      for (int u = 0; u < sub; ++u) {
        const int j0 = 4 * u;
        const bool in0 = (c0 >= j0 && c0 < j0 + 4), in1 = (c1 >= j0 && c1 < j0 + 4);
        uint32_t w, nb;
        if (in0 && in1) {
          w = v;
          nb = static_cast<uint32_t>(c0 - j0) | (static_cast<uint32_t>(c1 - j0) << 2);
        } else if (in0 || in1) {
          const uint32_t x = in0 ? (v & 0xFFFFu) : (v >> 16);
          const uint32_t i = static_cast<uint32_t>((in0 ? c0 : c1) - j0);
          w = (i == 0u) ? x : (x << 16);
          nb = (i == 0u) ? 0x4u : (i << 2);
        } else {
          w = 0u;
          nb = 0x4u;
        }
        const int64_t j = g * sub + u;
        values2[row * G2 + j] = w;
        if (j & 1) {
          metadata2[row * meta_row2 + (j >> 1)] = static_cast<uint8_t>(acc | (nb << 4));
          acc = 0;
        } else {
          acc = nb;
          if (j == G2 - 1) metadata2[row * meta_row2 + (j >> 1)] = static_cast<uint8_t>(acc);
        }
        if (row % V == 0) column_idx2[rb * G2 + j] = 0x03020100u;
      }
    }
  }
  if (bad && status != nullptr) atomicMax(status, kStatusCorruptMetadata);
}

// Tensor-core order of the metadata (DESIGN.md §5 "prepared metadata"): the canonical nibbles
// permuted into the TMEM layout tcgen05.mma.sp reads, one 2 KB block per (128-row tile mt, k-stage
// ks of 32 groups): u32 out[mt][ks][L][kb] for lane L = 0..127 and K = 32 MMA kb = 0..3 holds the 16
// bits of groups ks·32 + kb·8 + 4·k1 .. +3 (k1 = (L >> 3) & 1) for row (L & 7) + 16·(L >> 4) in its
// low half and for that row + 8 in its high half. Rows >= R and groups >= G read as 0x4 nibbles
// (m-indices {0,1} of all-zero values). Thread per (mt, ks, L): one 16-byte store.
__global__ void __launch_bounds__(256) vnm_order_metadata_kernel(const uint8_t* __restrict__ metadata,
                                                                 int64_t R, int64_t G,
                                                                 int64_t num_ks, int64_t total,
                                                                 uint32_t* __restrict__ out) {
  // thread per output word: idx = ((mt·num_ks + ks)·128 + L)·4 + kb; metadata rows are G/2 bytes
  // (G % 4 == 0), so every 4-group chunk is one aligned 16-bit word
  // G % 4 == 0: metadata rows are G/2 bytes, every 4-group chunk one aligned 16-bit word; any
  // other G: the nibbles are read one byte at a time and groups >= G get the 0x4 code
  const int64_t meta_row = (G + 1) / 2;
  const bool words = (G % 4) == 0;
  const uint16_t* m16 = reinterpret_cast<const uint16_t*>(metadata);
  auto quad = [&](int64_t row, int64_t g0) -> uint32_t {  // nibbles of groups g0 .. g0+3
    if (row >= R || g0 >= G) return 0x4444u;
    if (words) return __ldg(m16 + row * (meta_row / 2) + g0 / 4);
    uint32_t h = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int64_t g = g0 + t;
      const uint32_t nib = g < G ? (__ldg(metadata + row * meta_row + g / 2) >> (4 * (g & 1))) & 0xFu : 0x4u;
      h |= nib << (4 * t);
    }
    return h;
  };
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int kb = static_cast<int>(idx & 3);
    const int L = static_cast<int>((idx >> 2) & 127);
    const int64_t blk = idx >> 9;  // mt * num_ks + ks
    const int64_t ks = blk % num_ks, mt = blk / num_ks;
    const int64_t ra = mt * 128 + (L & 7) + 16 * (L >> 4), rb = ra + 8;
    const int64_t g0 = 4 * (ks * 8 + kb * 2 + ((L >> 3) & 1));  // groups g0 .. g0 + 3
    out[idx] = quad(ra, g0) | (quad(rb, g0) << 16);
  }
}

// Values with the row pitch padded to G4 = ceil(G/4)·4 groups (venom_pad_values, the execution form
// for G % 4 != 0): thread per output group (two 16-bit values as one word), +0.0 past G.
__global__ void __launch_bounds__(256) vnm_pad_values_kernel(const uint32_t* __restrict__ values, int64_t R,
                                                             int64_t G, int64_t G4, uint32_t* __restrict__ out) {
  const int64_t total = R * G4;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / G4, g = i - row * G4;
    out[i] = g < G ? __ldg(values + row * G + g) : 0u;
  }
}

// Token-major activations -> feature-major B for the gathered operand (venom_spmm_ex with b_kmajor
// and M > 4): Y[k][t] = X[t][k], X = dtype[T][ldx], Y = dtype[K][T] (the caller
// guarantees K % 8 == 0, T % 8 == 0, ldx % 8 == 0 and 16-byte aligned X, Y). 64 × 64 tiles through
// shared memory stored k-major with a 72-element pitch (16-byte aligned rows): 16-byte global
// loads and stores in both passes.
__global__ void __launch_bounds__(256) vnm_transpose16_kernel(const uint16_t* __restrict__ X, int64_t T, int64_t K,
                                                              int64_t ldx, uint16_t* __restrict__ Y) {
  constexpr int P = 72;
  __shared__ __align__(16) uint16_t tile[64 * P];  // [k][t]
  const int64_t t0 = static_cast<int64_t>(blockIdx.y) * 64, k0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int vec = threadIdx.x & 7, row = threadIdx.x >> 3;  // 8 × 16-byte vectors per 64-element row
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int tl = row + 32 * j;
    const int64_t t = t0 + tl, k = k0 + 8 * vec;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (t < T && k < K) v = __ldcs(reinterpret_cast<const uint4*>(X + t * ldx + k));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 8; ++e)
      tile[(8 * vec + e) * P + tl] = static_cast<uint16_t>((w[e >> 1] >> (16 * (e & 1))) & 0xFFFFu);
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int kl = row + 32 * j;
    const int64_t k = k0 + kl, t = t0 + 8 * vec;
    if (k < K && t < T)
      *reinterpret_cast<uint4*>(Y + k * T + t) = *reinterpret_cast<const uint4*>(tile + kl * P + 8 * vec);
  }
}

// ------------------------------------------------------------------ masked compression
// venom_compress_masked (include/venom.h; reading #20): the kept set comes from an
// external V:N:M mask. One thread per (row block, pair of groups) so that every metadata byte has
// a single writer. Per group: the block's kept columns (a bitmap over M <= 256 columns), completed
// to four with the lowest free columns; per row the kept m-indices, completed to two with the
// lowest free ones; raw bits for kept entries, +0.0 for filled ones. Offline (once per weight):
// exact and simple rather than fast.
constexpr int kStatusInvalidMask = 10;

template <bool kBF16>
__global__ void vnm_compress_masked_kernel(const uint16_t* __restrict__ A, const uint8_t* __restrict__ mask,
                                           int64_t R, int64_t K, int64_t lda, int64_t ldm, int V, int M,
                                           int64_t G, uint16_t* __restrict__ values,
                                           uint8_t* __restrict__ metadata, uint8_t* __restrict__ column_idx,
                                           int32_t* __restrict__ status) {
  const int64_t H = (G + 1) / 2;  // metadata bytes per row
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= (R / V) * H) return;
  const int64_t rb = t / H, h = t - rb * H;
  bool bad = false, invalid = false;
  for (int64_t i = rb * V; i < rb * V + V; ++i) {
    const uint16_t* arow = A + i * lda;
    for (int64_t k = 2 * h * M; k < (2 * h + 2) * M && k < K; ++k) bad |= bits_non_finite<kBF16>(arow[k]);
  }
  for (int gg = 0; gg < 2; ++gg) {
    const int64_t g = 2 * h + gg;
    if (g >= G) break;
    // kept columns of the block
    uint32_t used[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t i = rb * V; i < rb * V + V; ++i) {
      const uint8_t* mrow = mask + i * ldm + g * M;
      for (int j = 0; j < M; ++j)
        if (mrow[j]) used[j >> 5] |= 1u << (j & 31);
    }
    int n = 0;
    for (int w = 0; w < 8; ++w) n += __popc(used[w]);
    if (n > 4) invalid = true;
    int c[4] = {0, 1, 2, 3};
    {
      int fill = 4 - n, q = 0;
      for (int j = 0; j < M && q < 4; ++j) {
        const bool u = (used[j >> 5] >> (j & 31)) & 1u;
        if (u || fill > 0) {
          if (!u) --fill;
          c[q++] = j;
        }
      }
    }
    const uint32_t word = static_cast<uint32_t>(c[0]) | (static_cast<uint32_t>(c[1]) << 8) |
                          (static_cast<uint32_t>(c[2]) << 16) | (static_cast<uint32_t>(c[3]) << 24);
    reinterpret_cast<uint32_t*>(column_idx)[rb * G + g] = word;
    for (int64_t i = rb * V; i < rb * V + V; ++i) {
      const uint8_t* mrow = mask + i * ldm + g * M;
      int keep[4], np = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        keep[q] = mrow[c[q]] != 0;
        np += keep[q];
      }
      if (np > 2) invalid = true;
      int p0 = -1, p1 = -1, need = 2 - np;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        bool take = keep[q];
        if (!take && need > 0) {
          take = true;
          --need;
        }
        if (take) {
          if (p0 < 0) p0 = q;
          else if (p1 < 0) p1 = q;
        }
      }
      if (p1 < 0) p1 = (p0 == 3) ? 2 : 3;  // only on invalid masks (outputs undefined)
      const uint16_t* arow = A + i * lda + g * M;
      const uint16_t v0 = keep[p0] ? arow[c[p0]] : static_cast<uint16_t>(0);
      const uint16_t v1 = keep[p1] ? arow[c[p1]] : static_cast<uint16_t>(0);
      reinterpret_cast<uint32_t*>(values)[i * G + g] = static_cast<uint32_t>(v0) | (static_cast<uint32_t>(v1) << 16);
      const uint8_t nib = static_cast<uint8_t>(p0 | (p1 << 2));
      uint8_t* mb = metadata + i * H + h;
      *mb = (gg == 0) ? nib : static_cast<uint8_t>(*mb | (nib << 4));
    }
  }
  if (status != nullptr) {
    if (bad) atomicMax(status, kStatusNonFinite);
    if (invalid) atomicMax(status, kStatusInvalidMask);
  }
}

// ------------------------------------------------------------------ energy
// out[0] += Σ|values|, out[1] += Σ|A| in fp64: rows of A grid-strided over CTAs, columns over
// threads (coalesced); one warp-shuffle + shared-memory reduction and two atomics per CTA.
template <bool kBF16>
__global__ void __launch_bounds__(256) vnm_energy_kernel(const uint16_t* __restrict__ A, int64_t R, int64_t K,
                                                         int64_t lda, const uint16_t* __restrict__ values,
                                                         int64_t nv, double* __restrict__ out) {
  double kept = 0.0, all = 0.0;
  for (int64_t i = blockIdx.x; i < R; i += gridDim.x) {
    const uint16_t* row = A + i * lda;
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) all += static_cast<double>(fabsf(bits_to_float<kBF16>(row[k])));
  }
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < nv;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x)
    kept += static_cast<double>(fabsf(bits_to_float<kBF16>(values[v])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kept += __shfl_xor_sync(0xFFFFFFFFu, kept, o);
    all += __shfl_xor_sync(0xFFFFFFFFu, all, o);
  }
  __shared__ double sk[8], sa[8];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sk[w] = kept;
    sa[w] = all;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double k2 = 0.0, a2 = 0.0;
    for (int j = 0; j < static_cast<int>(blockDim.x >> 5); ++j) {
      k2 += sk[j];
      a2 += sa[j];
    }
    atomicAdd(out, k2);
    atomicAdd(out + 1, a2);
  }
}

__global__ void vnm_energy_finish_kernel(double* out) {
  out[2] = (out[1] == 0.0) ? 1.0 : out[0] / out[1];
}

// C = bias (or 0) when K == 0 (no groups): nothing to multiply. transposed: C^T[t][r] layout.
__global__ void vnm_fill_bias_kernel(uint16_t* C, int64_t R, int64_t T, int64_t ldc, const uint16_t* bias,
                                     int transposed) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= R * T) return;
  const int64_t r = idx / T, t = idx - r * T;
  C[transposed ? t * ldc + r : r * ldc + t] = bias ? bias[r] : static_cast<uint16_t>(0);
}

}  // namespace venom
