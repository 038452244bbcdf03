// format_kernels.cuh — the V:N:M compressor and decompressor for sm_100a (HBM-bound kernels).
//
// venom_compress implements PAPER.md:187-189 (§3, Fig 2 ④): per V×M block pick the four most
// significant columns, then per row the two largest weights among them; PAPER.md:192-195 (Fig 3)
// fixes the three output arrays. The readings DESIGN.md lists (#1 L1 over the block's rows in fp64,
// ascending rows; #3 two-stage greedy; #5/#6 ties -> lower index; #7 ascending storage; #8 nibble
// packing) are what make the output byte-identical to the CPU oracle.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

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
  const int k0 = (blockIdx.x * blockDim.x + threadIdx.x) * kVec;
  if (k0 >= kk) return;
  bool bad = false;
  for (int64_t row = blockIdx.y; row < R; row += gridDim.y) {
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

// Re-encoding V:N:M (M % 4 == 0) -> V:2:4 over the original K (reading #18; the oracle's
// oracle_expand_2to4 states the rules). grid (pairs of groups, rows); thread per (row, 2 groups):
// the kept positions of each group are resolved through column_idx and the m-indices, and every
// 4-column subgroup is written as two values + one nibble. The output column_idx is the identity.
__global__ void __launch_bounds__(256) vnm_expand_2to4_kernel(
    const uint32_t* __restrict__ values, const uint8_t* __restrict__ metadata,
    const uint32_t* __restrict__ column_idx, int64_t R, int V, int M, int64_t G,
    uint32_t* __restrict__ values2, uint8_t* __restrict__ metadata2,
    uint32_t* __restrict__ column_idx2, int32_t* __restrict__ status) {
  const int64_t npairs = (G + 1) / 2;
  const int64_t pp = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pp >= npairs) return;
  const int sub = M / 4;                       // subgroups per group
  const int64_t G2 = G * sub, meta_row = (G + 1) / 2, meta_row2 = (G2 + 1) / 2;
  bool bad = false;
  for (int64_t row = blockIdx.y; row < R; row += gridDim.y) {
    const int64_t rb = row / V;
    uint32_t acc = 0;   // pending nibbles of the current output byte
    for (int h = 0; h < 2; ++h) {
      const int64_t g = 2 * pp + h;
      if (g >= G) break;
      const uint32_t cw = __ldg(column_idx + rb * G + g);
      const uint32_t nib = (__ldg(metadata + row * meta_row + (g >> 1)) >> (4 * (g & 1))) & 0xFu;
      const uint32_t p0 = nib & 3u, p1 = nib >> 2;
      bad |= !(p0 < p1) || ((cw >> 24) >= static_cast<uint32_t>(M));
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

}  // namespace venom
