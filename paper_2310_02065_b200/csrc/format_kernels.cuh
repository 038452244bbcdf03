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
//   phase 1: thread per column: s = Σ_{rows ascending} |a| in fp64 (coalesced row sweeps)
//   phase 2: thread per group: top-4 columns by (s desc, index asc), sorted ascending
//   phase 3: thread per (row, pair of groups): top-2 of the 4 by (|a| desc, position asc),
//            raw-bit value copy, nibble packing — one metadata byte and 8 value bytes per thread.
template <bool kBF16>
__global__ void __launch_bounds__(256) vnm_compress_kernel(
    const uint16_t* __restrict__ A, int64_t R, int64_t K, int64_t lda, int V, int M, int64_t G,
    int gpc, uint16_t* __restrict__ values, uint8_t* __restrict__ metadata,
    uint8_t* __restrict__ column_idx, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  double* s_score = reinterpret_cast<double*>(smem_raw);                       // gpc * M
  uint8_t* s_sel = smem_raw + sizeof(double) * static_cast<size_t>(gpc) * M;   // gpc * 4

  const int64_t rb = blockIdx.y;
  const int64_t g0 = static_cast<int64_t>(blockIdx.x) * gpc;
  const int ng = static_cast<int>((G - g0) < gpc ? (G - g0) : gpc);  // groups in this chunk
  const int ncols = ng * M;
  const int64_t k0 = g0 * M;
  const int64_t row0 = rb * V;
  const int64_t meta_row = (G + 1) / 2;

  // ---- phase 1: column L1 mass, fp64, ascending rows (exact for fp16; fixed order for bf16)
  bool bad = false;
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
    const uint16_t* col = A + row0 * lda + k0 + c;
    double s = 0.0;
    int i = 0;
    for (; i + 8 <= V; i += 8) {
      uint16_t b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) b[u] = __ldg(col + static_cast<int64_t>(i + u) * lda);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        bad |= bits_non_finite<kBF16>(b[u]);
        s = __dadd_rn(s, static_cast<double>(fabsf(bits_to_float<kBF16>(b[u]))));
      }
    }
    for (; i < V; ++i) {
      uint16_t b = __ldg(col + static_cast<int64_t>(i) * lda);
      bad |= bits_non_finite<kBF16>(b);
      s = __dadd_rn(s, static_cast<double>(fabsf(bits_to_float<kBF16>(b))));
    }
    s_score[c] = s;
  }
  if (bad && status != nullptr) atomicMax(status, kStatusNonFinite);
  __syncthreads();

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

// Decompression: thread per (row, 8 consecutive output elements). Output +0.0 except the kept
// positions. Validates metadata when `status` is non-null.
template <int kVec>
__global__ void __launch_bounds__(256) vnm_decompress_kernel(
    const uint16_t* __restrict__ values, const uint8_t* __restrict__ metadata,
    const uint8_t* __restrict__ column_idx, int64_t R, int64_t K, int V, int M, int64_t G,
    uint16_t* __restrict__ out, int64_t lda, int32_t* __restrict__ status) {
  const int64_t meta_row = (G + 1) / 2;
  const int64_t chunks = (K + kVec - 1) / kVec;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= R * chunks) return;
  const int64_t row = idx / chunks;
  const int64_t k0 = (idx - row * chunks) * kVec;
  const int64_t rb = row / V;
  uint16_t o[kVec];
  int64_t cur_g = -1;
  int c0 = 0, c1 = 0;
  uint16_t v0 = 0, v1 = 0;
  bool bad = false;
#pragma unroll
  for (int u = 0; u < kVec; ++u) {
    const int64_t k = k0 + u;
    o[u] = 0;
    if (k >= K) continue;
    const int64_t g = k / M;
    if (g != cur_g) {
      cur_g = g;
      const uint32_t cw = __ldg(reinterpret_cast<const uint32_t*>(column_idx) + rb * G + g);
      const int c[4] = {int(cw & 0xFF), int((cw >> 8) & 0xFF), int((cw >> 16) & 0xFF),
                        int(cw >> 24)};
      const uint32_t nib = (__ldg(metadata + row * meta_row + g / 2) >> (4 * (g & 1))) & 0xF;
      const int p0 = nib & 3, p1 = nib >> 2;
      bad |= !(c[0] < c[1] && c[1] < c[2] && c[2] < c[3] && c[3] < M) || !(p0 < p1);
      c0 = c[p0];
      c1 = c[p1];
      const uint32_t vv = __ldg(reinterpret_cast<const uint32_t*>(values) + row * G + g);
      v0 = static_cast<uint16_t>(vv & 0xFFFF);
      v1 = static_cast<uint16_t>(vv >> 16);
    }
    const int j = static_cast<int>(k - g * M);
    o[u] = (j == c0) ? v0 : ((j == c1) ? v1 : static_cast<uint16_t>(0));
  }
  if (bad && status != nullptr) atomicMax(status, kStatusCorruptMetadata);
  uint16_t* dst = out + row * lda + k0;
  if (kVec == 8 && k0 + 8 <= K) {
    uint4 w;
    w.x = o[0] | (uint32_t(o[1]) << 16);
    w.y = o[2] | (uint32_t(o[3]) << 16);
    w.z = o[4] | (uint32_t(o[5]) << 16);
    w.w = o[6] | (uint32_t(o[7]) << 16);
    *reinterpret_cast<uint4*>(dst) = w;
  } else {
#pragma unroll
    for (int u = 0; u < kVec; ++u)
      if (k0 + u < K) dst[u] = o[u];
  }
}

}  // namespace venom
