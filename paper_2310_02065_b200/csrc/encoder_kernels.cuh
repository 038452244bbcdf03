// encoder_kernels.cuh — layout kernels for the sparse BERT encoder (include/venom_encoder.h).
// Not part of the V:N:M method: they convert activations between the token-major layout that
// attention / LayerNorm use and the feature-major B operand of the SpMM (reading #14).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

namespace venom {

template <bool kBF16>
__device__ __forceinline__ float enc_to_f(uint16_t b) {
  if constexpr (kBF16) return __uint_as_float(static_cast<uint32_t>(b) << 16);
  else return __half2float(__ushort_as_half(b));
}
template <bool kBF16>
__device__ __forceinline__ uint16_t enc_from_f(float v) {
  if constexpr (kBF16) return __bfloat16_as_ushort(__float2bfloat16_rn(v));
  else return __half_as_ushort(__float2half_rn(v));
}

// Residual add + LayerNorm, token-major in and out, plus the transposed (feature-major) copy.
// CTA = 32 tokens, 8 warps × 4 tokens; a lane owns NV chunks of 8 features (h = 256·NV). The
// normalised rows are staged in shared memory with an odd word pitch (h + 2 halves) so the
// transposed pass (lane = token, one feature per step) reads conflict-free and each warp store
// writes 64 contiguous bytes of a feature row.
template <bool kBF16, int NV>
__global__ void __launch_bounds__(256) vnm_enc_add_layernorm_kernel(
    const uint16_t* __restrict__ x, const uint16_t* __restrict__ y, const uint16_t* __restrict__ w,
    const uint16_t* __restrict__ bb, int64_t T, float eps, uint16_t* __restrict__ out_tm,
    uint16_t* __restrict__ out_fm, int64_t ld_fm) {
  constexpr int H = 256 * NV;
  constexpr int P = H + 2;  // tile pitch (halves): an odd number of 32-bit words
  extern __shared__ __align__(16) uint16_t tile[];  // [32][P]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * 32;
  float wf[NV][8], bf[NV][8];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int f0 = 8 * (lane + 32 * i);
    const uint4 wv = *reinterpret_cast<const uint4*>(w + f0);
    const uint4 bv = *reinterpret_cast<const uint4*>(bb + f0);
    const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w}, bw[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      wf[i][e] = enc_to_f<kBF16>(static_cast<uint16_t>(ww[e >> 1] >> (16 * (e & 1))));
      bf[i][e] = enc_to_f<kBF16>(static_cast<uint16_t>(bw[e >> 1] >> (16 * (e & 1))));
    }
  }
  for (int tt = 0; tt < 4; ++tt) {
    const int tl = 4 * warp + tt;
    const int64_t t = t0 + tl;
    float z[NV][8];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int f0 = 8 * (lane + 32 * i);
      const uint4 xv = *reinterpret_cast<const uint4*>(x + t * H + f0);
      const uint4 yv = *reinterpret_cast<const uint4*>(y + t * H + f0);
      const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w}, yw[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        z[i][e] = enc_to_f<kBF16>(static_cast<uint16_t>(xw[e >> 1] >> (16 * (e & 1)))) +
                  enc_to_f<kBF16>(static_cast<uint16_t>(yw[e >> 1] >> (16 * (e & 1))));
        s += z[i][e];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    const float mean = s / H;
    float v = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float d = z[i][e] - mean;
        v += d * d;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    const float rstd = rsqrtf(v / H + eps);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int f0 = 8 * (lane + 32 * i);
      uint32_t o4[4];
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        const uint16_t lo = enc_from_f<kBF16>((z[i][e] - mean) * rstd * wf[i][e] + bf[i][e]);
        const uint16_t hi = enc_from_f<kBF16>((z[i][e + 1] - mean) * rstd * wf[i][e + 1] + bf[i][e + 1]);
        o4[e >> 1] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
      }
      *reinterpret_cast<uint4*>(out_tm + t * H + f0) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
      if (out_fm != nullptr) {
        uint32_t* trow = reinterpret_cast<uint32_t*>(tile + tl * P + f0);  // 4-byte aligned
#pragma unroll
        for (int e = 0; e < 4; ++e) trow[e] = o4[e];
      }
    }
  }
  if (out_fm == nullptr) return;
  __syncthreads();
  // feature-major: warp handles features f = warp, warp + 8, ...; lane = token
  for (int f = warp; f < H; f += 8) out_fm[f * ld_fm + t0 + lane] = tile[lane * P + f];
}

// Attention output a[b][h][s][d] (D = 64 contiguous) -> out_fm[h*64 + d][b*S + s]: one CTA per
// (b, h, 64-token block) transposes a 64 × 64 tile through shared memory.
template <bool kBF16>
__global__ void __launch_bounds__(256) vnm_enc_heads_to_fm_kernel(
    const uint16_t* __restrict__ a, int64_t H, int64_t S, int64_t sb, int64_t sh, int64_t ss,
    uint16_t* __restrict__ out_fm, int64_t ld_fm) {
  constexpr int P = 72;  // 64 + 8 halves: 16-byte aligned rows
  __shared__ __align__(16) uint16_t tile[64 * P];
  const int64_t nsb = S / 64;
  const int64_t blk = blockIdx.x;
  const int64_t sbk = blk % nsb, hh = (blk / nsb) % H, b = blk / (nsb * H);
  const int64_t s0 = sbk * 64;
  const uint16_t* src = a + b * sb + hh * sh + s0 * ss;
  for (int i = threadIdx.x; i < 64 * 8; i += 256) {
    const int s = i >> 3, c = i & 7;
    *reinterpret_cast<uint4*>(tile + s * P + 8 * c) = *reinterpret_cast<const uint4*>(src + s * ss + 8 * c);
  }
  __syncthreads();
  uint16_t* dst = out_fm + (hh * 64) * ld_fm + b * S + s0;
  for (int i = threadIdx.x; i < 64 * 32; i += 256) {
    const int d = i >> 5, sp = i & 31;  // token pair sp: tokens 2sp, 2sp+1
    const uint32_t v = static_cast<uint32_t>(tile[(2 * sp) * P + d]) |
                       (static_cast<uint32_t>(tile[(2 * sp + 1) * P + d]) << 16);
    *reinterpret_cast<uint32_t*>(dst + d * ld_fm + 2 * sp) = v;
  }
}

}  // namespace venom
