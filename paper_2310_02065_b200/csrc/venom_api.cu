// venom_api.cu — the C ABI of libvenom (include/venom.h): argument validation, TMA descriptor
// encoding and kernel launch. All compute runs in the kernels of format_kernels.cuh and
// spmm_kernel.cuh; this file only marshals.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "../../include/venom.h"
#include "../../include/venom_encoder.h"
#include "format_kernels.cuh"
#include "spmm_launch.cuh"
#include "encoder_kernels.cuh"

namespace {

using venom::SpmmParams;
using venom::launch::EncodeTiledFn;
using venom::launch::launch_status;

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

venom_status_t check_arch() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return VENOM_ERR_CUDA;
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
    return VENOM_ERR_CUDA;
  if (major != 10 || minor != 0) return VENOM_ERR_ARCH;  // built for sm_100a only
  return VENOM_OK;
}

venom_status_t validate_format(int64_t R, int64_t K, venom_format_t f) {
  if (R < 0 || K < 0 || f.v < 1) return VENOM_ERR_INVALID_ARGUMENT;
  if (f.n != 2 || f.m < 4 || f.m > 256) return VENOM_ERR_UNSUPPORTED_PATTERN;
  if (R % f.v != 0) return VENOM_ERR_NON_DIVISIBLE_ROWS;
  if (K % f.m != 0) return VENOM_ERR_NON_DIVISIBLE_COLS;
  return VENOM_OK;
}

bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// compressor tile kernel: threads per CTA and the largest V × W tile (bytes); a smaller tile with
// fewer threads keeps more independent CTAs per SM (their load and compute phases overlap)
#ifndef VENOM_COMPRESS_THREADS
#define VENOM_COMPRESS_THREADS 256
#endif
#ifndef VENOM_COMPRESS_TILE_BYTES
#define VENOM_COMPRESS_TILE_BYTES 32768
#endif
constexpr int kCompressThreads = VENOM_COMPRESS_THREADS;
constexpr int64_t kCompressTileBytes = VENOM_COMPRESS_TILE_BYTES;

// ablation flags for the analysis tools (VENOM_DEBUG_FLAGS): honoured only by the separate
// -DVENOM_ABLATION build (libvenom_ablation.so); the production library always passes 0
int debug_flags() {
#ifdef VENOM_ABLATION
  const char* d = getenv("VENOM_DEBUG_FLAGS");
  return d ? atoi(d) : 0;
#else
  return 0;
#endif
}

// The persistent TMA compressor applies when A can be described by a tensor map (16-byte aligned
// base and row pitch) and the V × W tile is one TMA box (each box dimension <= 256 elements).
bool tma_compress_ok(const void* A, int64_t lda, int V, int W) {
  return aligned(A, 16) && (lda % 8 == 0) && V <= 256 && W <= 256 && (W % 64 == 0) && encode_fn() != nullptr;
}

template <typename Kern>
venom_status_t launch_compress_tma(Kern kern, const void* A, int64_t R, int64_t K, int64_t lda, venom_format_t f,
                                   int gt, bool expand, void* values, uint8_t* metadata, uint8_t* column_idx,
                                   int32_t* dev_status, uint32_t* values2, uint32_t* meta_tc, cudaStream_t s) {
  const int W = gt * f.m;
  const int64_t G = K / f.m;
  CUtensorMap tm;
  {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(R)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(2 * lda)};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(f.v)};  // 64-column boxes, 128-byte swizzle
    cuuint32_t es[2] = {1, 1};
    if (encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(A), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return VENOM_ERR_CUDA;
  }
  const size_t smem = venom::CompressTileLayout(f.v, W, gt, expand, 2, true).total;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
    return VENOM_ERR_CUDA;
  const int64_t nchunks = (G + gt - 1) / gt, ntiles = nchunks * (R / f.v);
  int per_sm = static_cast<int>((227 * 1024) / (smem + 1024));
  if (per_sm > 8) per_sm = 8;
  if (per_sm < 1) per_sm = 1;
  const int64_t cap = static_cast<int64_t>(venom::launch::sm_count()) * per_sm;
  const unsigned grid = static_cast<unsigned>(ntiles < cap ? ntiles : cap);
  kern<<<grid, 256, smem, s>>>(tm, R, K, f.v, f.m, G, gt, nchunks, ntiles, static_cast<uint16_t*>(values), metadata,
                               column_idx, dev_status, values2, meta_tc, debug_flags());
  return launch_status();
}

}  // namespace

extern "C" {

const char* venom_version(void) { return "venom-b200 0.1 (sm_100a)"; }

int32_t venom_kernels_per_call(void) { return 1; }

const char* venom_status_string(venom_status_t s) {
  switch (s) {
    case VENOM_OK: return "ok";
    case VENOM_ERR_INVALID_ARGUMENT: return "invalid argument";
    case VENOM_ERR_NON_DIVISIBLE_ROWS: return "V does not divide R";
    case VENOM_ERR_NON_DIVISIBLE_COLS: return "M does not divide K";
    case VENOM_ERR_UNSUPPORTED_PATTERN: return "unsupported V:N:M pattern";
    case VENOM_ERR_UNSUPPORTED_DTYPE: return "unsupported dtype";
    case VENOM_ERR_NON_FINITE: return "non-finite input";
    case VENOM_ERR_CORRUPT_METADATA: return "corrupt metadata";
    case VENOM_ERR_ARCH: return "device is not sm_100";
    case VENOM_ERR_CUDA: return "CUDA error";
    case VENOM_ERR_INVALID_MASK: return "mask is not V:N:M";
  }
  return "unknown status";
}

venom_status_t venom_compressed_sizes(int64_t R, int64_t K, venom_format_t f, int64_t* values_elems,
                                      int64_t* metadata_bytes, int64_t* column_idx_bytes) {
  venom_status_t st = validate_format(R, K, f);
  if (st != VENOM_OK) return st;
  const int64_t G = K / f.m;
  if (values_elems) *values_elems = R * G * 2;
  if (metadata_bytes) *metadata_bytes = R * ((G + 1) / 2);
  if (column_idx_bytes) *column_idx_bytes = (R / f.v) * G * 4;
  return VENOM_OK;
}

venom_status_t venom_compress(const void* A, int64_t R, int64_t K, int64_t lda, venom_dtype_t dt,
                              venom_format_t f, void* values, uint8_t* metadata,
                              uint8_t* column_idx, int32_t* dev_status, venom_stream_t stream) {
  venom_status_t st = validate_format(R, K, f);
  if (st != VENOM_OK) return st;
  if (dt != VENOM_F16 && dt != VENOM_BF16) return VENOM_ERR_UNSUPPORTED_DTYPE;
  if (lda < K) return VENOM_ERR_INVALID_ARGUMENT;
  if (R == 0 || K == 0) return VENOM_OK;
  if (!A || !values || !metadata || !column_idx) return VENOM_ERR_INVALID_ARGUMENT;
  if (!aligned(values, 8) || !aligned(column_idx, 4) || !aligned(A, 2)) return VENOM_ERR_INVALID_ARGUMENT;
  if ((st = check_arch()) != VENOM_OK) return st;
  const int64_t G = K / f.m;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t nrb = R / f.v;
  // grid.y is limited to 65535: row blocks beyond it are compressed by further launches on
  // row-offset views (every kernel addresses rows relative to its pointers)
  constexpr int64_t kMaxRowBlocks = 65535;
  {
    // shared-memory tile kernel: ~256 columns per CTA (even number of groups, W % 8 == 0), the
    // V × W tile at most kCompressTileBytes; narrower chunks when the grid would have < 2 CTAs per SM
    int gt = 256 / f.m;
    gt -= gt & 1;
    if (gt < 2) gt = 2;
    while ((gt * f.m) % 8 != 0) gt += 2;
    while (gt > 2 && static_cast<int64_t>(f.v) * gt * f.m * 2 > kCompressTileBytes) gt -= 2;
    while ((gt * f.m) % 8 != 0 && gt > 2) gt -= 2;
    if (gt > G + (G & 1)) gt = static_cast<int>(G + (G & 1));
    while ((gt * f.m) % 8 != 0) gt += 2;  // pitch alignment (may exceed G: extra columns unused)
    while (gt >= 8 && ((G + gt - 1) / gt) * nrb < 2 * 148 && ((gt / 2) * f.m) % 8 == 0 && (gt / 2) % 2 == 0)
      gt /= 2;
    const size_t tsmem = venom::CompressTileLayout(f.v, gt * f.m, gt, false).total;
    if (tsmem <= 100 * 1024 && tma_compress_ok(A, lda, f.v, gt * f.m)) {
      auto kern = (dt == VENOM_BF16) ? venom::vnm_compress_tma_kernel<true, false>
                                     : venom::vnm_compress_tma_kernel<false, false>;
      // compile-time shapes (no per-tile divisions) for the configurations the benchmarks run
      const bool full = G % gt == 0;
      if (full && f.m == 16 && gt == 8)
        kern = (dt == VENOM_BF16) ? venom::vnm_compress_tma_kernel<true, false, 16, 8>
                                  : venom::vnm_compress_tma_kernel<false, false, 16, 8>;
      else if (full && f.m == 8 && gt == 32)
        kern = (dt == VENOM_BF16) ? venom::vnm_compress_tma_kernel<true, false, 8, 32>
                                  : venom::vnm_compress_tma_kernel<false, false, 8, 32>;
      else if (full && f.m == 32 && gt == 4)
        kern = (dt == VENOM_BF16) ? venom::vnm_compress_tma_kernel<true, false, 32, 4>
                                  : venom::vnm_compress_tma_kernel<false, false, 32, 4>;
      return launch_compress_tma(kern, A, R, K, lda, f, gt, false, values, metadata, column_idx, dev_status,
                                 nullptr, nullptr, s);
    }
    if (tsmem <= 100 * 1024) {
      auto kern = (dt == VENOM_BF16) ? venom::vnm_compress_tile_kernel<true, false>
                                     : venom::vnm_compress_tile_kernel<false, false>;
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(tsmem)) != cudaSuccess)
        return VENOM_ERR_CUDA;
      for (int64_t rb0 = 0; rb0 < nrb; rb0 += kMaxRowBlocks) {
        const int64_t nb = (nrb - rb0) < kMaxRowBlocks ? (nrb - rb0) : kMaxRowBlocks;
        const int64_t r0 = rb0 * f.v;
        const dim3 grid(static_cast<unsigned>((G + gt - 1) / gt), static_cast<unsigned>(nb));
        kern<<<grid, kCompressThreads, tsmem, s>>>(
            static_cast<const uint16_t*>(A) + r0 * lda, nb * f.v, K, lda, f.v, f.m, G, gt,
            static_cast<uint16_t*>(values) + r0 * G * 2, metadata + r0 * ((G + 1) / 2), column_idx + rb0 * G * 4,
            dev_status, nullptr, nullptr, debug_flags());
        if ((st = launch_status()) != VENOM_OK) return st;
      }
      return VENOM_OK;
    }
  }
  // very tall blocks: streaming kernel (partial sums over row ranges, no tile copy)
  // ~256 columns per CTA (whole, even number of groups), so that R/V × K/256 CTAs stream A
  int gpc = 256 / f.m;
  gpc -= gpc & 1;
  if (gpc < 2) gpc = 2;
  if (gpc > G + (G & 1)) gpc = static_cast<int>(G + (G & 1));
  // latency hiding: at least ~4 CTAs per SM (narrower column chunks when R/V × K/256 is small)
  while (gpc >= 4 && ((G + gpc - 1) / gpc) * nrb < 4 * 148) gpc = (gpc / 2) & ~1;
  const bool vec = aligned(A, 16) && (lda % 8 == 0) && ((static_cast<int64_t>(gpc) * f.m) % 8 == 0);
  const int wmax = gpc * f.m;
  const int vecw = vec ? 8 : 1;
  const int ncv_max = (wmax + vecw - 1) / vecw;
  const int nsplit_max = (dt == VENOM_BF16) ? 1 : (256 / ncv_max > 0 ? 256 / ncv_max : 1);
  const size_t smem = sizeof(double) * static_cast<size_t>(nsplit_max) * wmax + 4 * static_cast<size_t>(gpc);
  for (int64_t rb0 = 0; rb0 < nrb; rb0 += kMaxRowBlocks) {
    const int64_t nb = (nrb - rb0) < kMaxRowBlocks ? (nrb - rb0) : kMaxRowBlocks;
    const int64_t r0 = rb0 * f.v;
    const dim3 grid(static_cast<unsigned>((G + gpc - 1) / gpc), static_cast<unsigned>(nb));
    const uint16_t* Ar = static_cast<const uint16_t*>(A) + r0 * lda;
    uint16_t* vr = static_cast<uint16_t*>(values) + r0 * G * 2;
    uint8_t* mr = metadata + r0 * ((G + 1) / 2);
    uint8_t* cr = column_idx + rb0 * G * 4;
#define VENOM_COMPRESS(BF, VW) \
  venom::vnm_compress_kernel<BF, VW><<<grid, 256, smem, s>>>(Ar, nb * f.v, K, lda, f.v, f.m, G, gpc, vr, mr, cr, dev_status)
    if (dt == VENOM_BF16) {
      if (vec) VENOM_COMPRESS(true, 8); else VENOM_COMPRESS(true, 1);
    } else {
      if (vec) VENOM_COMPRESS(false, 8); else VENOM_COMPRESS(false, 1);
    }
#undef VENOM_COMPRESS
    if ((st = launch_status()) != VENOM_OK) return st;
  }
  return VENOM_OK;
}

venom_status_t venom_compress_2to4(const void* A, int64_t R, int64_t K, int64_t lda, venom_dtype_t dt,
                                  venom_format_t f, void* values, uint8_t* metadata,
                                  uint8_t* column_idx, void* values_2to4, uint8_t* metadata_2to4_tc,
                                  int32_t* dev_status, venom_stream_t stream) {
  venom_status_t st = validate_format(R, K, f);
  if (st != VENOM_OK) return st;
  if (dt != VENOM_F16 && dt != VENOM_BF16) return VENOM_ERR_UNSUPPORTED_DTYPE;
  if (f.m % 8 != 0 || 128 % f.m != 0 || f.v % 16 != 0 || K % 16 != 0 || f.v > 256)
    return VENOM_ERR_UNSUPPORTED_PATTERN;
  if (lda < K) return VENOM_ERR_INVALID_ARGUMENT;
  if (R == 0 || K == 0) return VENOM_OK;
  if (!A || !values || !metadata || !column_idx || !values_2to4 || !metadata_2to4_tc)
    return VENOM_ERR_INVALID_ARGUMENT;
  if (!aligned(values, 8) || !aligned(column_idx, 4) || !aligned(A, 2) || !aligned(values_2to4, 16) ||
      !aligned(metadata_2to4_tc, 16))
    return VENOM_ERR_INVALID_ARGUMENT;
  if (R / f.v > 65535) return VENOM_ERR_INVALID_ARGUMENT;
  if ((st = check_arch()) != VENOM_OK) return st;
  const int64_t G = K / f.m;
  // whole k-stages of the re-encoded operand per CTA: W = gt·M a multiple of 128 columns
  const int W = (f.v <= 128 && !(debug_flags() & 16)) ? 256 : 128;
  const int gt = W / f.m > 0 ? W / f.m : 1;
  if (gt * f.m != W) return VENOM_ERR_UNSUPPORTED_PATTERN;  // M must divide W (M | 128)
  const size_t tsmem = venom::CompressTileLayout(f.v, W, gt, true).total;
  if (tma_compress_ok(A, lda, f.v, W) && !(debug_flags() & 32)) {
    auto kt = (dt == VENOM_BF16) ? venom::vnm_compress_tma_kernel<true, true>
                                 : venom::vnm_compress_tma_kernel<false, true>;
    if (G % gt == 0 && f.m == 8 && gt == 32)
      kt = (dt == VENOM_BF16) ? venom::vnm_compress_tma_kernel<true, true, 8, 32>
                              : venom::vnm_compress_tma_kernel<false, true, 8, 32>;
    else if (G % gt == 0 && f.m == 16 && gt == 16)
      kt = (dt == VENOM_BF16) ? venom::vnm_compress_tma_kernel<true, true, 16, 16>
                              : venom::vnm_compress_tma_kernel<false, true, 16, 16>;
    return launch_compress_tma(kt, A, R, K, lda, f, gt, true, values, metadata, column_idx, dev_status,
                               static_cast<uint32_t*>(values_2to4), reinterpret_cast<uint32_t*>(metadata_2to4_tc),
                               static_cast<cudaStream_t>(stream));
  }
  const dim3 grid(static_cast<unsigned>((G + gt - 1) / gt), static_cast<unsigned>(R / f.v));
  auto kern = (dt == VENOM_BF16) ? venom::vnm_compress_tile_kernel<true, true>
                                 : venom::vnm_compress_tile_kernel<false, true>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(tsmem)) != cudaSuccess)
    return VENOM_ERR_CUDA;
  kern<<<grid, (debug_flags() & 32) ? 256 : kCompressThreads, tsmem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(A), R, K, lda, f.v, f.m, G, gt, static_cast<uint16_t*>(values),
      metadata, column_idx, dev_status, static_cast<uint32_t*>(values_2to4),
      reinterpret_cast<uint32_t*>(metadata_2to4_tc), debug_flags());
  return launch_status();
}

venom_status_t venom_compress_masked(const void* A, int64_t R, int64_t K, int64_t lda,
                                     const uint8_t* mask, int64_t ldm, venom_dtype_t dt,
                                     venom_format_t f, void* values, uint8_t* metadata,
                                     uint8_t* column_idx, int32_t* dev_status, venom_stream_t stream) {
  venom_status_t st = validate_format(R, K, f);
  if (st != VENOM_OK) return st;
  if (dt != VENOM_F16 && dt != VENOM_BF16) return VENOM_ERR_UNSUPPORTED_DTYPE;
  if (lda < K || ldm < K) return VENOM_ERR_INVALID_ARGUMENT;
  if (R == 0 || K == 0) return VENOM_OK;
  if (!A || !mask || !values || !metadata || !column_idx) return VENOM_ERR_INVALID_ARGUMENT;
  if (!aligned(values, 4) || !aligned(column_idx, 4) || !aligned(A, 2)) return VENOM_ERR_INVALID_ARGUMENT;
  if ((st = check_arch()) != VENOM_OK) return st;
  const int64_t G = K / f.m;
  const int64_t n = (R / f.v) * ((G + 1) / 2);
  const unsigned blocks = static_cast<unsigned>((n + 127) / 128);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dt == VENOM_BF16)
    venom::vnm_compress_masked_kernel<true><<<blocks, 128, 0, s>>>(
        static_cast<const uint16_t*>(A), mask, R, K, lda, ldm, f.v, f.m, G, static_cast<uint16_t*>(values),
        metadata, column_idx, dev_status);
  else
    venom::vnm_compress_masked_kernel<false><<<blocks, 128, 0, s>>>(
        static_cast<const uint16_t*>(A), mask, R, K, lda, ldm, f.v, f.m, G, static_cast<uint16_t*>(values),
        metadata, column_idx, dev_status);
  return launch_status();
}

venom_status_t venom_energy(const void* A, int64_t R, int64_t K, int64_t lda, const void* values,
                            int64_t n_values, venom_dtype_t dt, double* out, venom_stream_t stream) {
  if (dt != VENOM_F16 && dt != VENOM_BF16) return VENOM_ERR_UNSUPPORTED_DTYPE;
  if (R < 0 || K < 0 || n_values < 0 || lda < K || !out || (R * K > 0 && !A) || (n_values > 0 && !values))
    return VENOM_ERR_INVALID_ARGUMENT;
  if (!aligned(out, 8) || !aligned(A, 2) || !aligned(values, 2)) return VENOM_ERR_INVALID_ARGUMENT;
  venom_status_t st = check_arch();
  if (st != VENOM_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(out, 0, 2 * sizeof(double), s) != cudaSuccess) return VENOM_ERR_CUDA;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = static_cast<unsigned>(sms * 8);
  if (dt == VENOM_BF16)
    venom::vnm_energy_kernel<true><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(A), R, K, lda,
                                                        static_cast<const uint16_t*>(values), n_values, out);
  else
    venom::vnm_energy_kernel<false><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(A), R, K, lda,
                                                         static_cast<const uint16_t*>(values), n_values, out);
  venom::vnm_energy_finish_kernel<<<1, 1, 0, s>>>(out);
  return launch_status();
}

venom_status_t venom_decompress(const void* values, const uint8_t* metadata,
                                const uint8_t* column_idx, int64_t R, int64_t K, venom_dtype_t dt,
                                venom_format_t f, void* A_out, int64_t lda, int32_t* dev_status,
                                venom_stream_t stream) {
  venom_status_t st = validate_format(R, K, f);
  if (st != VENOM_OK) return st;
  if (dt != VENOM_F16 && dt != VENOM_BF16) return VENOM_ERR_UNSUPPORTED_DTYPE;
  if (lda < K) return VENOM_ERR_INVALID_ARGUMENT;
  if (R == 0 || K == 0) return VENOM_OK;
  if (!values || !metadata || !column_idx || !A_out) return VENOM_ERR_INVALID_ARGUMENT;
  if (!aligned(values, 4) || !aligned(column_idx, 4) || !aligned(A_out, 2)) return VENOM_ERR_INVALID_ARGUMENT;
  if ((st = check_arch()) != VENOM_OK) return st;
  const int64_t G = K / f.m;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool vec = aligned(A_out, 16) && (lda % 8 == 0);
  const int kv = vec ? 8 : 1;
  const int64_t chunks = (K + kv - 1) / kv;
  if (K > 0x7FFFFFFF) return VENOM_ERR_INVALID_ARGUMENT;
  if (R * chunks >= 0x7FFFFFFF) return VENOM_ERR_INVALID_ARGUMENT;
  const int64_t blocks = (R * chunks + 255) / 256;
  const dim3 grid(static_cast<unsigned>(blocks < 148 * 64 ? blocks : 148 * 64));
  if (vec && f.m % 8 == 0 && R <= 0x7FFFFFFF) {
    constexpr int kRows = 4;  // rows per thread (loads of all of them in flight together)
    const int64_t slots = (R + kRows - 1) / kRows;
    const int64_t units = (f.m == 8 || f.m == 16 || f.m == 32) ? G : K / 8;  // groups (compile-time M) or chunks
    const dim3 g2(static_cast<unsigned>((units + 255) / 256), static_cast<unsigned>(slots < 65535 ? slots : 65535));
#define VENOM_DEC8(C)                                                                                  \
  venom::vnm_decompress_m8_kernel<C, kRows><<<g2, 256, 0, s>>>(                                        \
      static_cast<const uint32_t*>(values), metadata, reinterpret_cast<const uint32_t*>(column_idx), \
      static_cast<int>(R), static_cast<int>(K), f.v, f.m, static_cast<int>(G),                        \
      static_cast<uint16_t*>(A_out), lda, dev_status)
    if (f.m == 8) VENOM_DEC8(1);
    else if (f.m == 16) VENOM_DEC8(2);
    else if (f.m == 32) VENOM_DEC8(4);
    else VENOM_DEC8(0);
#undef VENOM_DEC8
    return launch_status();
  }
  if (vec)
    venom::vnm_decompress_kernel<8><<<grid, 256, 0, s>>>(
        static_cast<const uint16_t*>(values), metadata, column_idx, R, K, f.v, f.m, G,
        static_cast<uint16_t*>(A_out), lda, dev_status);
  else
    venom::vnm_decompress_kernel<1><<<grid, 256, 0, s>>>(
        static_cast<const uint16_t*>(values), metadata, column_idx, R, K, f.v, f.m, G,
        static_cast<uint16_t*>(A_out), lda, dev_status);
  return launch_status();
}

int32_t venom_prefer_2to4(int64_t R, int64_t K, int64_t T, venom_format_t f) {
  if (validate_format(R, K, f) != VENOM_OK || f.m % 4 != 0 || f.m == 4) return 0;
  if ((K / 4) % 4 != 0 || T < 256) return 0;
  // the fused preparation (venom_compress_2to4) must apply
  if (f.m % 8 != 0 || 128 % f.m != 0 || f.v % 16 != 0 || f.v > 256 || K % 16 != 0) return 0;
  // measured crossover (profiles/r02b_vscaling.txt, 4096³ for V in
  // {32, 64, 128, 256} and M in {8, 16, 32}): the gathered path lands bytes per useful FLOP that
  // fall with V and M, while the V:2:4 form's time does not depend on V or M; the V:2:4 form wins
  // for M = 8 below V = 256 and for V·M < 1024 otherwise (round 2's M64 lane-half MMAs moved the
  // crossover: 64:2:16 and 256:2:8 now run faster gathered)
  return ((f.m <= 8 && f.v < 256) || static_cast<int64_t>(f.v) * f.m < 1024) ? 1 : 0;
}

venom_status_t venom_expand_2to4(const void* values, const uint8_t* metadata,
                                const uint8_t* column_idx, int64_t R, int64_t K, venom_dtype_t dt,
                                venom_format_t f, void* values_out, uint8_t* metadata_out,
                                uint8_t* column_idx_out, int32_t* dev_status,
                                venom_stream_t stream) {
  venom_status_t st = validate_format(R, K, f);
  if (st != VENOM_OK) return st;
  if (f.m % 4 != 0) return VENOM_ERR_UNSUPPORTED_PATTERN;
  if (dt != VENOM_F16 && dt != VENOM_BF16) return VENOM_ERR_UNSUPPORTED_DTYPE;
  if (R == 0 || K == 0) return VENOM_OK;
  if (!values || !metadata || !column_idx || !values_out || !metadata_out || !column_idx_out)
    return VENOM_ERR_INVALID_ARGUMENT;
  if (!aligned(values, 4) || !aligned(column_idx, 4) || !aligned(values_out, 4) ||
      !aligned(column_idx_out, 4))
    return VENOM_ERR_INVALID_ARGUMENT;
  if ((st = check_arch()) != VENOM_OK) return st;
  const int64_t G = K / f.m;
  const int64_t npairs = (G + 1) / 2;
  if (R * npairs >= 0x7FFFFFFF) return VENOM_ERR_INVALID_ARGUMENT;
  const int64_t blocks = (R * npairs + 255) / 256;
  const dim3 grid(static_cast<unsigned>(blocks < 148 * 64 ? blocks : 148 * 64));
  venom::vnm_expand_2to4_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint32_t*>(values), metadata, reinterpret_cast<const uint32_t*>(column_idx), R,
      f.v, f.m, G, static_cast<uint32_t*>(values_out), metadata_out,
      reinterpret_cast<uint32_t*>(column_idx_out), dev_status);
  return launch_status();
}

venom_status_t venom_spmm_ex(const void* values, const uint8_t* metadata, const uint8_t* column_idx,
                             int64_t R, int64_t K, venom_format_t f, const void* B, int64_t T,
                             int64_t ldb, void* C, int64_t ldc, const void* bias, venom_dtype_t dt,
                             const venom_spmm_opts_t* opts, venom_stream_t stream) {
  venom_status_t st = validate_format(R, K, f);
  if (st != VENOM_OK) return st;
  if (dt != VENOM_F16 && dt != VENOM_BF16) return VENOM_ERR_UNSUPPORTED_DTYPE;
  const int V = f.v;
  const int64_t G = K / f.m;
  // G % 4 != 0 (a K' tail): the values' TMA map needs the padded execution form, and the
  // canonical metadata (16-bit words) cannot be read by the kernel: metadata_tc is required
  const bool padded = (G % 4 != 0) && opts && opts->values_padded && opts->metadata_tc;
  const bool can_gather = (f.m == 4 || V == 32 || V == 64 || V % 128 == 0) && (G % 4 == 0 || padded);
  // dense-K is instantiated for M in {4, 8, 16, 32} only (spmm_launch.cuh run_densek_m)
  const bool can_densek = (f.m == 4 || f.m == 8 || f.m == 16 || f.m == 32) && (G % 4 == 0);
  const int strategy = opts ? opts->strategy : VENOM_STRATEGY_AUTO;
  // cta_pair sizes the B tensor-map boxes: a value outside {0, 1, 2} would make the TMA deliver
  // fewer bytes than the stage barrier expects (a hang), so it is refused before anything runs
  if (opts && (opts->cta_pair < 0 || opts->cta_pair > 2)) return VENOM_ERR_INVALID_ARGUMENT;
  // the pipeline depth is fixed per tile configuration (spmm_launch.cuh); no override exists
  if (opts && opts->stages != 0) return VENOM_ERR_INVALID_ARGUMENT;
  if (strategy == VENOM_STRATEGY_GATHER && !can_gather) return VENOM_ERR_UNSUPPORTED_PATTERN;
  if (strategy == VENOM_STRATEGY_DENSE_K && !can_densek) return VENOM_ERR_UNSUPPORTED_PATTERN;
  if (strategy < 0 || strategy > 2) return VENOM_ERR_INVALID_ARGUMENT;
  if (!can_gather && !can_densek) return VENOM_ERR_UNSUPPORTED_PATTERN;
  const bool ct = opts && opts->c_transposed;  // token-major C^T[T][ldc]
  const bool bk = opts && opts->b_kmajor;      // token-major B[T][ldb]
  if (T < 0) return VENOM_ERR_INVALID_ARGUMENT;
  if (R == 0 || T == 0) return VENOM_OK;  // nothing to compute (leading dimensions are then moot)
  if ((bk ? ldb < K : ldb < T) || (ct ? ldc < R : ldc < T) || T % 8 != 0 || ldb % 8 != 0 || ldc % 8 != 0)
    return VENOM_ERR_INVALID_ARGUMENT;
  if (ct && (strategy == VENOM_STRATEGY_DENSE_K || !can_gather || (opts && opts->tile_t == 240)))
    return VENOM_ERR_INVALID_ARGUMENT;
  if (bk && f.m != 4) {
    // gathered operand with token-major activations: the selected K-rows of B would be columns
    // of B^T, which tile::gather4 cannot fetch; B^T is transposed once into the caller's scratch
    // (feature-major [K][T], 2·|B| of HBM traffic) and the feature-major path runs on it
    // (cheaper than compacting raw K-major tiles in shared memory)
    if (!opts->b_scratch || !aligned(opts->b_scratch, 16) || strategy == VENOM_STRATEGY_DENSE_K ||
        opts->tile_t == 240 || K % 8 != 0 || ldb < K || !aligned(B, 16))
      return VENOM_ERR_INVALID_ARGUMENT;
    if ((st = check_arch()) != VENOM_OK) return st;
    if (K > 0) {
      const dim3 grid(static_cast<unsigned>((K + 63) / 64), static_cast<unsigned>((T + 63) / 64));
      if (grid.y > 65535) return VENOM_ERR_INVALID_ARGUMENT;
      venom::vnm_transpose16_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
          static_cast<const uint16_t*>(B), T, K, ldb, static_cast<uint16_t*>(opts->b_scratch));
      if ((st = launch_status()) != VENOM_OK) return st;
    }
    venom_spmm_opts_t o2 = *opts;
    o2.b_kmajor = 0;
    o2.b_scratch = nullptr;
    return venom_spmm_ex(values, metadata, column_idx, R, K, f, opts->b_scratch, T, T, C, ldc, bias, dt, &o2,
                         stream);
  }
  if (bk && (strategy == VENOM_STRATEGY_DENSE_K || (opts && opts->tile_t == 240) || K % 8 != 0))
    return VENOM_ERR_INVALID_ARGUMENT;
  const int act = opts ? opts->activation : 0;
  if (act != 0 && ((act != 1 && act != 2) || ct || bk || strategy == VENOM_STRATEGY_DENSE_K || !can_gather ||
                   (opts && opts->tile_t == 240)))
    return VENOM_ERR_INVALID_ARGUMENT;
  const bool has_tc = opts && opts->metadata_tc;
  // metadata is not read with pre-ordered metadata; column_idx is not read when M = 4 (identity)
  if (!C || (K > 0 && (!values || !B || (!metadata && !has_tc) || (!column_idx && f.m != 4))))
    return VENOM_ERR_INVALID_ARGUMENT;
  if (!aligned(C, 16) || (K > 0 && (!aligned(values, 16) || !aligned(B, 16) || !aligned(column_idx, 4))))
    return VENOM_ERR_INVALID_ARGUMENT;
  // canonical metadata is read with 16-byte vector loads (gathered kernel without metadata_tc, and
  // the dense-K expanders), column_idx with 16-byte loads by the dense-K expanders: a misaligned
  // view would fault on the device, so it is refused here
  if (K > 0 && !has_tc && !aligned(metadata, 16)) return VENOM_ERR_INVALID_ARGUMENT;
  if (K > 0x7FFFFFFF || T > 0x7FFFFFFF || R > 0x7FFFFFFF) return VENOM_ERR_INVALID_ARGUMENT;
  if ((st = check_arch()) != VENOM_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool bf16 = dt == VENOM_BF16;

  if (K == 0) {
    const int64_t n = R * T;
    venom::vnm_fill_bias_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
        static_cast<uint16_t*>(C), R, T, ldc, static_cast<const uint16_t*>(bias), ct ? 1 : 0);
    return launch_status();
  }

  EncodeTiledFn enc = encode_fn();
  if (!enc) return VENOM_ERR_CUDA;
  const int NB = (V % 128 == 0) ? 1 : 128 / V;
  const int max_ctas = opts ? opts->max_ctas : 0;
  int tile_t = opts ? opts->tile_t : 0;

  bool use_densek;
  if (strategy == VENOM_STRATEGY_GATHER) use_densek = false;
  else if (strategy == VENOM_STRATEGY_DENSE_K) use_densek = true;
  else if (!can_gather) use_densek = true;
  else if (!can_densek) use_densek = false;
  else use_densek = false;  // measured: the gathered / contiguous kernel wins wherever it applies
  if (opts && opts->n_peers != 0 && use_densek) return VENOM_ERR_INVALID_ARGUMENT;  // no fan-out in dense-K

  SpmmParams p;
  p.values = static_cast<const uint16_t*>(values);
  p.metadata = metadata;
  p.column_idx = column_idx;
  p.bias = static_cast<const uint16_t*>(bias);
  p.C = static_cast<uint16_t*>(C);
  p.R = R;
  p.K = K;
  p.T = T;
  p.ldc = ldc;
  p.V = V;
  p.M = f.m;
  p.G = static_cast<int>(G);
  p.meta_row = static_cast<int>((G + 1) / 2);
  p.m_tiles = static_cast<int>((R + 127) / 128);
  p.group_n = opts ? opts->group_n : 0;  // 0: the planner's tile order (spmm_launch.cuh)
  p.is_bf16 = bf16;
  p.b3d = 0;
  p.bk = 0;
  p.act = 0;
  p.c_t = ct ? 1 : 0;
  p.bk = bk ? 1 : 0;
  p.act = act;
  p.tma_c = 0;
  p.e4d = 0;
  p.last_kb = 4;
  p.n_peers = 0;
  for (int i = 0; i < venom::kMaxPeers; ++i) p.c_peers[i] = nullptr;
  if (opts && opts->n_peers != 0) {
    // fused all-gather: peer output buffers (row-major C through the TMA-store epilogue, or
    // token-major C); each 16-byte aligned, addressed like C (same ldc)
    if (opts->n_peers < 0 || opts->n_peers > venom::kMaxPeers || !opts->c_peers || strategy == VENOM_STRATEGY_DENSE_K ||
        (opts->tile_t == 240))
      return VENOM_ERR_INVALID_ARGUMENT;
    for (int i = 0; i < opts->n_peers; ++i) {
      if (!opts->c_peers[i] || !aligned(opts->c_peers[i], 16)) return VENOM_ERR_INVALID_ARGUMENT;
      p.c_peers[i] = static_cast<uint16_t*>(opts->c_peers[i]);
    }
    p.n_peers = opts->n_peers;
  }
  p.dbg = debug_flags();
  auto set_tiles = [&](int bn) {
    p.n_tiles = static_cast<int>((T + bn - 1) / bn);
    p.num_tiles = p.m_tiles * p.n_tiles;
  };

  auto encode_b = [&](CUtensorMap* tb, cuuint32_t box_rows) -> bool {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(T), static_cast<cuuint64_t>(K)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(2 * ldb)};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t es[2] = {1, 1};
    return enc(tb, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(B), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };

  if (use_densek && (!metadata || !column_idx || !aligned(metadata, 16) || !aligned(column_idx, 16)))
    return VENOM_ERR_INVALID_ARGUMENT;
  if (use_densek) {
    // B: 2-D [K rows][T], box 64 columns × 128 rows (one K-stage of one 64-column chunk), SW128
    CUtensorMap tb;
    if (!encode_b(&tb, 128)) return VENOM_ERR_CUDA;
    p.num_ks = static_cast<int>((K + 127) / 128);
    if (tile_t == 0) tile_t = 256;
    set_tiles(tile_t);
    const int pair = opts && opts->cta_pair ? opts->cta_pair : 2;
    return bf16 ? venom::launch::densek_bf16(f.m, pair, tile_t, tb, enc, p, max_ctas, s)
                : venom::launch::densek_f16(f.m, pair, tile_t, tb, enc, p, max_ctas, s);
  }

  // gathered strategy
  // values: 2-D [R rows][2G] 16-bit, box 64 × 128 rows, 128B swizzle (UMMA K-major SW128); for
  // G % 4 != 0 the padded execution form [R][2·G4] (16-byte row pitch)
  CUtensorMap tv, tb;
  if (padded && !aligned(opts->values_padded, 16)) return VENOM_ERR_INVALID_ARGUMENT;
  {
    const int64_t Gp = padded ? (G + 3) / 4 * 4 : G;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(2 * Gp), static_cast<cuuint64_t>(R)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(4 * Gp)};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tv, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(padded ? opts->values_padded : values), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return VENOM_ERR_CUDA;
  }
  // B: 2-D [K rows][T] 16-bit, 128B swizzle; box 64 × 1 row for gather4 (4 rows per op), or
  // 64 × 128 rows when M = 4 (every group's 4 columns are selected: plain K-slices of B). With
  // T % 64 == 0 the M = 4 map is 3-D [T/64 chunks][K rows][64 columns] (chunk stride 128 B) so one
  // box [NCH][128][64] lands the CTA's whole B' stage in the chunked SW128 layout.
  const bool contiguous = (f.m == 4);
  p.num_ks = static_cast<int>((G + 31) / 32);
  // K = 32 MMAs (8 groups each) that carry real groups in the last k-stage: the rest are neither
  // gathered nor multiplied (e.g. G = 104: 8 of the last stage's 32 groups)
  p.last_kb = static_cast<int>((G - 32 * (static_cast<int64_t>(p.num_ks) - 1) + 7) / 8);
  const int NBg = contiguous ? 1 : NB;  // M = 4 ignores V (column_idx is the identity)
  const bool pair_ok = NBg == 1 && (contiguous || V % 256 == 0);
  const int pair = (opts && opts->cta_pair) ? opts->cta_pair : (pair_ok ? 2 : 1);
  if (pair == 2 && !pair_ok) return VENOM_ERR_INVALID_ARGUMENT;
  if (tile_t == 0) {
    tile_t = (NBg == 1) ? 256 : (NBg == 2 ? 128 : 64);
    // 512 × 240 pair tiles (two accumulators per CTA) land 1.45× fewer bytes per FLOP but expose a
    // larger last epilogue: measured better only with long k-loops and at least one full wave of
    // pair tiles
    if (contiguous && pair == 2 && opts && opts->metadata_tc && !ct && !bk && !act) {
      int sms = 148, dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int64_t tiles240 = ((R + 511) / 512) * ((T + 239) / 240);
      if (p.num_ks >= 24 && tiles240 >= sms / 2) tile_t = 240;
    }
  }
  set_tiles(tile_t);
  p.b3d = contiguous && !bk && (T % 64 == 0) && ((tile_t / pair) % 64 == 0);
  if (p.b3d) {
    const int nch = (tile_t / pair + 63) / 64;
    cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(T / 64)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(2 * ldb), 128};
    cuuint32_t box[3] = {64, 128, static_cast<cuuint32_t>(nch)};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(B), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      p.b3d = 0;  // driver refused the chunk-stride map: 2-D boxes below
  }
  if (bk) {
    // K-major B: 2-D [T rows][K] with a box of BNH token rows × 64 K-elements (K-major SW128)
    const int bnh = tile_t / pair;
    if (bnh % 64 != 0) return VENOM_ERR_INVALID_ARGUMENT;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(T)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(2 * ldb)};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(bnh)};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(B), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return VENOM_ERR_CUDA;
  } else if (!p.b3d && !encode_b(&tb, contiguous ? 128 : 1)) {
    return VENOM_ERR_CUDA;
  }
  // C: row-major output through TMA boxes of 32 rows × 32 columns (64-byte swizzle, the epilogue's
  // staging layout); token-major C keeps its direct stores
  CUtensorMap tc = tv;
  p.tma_c = 0;
  if (ct) {
    // token-major C^T [T rows][R]: boxes of 32 columns t × 32 rows r (64-byte swizzle), or × 16
    // rows r for V = 64 (each warp holds two 16-row halves; 32-byte swizzle)
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(R), static_cast<cuuint64_t>(T)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(2 * ldc)};
    cuuint32_t box[2] = {NBg >= 2 ? 16u : 32u, 32};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tc, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, C, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            NBg >= 2 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      p.tma_c = 1;
    else
      tc = tv;
  } else {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(T), static_cast<cuuint64_t>(R)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(2 * ldc)};
    // V = 64 (two M = 64 blocks per tile): a warp's 32 lanes hold two 16-row halves -> 16-row boxes
    cuuint32_t box[2] = {32, NBg >= 2 ? 16u : 32u};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tc, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, C, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
        CUDA_SUCCESS)
      p.tma_c = 1;
    else
      tc = tv;
  }
  if (p.n_peers > 0 && !ct && !p.tma_c) return VENOM_ERR_INVALID_ARGUMENT;
  const uint8_t* meta_tc = opts ? opts->metadata_tc : nullptr;
  if (meta_tc == nullptr)
    return bf16 ? venom::launch::gather_nopre_bf16(NBg, pair, tile_t, tv, tb, tv, tc, p, max_ctas, s)
                : venom::launch::gather_nopre_f16(NBg, pair, tile_t, tv, tb, tv, tc, p, max_ctas, s);
  // pre-ordered metadata: the [tiles·num_ks] contiguous 2 KB stage blocks, mapped as 2-D
  // [blocks][256] u64 with a one-row box, so each block is one 2 KB TMA row (a 16-byte-wide box of
  // 128 rows would cost the TMA unit 128 row requests per stage)
  if (!aligned(meta_tc, 16)) return VENOM_ERR_INVALID_ARGUMENT;
  CUtensorMap te;
  p.e4d = 0;
  if (NBg >= 2) {
    // V = 64 / 32: the kernel's TMEM lane order for two M = 64 blocks is a permutation of the stored
    // 16-lane groups (group x + 4y of a block -> 2x + y, spmm_kernel.cuh M64); a 4-D map with
    // swapped strides does it in one TMA op: dims [256 B][y: 2, 1 KB][x: 4, 256 B][blocks, 2 KB]
    const int64_t blocks = ((R + 127) / 128) * p.num_ks;
    cuuint64_t dims[4] = {32, 2, 4, static_cast<cuuint64_t>(blocks)};
    cuuint64_t strides[3] = {1024, 256, 2048};
    cuuint32_t box[4] = {32, 2, 4, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&te, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, const_cast<uint8_t*>(meta_tc), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
      p.e4d = 1;
    } else {
      // fallback: 256-byte rows [blocks·8][32] u64, eight row loads per stage
      cuuint64_t d2[2] = {32, static_cast<cuuint64_t>(blocks * 8)};
      cuuint64_t s2[1] = {256};
      cuuint32_t b2[2] = {32, 1};
      if (enc(&te, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<uint8_t*>(meta_tc), d2, s2, b2, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return VENOM_ERR_CUDA;
    }
  } else {
    const int64_t blocks = ((R + 127) / 128) * p.num_ks;
    cuuint64_t dims[2] = {256, static_cast<cuuint64_t>(blocks)};
    cuuint64_t strides[1] = {2048};
    cuuint32_t box[2] = {256, 1};
    cuuint32_t es[2] = {1, 1};
    if (enc(&te, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<uint8_t*>(meta_tc), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return VENOM_ERR_CUDA;
  }
  return bf16 ? venom::launch::gather_pre_bf16(NBg, pair, tile_t, tv, tb, te, tc, p, max_ctas, s)
              : venom::launch::gather_pre_f16(NBg, pair, tile_t, tv, tb, te, tc, p, max_ctas, s);
}

int64_t venom_metadata_tc_bytes(int64_t R, int64_t K, venom_format_t f) {
  if (validate_format(R, K, f) != VENOM_OK) return -1;
  const int64_t G = K / f.m;
  return ((R + 127) / 128) * ((G + 31) / 32) * 128 * 16;
}

venom_status_t venom_order_metadata(const uint8_t* metadata, int64_t R, int64_t K, venom_format_t f,
                                    uint8_t* metadata_tc, venom_stream_t stream) {
  venom_status_t st = validate_format(R, K, f);
  if (st != VENOM_OK) return st;
  const int64_t G = K / f.m;
  if (R == 0 || K == 0) return VENOM_OK;
  if (!metadata || !metadata_tc || !aligned(metadata_tc, 16) || (G % 4 == 0 && !aligned(metadata, 2)))
    return VENOM_ERR_INVALID_ARGUMENT;
  if ((st = check_arch()) != VENOM_OK) return st;
  const int64_t num_ks = (G + 31) / 32;
  const int64_t total = ((R + 127) / 128) * num_ks * 128 * 4;  // 32-bit words
  const int64_t blocks = (total + 255) / 256;
  venom::vnm_order_metadata_kernel<<<static_cast<unsigned>(blocks < 148 * 64 ? blocks : 148 * 64), 256, 0,
                                     static_cast<cudaStream_t>(stream)>>>(
      metadata, R, G, num_ks, total, reinterpret_cast<uint32_t*>(metadata_tc));
  return launch_status();
}

int64_t venom_values_padded_bytes(int64_t R, int64_t K, venom_format_t f) {
  if (validate_format(R, K, f) != VENOM_OK) return -1;
  const int64_t G = K / f.m;
  return R * ((G + 3) / 4 * 4) * 4;
}

venom_status_t venom_pad_values(const void* values, int64_t R, int64_t K, venom_format_t f,
                                void* values_padded, venom_stream_t stream) {
  venom_status_t st = validate_format(R, K, f);
  if (st != VENOM_OK) return st;
  if (R == 0 || K == 0) return VENOM_OK;
  if (!values || !values_padded || !aligned(values, 4) || !aligned(values_padded, 16)) return VENOM_ERR_INVALID_ARGUMENT;
  if ((st = check_arch()) != VENOM_OK) return st;
  const int64_t G = K / f.m, G4 = (G + 3) / 4 * 4;
  const int64_t blocks = (R * G4 + 255) / 256;
  venom::vnm_pad_values_kernel<<<static_cast<unsigned>(blocks < 148 * 64 ? blocks : 148 * 64), 256, 0,
                                 static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint32_t*>(values), R, G, G4, static_cast<uint32_t*>(values_padded));
  return launch_status();
}

venom_status_t venom_spmm(const void* values, const uint8_t* metadata, const uint8_t* column_idx,
                          int64_t R, int64_t K, venom_format_t f, const void* B, int64_t T,
                          int64_t ldb, void* C, int64_t ldc, const void* bias, venom_dtype_t dt,
                          venom_stream_t stream) {
  return venom_spmm_ex(values, metadata, column_idx, R, K, f, B, T, ldb, C, ldc, bias, dt, nullptr,
                       stream);
}

}  // extern "C"

// ------------------------------------------------------------------ encoder layout kernels
// (include/venom_encoder.h; SURVEY §8(f) rank 1 plumbing, not the V:N:M method)
extern "C" venom_status_t venom_enc_add_layernorm(const void* x, const void* y, const void* w, const void* b,
                                                  int64_t T, int64_t h, float eps, venom_dtype_t dt,
                                                  void* out_tm, void* out_fm, int64_t ld_fm,
                                                  venom_stream_t stream) {
  if (dt != VENOM_F16 && dt != VENOM_BF16) return VENOM_ERR_UNSUPPORTED_DTYPE;
  if (!x || !y || !w || !b || !out_tm || T < 0 || h % 256 != 0 || h <= 0 || h > 1024 || T % 32 != 0)
    return VENOM_ERR_INVALID_ARGUMENT;
  if (out_fm && (ld_fm < T || ld_fm % 8 != 0)) return VENOM_ERR_INVALID_ARGUMENT;
  if (!aligned(x, 16) || !aligned(y, 16) || !aligned(w, 16) || !aligned(b, 16) || !aligned(out_tm, 16))
    return VENOM_ERR_INVALID_ARGUMENT;
  if (T == 0) return VENOM_OK;
  venom_status_t st = check_arch();
  if (st != VENOM_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nv = static_cast<int>(h / 256);
  const int smem = static_cast<int>(32 * (h + 2) * 2);
  const unsigned grid = static_cast<unsigned>(T / 32);
  auto go = [&](auto kern) -> venom_status_t {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return VENOM_ERR_CUDA;
    kern<<<grid, 256, smem, s>>>(static_cast<const uint16_t*>(x), static_cast<const uint16_t*>(y),
                                 static_cast<const uint16_t*>(w), static_cast<const uint16_t*>(b), T, eps,
                                 static_cast<uint16_t*>(out_tm), static_cast<uint16_t*>(out_fm), ld_fm);
    return launch_status();
  };
  const bool bf = dt == VENOM_BF16;
  switch (nv) {
    case 1: return bf ? go(venom::vnm_enc_add_layernorm_kernel<true, 1>) : go(venom::vnm_enc_add_layernorm_kernel<false, 1>);
    case 2: return bf ? go(venom::vnm_enc_add_layernorm_kernel<true, 2>) : go(venom::vnm_enc_add_layernorm_kernel<false, 2>);
    case 3: return bf ? go(venom::vnm_enc_add_layernorm_kernel<true, 3>) : go(venom::vnm_enc_add_layernorm_kernel<false, 3>);
    default: return bf ? go(venom::vnm_enc_add_layernorm_kernel<true, 4>) : go(venom::vnm_enc_add_layernorm_kernel<false, 4>);
  }
}

extern "C" venom_status_t venom_enc_heads_to_fm(const void* a, int64_t B, int64_t H, int64_t S, int64_t D,
                                                int64_t sb, int64_t sh, int64_t ss, venom_dtype_t dt,
                                                void* out_fm, int64_t ld_fm, venom_stream_t stream) {
  if (dt != VENOM_F16 && dt != VENOM_BF16) return VENOM_ERR_UNSUPPORTED_DTYPE;
  if (!a || !out_fm || B < 0 || H < 0 || D != 64 || S % 64 != 0 || ld_fm < B * S || ld_fm % 8 != 0 ||
      sb % 8 != 0 || sh % 8 != 0 || ss % 8 != 0 || !aligned(a, 16) || !aligned(out_fm, 4))
    return VENOM_ERR_INVALID_ARGUMENT;
  if (B * H * S == 0) return VENOM_OK;
  venom_status_t st = check_arch();
  if (st != VENOM_OK) return st;
  const unsigned grid = static_cast<unsigned>(B * H * (S / 64));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dt == VENOM_BF16)
    venom::vnm_enc_heads_to_fm_kernel<true><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(a), H, S, sb, sh,
                                                                 ss, static_cast<uint16_t*>(out_fm), ld_fm);
  else
    venom::vnm_enc_heads_to_fm_kernel<false><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(a), H, S, sb, sh,
                                                                  ss, static_cast<uint16_t*>(out_fm), ld_fm);
  return launch_status();
}
