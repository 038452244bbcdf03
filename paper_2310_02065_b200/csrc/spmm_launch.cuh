// spmm_launch.cuh — host-side launch templates of the SpMM kernels (internal to libvenom).
//
// The kernel instantiations are split over several translation units (tu_*.cu) so that nvcc
// compiles them in parallel; each unit defines one of the launchers declared at the bottom, and
// venom_api.cu (argument validation, tensor-map encoding) calls them. Nothing here is part of the
// C ABI (include/venom.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/venom.h"
#include "spmm_kernel.cuh"
#include "densek_kernel.cuh"

#ifndef VENOM_GATHER_P
#define VENOM_GATHER_P 11  // gather-issuing warps of the single-CTA 128 × 256 tile (tools builds vary it)
#endif

namespace venom {
namespace launch {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline venom_status_t launch_status() {
  return cudaGetLastError() == cudaSuccess ? VENOM_OK : VENOM_ERR_CUDA;
}

inline int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// Launch with an optional CTA-pair cluster (cg = 2 -> cluster dims {2,1,1}).
template <typename Kern, typename... Args>
venom_status_t launch_cg(Kern kern, int cg, int grid, int threads, int smem, cudaStream_t s,
                         Args... args) {
  if (cg == 1) {
    kern<<<grid, threads, smem, s>>>(args...);
    return launch_status();
  }
  grid -= grid % cg;
  if (grid < cg) grid = cg;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cg;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, args...) != cudaSuccess) return VENOM_ERR_CUDA;
  return launch_status();
}

// ------------------------------------------------------------------ gathered / contiguous kernel
template <class Cfg, bool kBF16>
venom_status_t run_spmm(const CUtensorMap& tv, const CUtensorMap& tb, const CUtensorMap& te,
                        const CUtensorMap& tc, SpmmParams p, int max_ctas, cudaStream_t s) {
  // token-major C is a separate instantiation: a runtime branch in the epilogue cost the row-major
  // kernels up to 12% (measured on BERT FFN1)
  auto kern = p.c_t ? (p.M == 4 ? vnm_spmm_kernel<Cfg, kBF16, true, true>
                                : vnm_spmm_kernel<Cfg, kBF16, false, true>)
                    : (p.M == 4 ? vnm_spmm_kernel<Cfg, kBF16, true, false>
                                : vnm_spmm_kernel<Cfg, kBF16, false, false>);
  if constexpr (Cfg::MB == 1) {
    // GELU epilogue (row-major C, row-major B; checked by the caller)
    if (p.act == 1) kern = p.M == 4 ? vnm_spmm_kernel<Cfg, kBF16, true, false, false, 1>
                                    : vnm_spmm_kernel<Cfg, kBF16, false, false, false, 1>;
    if (p.act == 2) kern = p.M == 4 ? vnm_spmm_kernel<Cfg, kBF16, true, false, false, 2>
                                    : vnm_spmm_kernel<Cfg, kBF16, false, false, false, 2>;
  } else {
    if (p.act) return VENOM_ERR_INVALID_ARGUMENT;
  }
  if constexpr (Cfg::MB == 1 && Cfg::NB == 1 && Cfg::BNH % 64 == 0) {
    // K-major B (token-major activations): M = 4 operand only (checked by the caller)
    if (p.bk) kern = p.c_t ? vnm_spmm_kernel<Cfg, kBF16, true, true, true>
                           : vnm_spmm_kernel<Cfg, kBF16, true, false, true>;
  } else {
    if (p.bk) return VENOM_ERR_INVALID_ARGUMENT;
  }
  // >= 116 KB of shared memory guarantees one CTA per SM (each CTA allocates all 512 TMEM columns)
  const int smem = Cfg::SMEM_BYTES < 116 * 1024 ? 116 * 1024 : Cfg::SMEM_BYTES;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return VENOM_ERR_CUDA;
  const int sms = sm_count();
  p.m_tiles = static_cast<int>((p.R + 128 * Cfg::CG * Cfg::MB - 1) / (128 * Cfg::CG * Cfg::MB));
  p.num_tiles = p.m_tiles * p.n_tiles;
  int grid = p.num_tiles * Cfg::CG < sms ? p.num_tiles * Cfg::CG : sms;
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  if (grid < 1) return VENOM_OK;
  // tile order (opts.group_n): the T-band order (1) is the default. Grouping column tiles so that A
  // is re-read from HBM less often (group_n = 3 roughly halves the GPT-3 FFN layer's DRAM traffic)
  // measured slower there (2.16 vs 2.01 ms): the gathers of B are the latency-critical stream, and
  // the T-band order keeps the fewest B column slabs live in L2
  if (p.group_n <= 0) p.group_n = 1;
  if (Cfg::MB != 1) p.tma_c = 0;  // the two-accumulator epilogue stores directly
  return launch_cg(kern, Cfg::CG, grid, Cfg::NUM_THREADS, smem, s, tv, tb, te, tc, p);
}

// Gathered / contiguous kernel configurations. PRE: metadata pre-ordered for the tensor core.
template <bool PRE, bool kBF16>
venom_status_t run_gather(int NBg, int pair, int tile_t, const CUtensorMap& tv, const CUtensorMap& tb,
                          const CUtensorMap& te, const CUtensorMap& tc, SpmmParams p, int max_ctas, cudaStream_t s) {
  if constexpr (PRE) {
    // two 128-row blocks per CTA of a pair (512 × 240 pair tiles): 1.45× fewer landed bytes per
    // useful FLOP than 256 × 256 pair tiles, for the contiguous (M = 4) operand
    if (tile_t == 240 && NBg == 1 && pair == 2 && p.M == 4)
      return run_spmm<SpmmCfg<1, 240, 3, 4, 2, true, 2>, kBF16>(tv, tb, te, tc, p, max_ctas, s);
  }
  if (NBg == 1 && pair == 2) {
    if (tile_t == 256) return run_spmm<SpmmCfg<1, 256, 4, 8, 2, PRE>, kBF16>(tv, tb, te, tc, p, max_ctas, s);
    if (tile_t == 128) return run_spmm<SpmmCfg<1, 128, 6, 8, 2, PRE>, kBF16>(tv, tb, te, tc, p, max_ctas, s);
  } else if (NBg == 1) {
    // 11 gather-issuing warps: TMA instructions issue serially within a warp, and a stage's 128
    // gather4 ops spread over 12-15 warps land ~1.1-1.15x faster than over 8
    // (tools/microbench_feed.cu); 20 warps in all keep 96 registers per thread (21 would cap at 80)
    if (tile_t == 256) return run_spmm<SpmmCfg<1, 256, 2, VENOM_GATHER_P, 1, PRE>, kBF16>(tv, tb, te, tc, p, max_ctas, s);
    if (tile_t == 192) return run_spmm<SpmmCfg<1, 192, 3, 8, 1, PRE>, kBF16>(tv, tb, te, tc, p, max_ctas, s);
    if (tile_t == 128) return run_spmm<SpmmCfg<1, 128, 4, 8, 1, PRE>, kBF16>(tv, tb, te, tc, p, max_ctas, s);
    if (tile_t == 64) return run_spmm<SpmmCfg<1, 64, 4, 8, 1, PRE>, kBF16>(tv, tb, te, tc, p, max_ctas, s);
  } else if (NBg == 2) {
    // 11 gather-issuing warps as for V = 128 (8 with the 4 metadata warps: 768 threads would cap
    // registers at 80)
    if (tile_t == 128) return run_spmm<SpmmCfg<2, 128, 2, PRE ? 11 : 8, 1, PRE>, kBF16>(tv, tb, te, tc, p, max_ctas, s);
    if (tile_t == 64) return run_spmm<SpmmCfg<2, 64, 4, 8, 1, PRE>, kBF16>(tv, tb, te, tc, p, max_ctas, s);
  } else {
    if (tile_t == 64) return run_spmm<SpmmCfg<4, 64, 2, PRE ? 11 : 8, 1, PRE>, kBF16>(tv, tb, te, tc, p, max_ctas, s);
  }
  return VENOM_ERR_INVALID_ARGUMENT;  // tile override not available for this V
}

// ------------------------------------------------------------------ dense-K kernel
template <class Cfg, bool kBF16>
venom_status_t run_densek(const CUtensorMap& tb, EncodeTiledFn enc, SpmmParams p, int max_ctas,
                          cudaStream_t s) {
  // compressed values: 2-D [R rows][2G] 16-bit, box VE × 128 rows (one k-stage), no swizzle
  CUtensorMap tv;
  {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(2 * p.G), static_cast<cuuint64_t>(p.R)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(4 * static_cast<int64_t>(p.G))};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(Cfg::VE), 128};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tv, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<uint16_t*>(p.values), dims, strides,
            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return VENOM_ERR_CUDA;
  }
  auto kern = vnm_spmm_densek_kernel<Cfg, kBF16>;
  const int smem = Cfg::SMEM_BYTES < 116 * 1024 ? 116 * 1024 : Cfg::SMEM_BYTES;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return VENOM_ERR_CUDA;
  const int sms = sm_count();
  int grid = p.num_tiles * Cfg::CG < sms ? p.num_tiles * Cfg::CG : sms;
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  if (grid < 1) return VENOM_OK;
  return launch_cg(kern, Cfg::CG, grid, Cfg::NUM_THREADS, smem, s, tb, tv, p);
}

template <int BN, int ST, int CG, bool kBF16>
venom_status_t run_densek_m(int M, const CUtensorMap& tb, EncodeTiledFn enc, SpmmParams p, int max_ctas,
                            cudaStream_t s) {
  p.m_tiles = static_cast<int>((p.R + 128 * CG - 1) / (128 * CG));
  p.num_tiles = p.m_tiles * p.n_tiles;
  p.group_n = 1;
  switch (M) {
    case 4: return run_densek<DenseKCfg<BN, ST, 4, CG>, kBF16>(tb, enc, p, max_ctas, s);
    case 8: return run_densek<DenseKCfg<BN, ST, 8, CG>, kBF16>(tb, enc, p, max_ctas, s);
    case 16: return run_densek<DenseKCfg<BN, ST, 16, CG>, kBF16>(tb, enc, p, max_ctas, s);
    case 32: return run_densek<DenseKCfg<BN, ST, 32, CG>, kBF16>(tb, enc, p, max_ctas, s);
  }
  return VENOM_ERR_UNSUPPORTED_PATTERN;
}

template <bool kBF16>
venom_status_t run_densek_cfg(int M, int pair, int tile_t, const CUtensorMap& tb, EncodeTiledFn enc,
                              SpmmParams p, int max_ctas, cudaStream_t s) {
  if (pair == 2) {
    if (tile_t == 256) return run_densek_m<256, 4, 2, kBF16>(M, tb, enc, p, max_ctas, s);
    if (tile_t == 128) return run_densek_m<128, 6, 2, kBF16>(M, tb, enc, p, max_ctas, s);
  } else {
    if (tile_t == 256) return run_densek_m<256, 2, 1, kBF16>(M, tb, enc, p, max_ctas, s);
    if (tile_t == 128) return run_densek_m<128, 4, 1, kBF16>(M, tb, enc, p, max_ctas, s);
  }
  return VENOM_ERR_INVALID_ARGUMENT;
}

// ------------------------------------------------------------------ launchers (one per unit)
#define VENOM_GATHER_ARGS                                                                       \
  int NBg, int pair, int tile_t, const CUtensorMap &tv, const CUtensorMap &tb, const CUtensorMap &te, \
      const CUtensorMap &tc, SpmmParams p, int max_ctas, cudaStream_t s
#define VENOM_DENSEK_ARGS \
  int M, int pair, int tile_t, const CUtensorMap &tb, EncodeTiledFn enc, SpmmParams p, int max_ctas, cudaStream_t s

venom_status_t gather_pre_f16(VENOM_GATHER_ARGS);     // tu_gather_pre_f16.cu
venom_status_t gather_pre_bf16(VENOM_GATHER_ARGS);    // tu_gather_pre_bf16.cu
venom_status_t gather_nopre_f16(VENOM_GATHER_ARGS);   // tu_gather_nopre_*.cu
venom_status_t gather_nopre_bf16(VENOM_GATHER_ARGS);  // tu_gather_nopre_*.cu
venom_status_t densek_f16(VENOM_DENSEK_ARGS);         // tu_densek_*.cu
venom_status_t densek_bf16(VENOM_DENSEK_ARGS);        // tu_densek_*.cu

}  // namespace launch
}  // namespace venom
