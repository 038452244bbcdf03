// microbench_stream.cu — chip-wide TMA tile streaming throughput from L2 (DESIGN.md §6 "feed").
// Every CTA streams 16 KB boxes (64 columns × 128 rows, 128B swizzle) through an S-stage ring of
// `boxes` boxes per stage: one thread issues, one thread consumes (wait full -> arrive empty), no
// MMA. Sources are L2-resident (the buffer is read once before timing). `share` = how many CTAs read
// the same box sequence at the same time (1 = all distinct; 16 ≈ the SpMM's B slab sharing);
// `mc` = cluster size for TMA multicast (each CTA of the cluster issues 1/mc of every stage's boxes
// and multicasts them to all CTAs of the cluster).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/microbench_stream tools/microbench_stream.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2310_02065_b200/csrc/ptx_sm100.cuh"

using namespace venom::ptx;

__device__ __forceinline__ void tma_load_mc(uint32_t dst, const void* map, uint32_t bar, int c0, int c1,
                                            uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, int rows,
                                                        int colblocks, int iters, int S, int boxes,
                                                        int share, int mc, unsigned long long* out) {
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16], empty[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = mc > 1 ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), mc);  // every CTA of the cluster must release a stage
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (mc > 1) cluster_sync();
  const int group = blockIdx.x / (share * mc);  // CTAs of one group read the same sequence
  const unsigned long long t0 = clock64();
  const int per = boxes / mc;                    // boxes this CTA issues per stage
  if (warp == 0 && lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      mbar_wait(smem_u32(&empty[s]), ((it / S) & 1) ^ 1);
      mbar_arrive_expect_tx(smem_u32(&full[s]), boxes * 16384);
      for (int b = 0; b < per; ++b) {
        const int bb = rank * per + b;
        const long long lin = (static_cast<long long>(group) * 7919 + static_cast<long long>(it) * boxes + bb);
        const int cb = static_cast<int>(lin % colblocks);
        const int rb = static_cast<int>((lin / colblocks) % (rows / 128));
        const uint32_t dst = smem_u32(smem) + (s * boxes + bb) * 16384;
        if (mc > 1) tma_load_mc(dst, &tm, smem_u32(&full[s]), cb * 64, rb * 128, (1u << mc) - 1);
        else tma_load_2d(dst, &tm, smem_u32(&full[s]), cb * 64, rb * 128, 0);
      }
    }
  } else if (warp == 1 && lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      mbar_wait(smem_u32(&full[s]), (it / S) & 1);
      // release the stage in every CTA of the cluster (their multicasts write into our smem)
      for (int c = 0; c < mc; ++c) {
        if (mc > 1) mbar_arrive_cluster(mapa_shared(smem_u32(&empty[s]), c));
        else mbar_arrive(smem_u32(&empty[s]));
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  if (mc > 1) cluster_sync();
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
  const int rows = 8192, cols = 4096;  // 64 MB fp16: L2-resident
  uint16_t* buf;
  cudaMalloc(&buf, size_t(rows) * cols * 2);
  cudaMemset(buf, 0, size_t(rows) * cols * 2);
  CUtensorMap tm;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* d;
  cudaMalloc(&d, 8 * 1024);
  struct Case { int S, boxes, share, mc; };
  std::vector<Case> cases = {{4, 3, 1, 1}, {6, 2, 1, 1}, {12, 1, 1, 1}, {3, 4, 1, 1}, {4, 3, 16, 1},
                             {4, 2, 1, 2}, {4, 2, 1, 1}, {6, 2, 1, 2}, {4, 4, 1, 4}, {3, 4, 1, 4},
                             {4, 2, 8, 2}, {4, 3, 1, 1}};
  const int grids[4] = {0, 74, 32, 8};
  for (int gi = 0; gi < 4; ++gi)
  for (const Case& c : cases) {
    if (gi > 0 && !(c.mc == 1 && c.share == 1 && c.S == 4 && c.boxes == 3) && !(c.mc == 2 && c.S == 4 && c.share == 1)) continue;
    const int smem = c.S * c.boxes * 16384 + 1024;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    const int grid = (gi == 0 ? sms : grids[gi]) - (gi == 0 ? sms : grids[gi]) % (c.mc);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c.mc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, stream_kernel, tm, rows, cols / 64, 50, c.S, c.boxes, c.share, c.mc, d);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, stream_kernel, tm, rows, cols / 64, iters, c.S, c.boxes, c.share, c.mc, d);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = double(grid) * iters * c.boxes * 16384;  // bytes landed in SMEM
    printf("grid=%3d S=%2d boxes/stage=%d (%3d KB/stage) share=%2d mc=%d: %7.2f TB/s landed in SMEM (%.1f B/ns per SM), "
           "L2 reads %.2f TB/s %s\n",
           grid, c.S, c.boxes, c.boxes * 16, c.share, c.mc, bytes / ms / 1e9, bytes / ms / 1e6 / grid,
           bytes / c.mc / ms / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
