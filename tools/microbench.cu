// microbench.cu — feasibility microbenchmarks for the SpMM design:
//   gather : TMA tile::gather4 throughput (L2/HBM -> SMEM) per SM and chip-wide, vs tile loads
//   mma    : tcgen05.mma.sp (kind::f16, M=128) issue rate from SMEM operands, vs dense
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o microbench tools/microbench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2310_02065_b200/csrc/ptx_sm100.cuh"

using namespace venom::ptx;

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

// ---------------------------------------------------------------------------- gather
// mode 0: gather4 of pseudo-random rows; mode 1: gather4 of consecutive rows;
// mode 2: tile box {64 cols, 4 rows}; mode 3: tile box {64 cols, 32 rows};
// mode 4: cp.async 16-byte gathers of pseudo-random 128-byte rows (all 32 lanes, 4 rows / instr)
// Each of `nw` warps runs an independent ring of `stages` stages in its own smem region.
__global__ void __launch_bounds__(256, 1) gather_kernel(const __grid_constant__ CUtensorMap tm1,
                                                        const __grid_constant__ CUtensorMap tm4,
                                                        const __grid_constant__ CUtensorMap tm32,
                                                        const uint16_t* __restrict__ Bp,
                                                        int mode, int stages, int ops_per_stage,
                                                        int iters, int K, int T, int issuers, int nw,
                                                        unsigned long long* cycles) {
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  const int stage_bytes = ops_per_stage * 512;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + nw * stages * stage_bytes);
  const uint32_t bar0 = smem_u32(bars) + warp * 8 * stages;
  const uint32_t s0 = smem_u32(smem) + warp * stages * stage_bytes;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages * nw; ++s) mbar_init(smem_u32(bars) + 8 * s, (mode == 4 || mode == 6 || ((mode == 5 || mode == 7) && s >= ((mode == 5 ? nw / 2 : (3 * nw) / 4) * stages))) ? 32 : 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (warp >= nw) return;
  if (mode == 5) mode = (warp < nw / 2) ? 0 : 4;
  if (mode == 7) mode = (warp < (3 * nw) / 4) ? 0 : 4;
  const uint64_t pol = policy_evict_normal();
  unsigned long long t0 = clock64();
  uint32_t rng = 12345u + blockIdx.x * 7919u + lane * 104729u + warp * 7u;
  for (int it = 0; it < iters; ++it) {
    const int s = it % stages;
    if (it >= stages) mbar_wait(bar0 + 8 * s, ((it / stages) - 1) & 1);
    const uint32_t dst = s0 + s * stage_bytes;
    if (mode == 6) {
      // plain LDG.128 -> registers -> STS.128 (4 rows of 128 B per warp instruction)
      const int rr = lane >> 3, ch = lane & 7;
      for (int op0 = 0; op0 < ops_per_stage; op0 += 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          rng = rng * 1664525u + 1013904223u;
          const int row = (__shfl_sync(0xffffffffu, (int)((rng >> 8) % K), rr * 8));
          const int col = (((op0 + u) * 64) + blockIdx.x * 128) % T;
          v[u] = __ldcg(reinterpret_cast<const uint4*>(Bp + (size_t)row * T + col + ch * 8));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          uint8_t* d = smem + (dst - smem_u32(smem)) + (op0 + u) * 512 + rr * 128 + ((ch ^ rr) << 4);
          *reinterpret_cast<uint4*>(d) = v[u];
        }
      }
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar0 + 8 * s) : "memory");
      continue;
    }
    if (mode == 4) {
      // lane = 8 * row_in_op + chunk: 4 rows of 128 B per warp instruction
      const int rr = lane >> 3, ch = lane & 7;
      for (int op = 0; op < ops_per_stage; ++op) {
        rng = rng * 1664525u + 1013904223u;
        const int row = (__shfl_sync(0xffffffffu, (int)((rng >> 8) % K), rr * 8));
        const int col = ((op * 64) + blockIdx.x * 128) % T;
        const uint16_t* src = Bp + (size_t)row * T + col + ch * 8;
        const uint32_t d = dst + op * 512 + rr * 128 + ((ch ^ (rr + 4 * (op & 1))) << 4);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar0 + 8 * s) : "memory");
      continue;
    }
    if (lane == 0) mbar_arrive_expect_tx(bar0 + 8 * s, stage_bytes);
    __syncwarp();
    for (int op = lane; op < ops_per_stage; op += issuers) {
      if (lane >= issuers) break;
      const int col = ((op * 64) + blockIdx.x * 128) % T;
      if (mode == 0) {
        int r[4];
        for (int t = 0; t < 4; ++t) {
          rng = rng * 1664525u + 1013904223u;
          r[t] = (rng >> 8) % K;
        }
        tma_gather4(dst + op * 512, &tm1, bar0 + 8 * s, col, r[0], r[1], r[2], r[3], pol);
      } else if (mode == 1) {
        const int r0 = ((it * ops_per_stage + op) * 4 + blockIdx.x * 64) % (K - 4);
        tma_gather4(dst + op * 512, &tm1, bar0 + 8 * s, col, r0, r0 + 1, r0 + 2, r0 + 3, pol);
      } else if (mode == 2) {
        const int r0 = ((it * ops_per_stage + op) * 4 + blockIdx.x * 64) % (K - 4);
        tma_load_2d(dst + op * 512, &tm4, bar0 + 8 * s, col, r0, pol);
      } else {
        if (op % 8 == 0) {
          const int r0 = ((it * ops_per_stage + op) * 4 + blockIdx.x * 64) % (K - 32);
          tma_load_2d(dst + op * 512, &tm32, bar0 + 8 * s, col, r0, pol);
        }
      }
    }
  }
  for (int s = 0; s < stages && s < iters; ++s) {
    const int last = iters - 1 - ((iters - 1 - s) % stages);
    mbar_wait(bar0 + 8 * s, (last / stages) & 1);
  }
  unsigned long long t1 = clock64();
  if (lane == 0 && warp == 0) cycles[blockIdx.x] = t1 - t0;
}

// ---------------------------------------------------------------------------- mma
template <bool kSparse, int BN>
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  // zero operands (values irrelevant for rate)
  for (int i = threadIdx.x; i < (16384 + 65536 + 2048) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0x44444444u);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<512>(smem_u32(&tbase));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase;
  const uint32_t sA = smem_u32(smem), sB = sA + 16384, sE = sB + 65536;
  unsigned long long t0 = clock64();
  if (warp == 1 && (threadIdx.x & 31) == 0) {
    if (kSparse) tc_cp_128x128b(tb + 504, smem_desc(sE, 16, 128, 0));
    const uint32_t idesc = kSparse ? idesc_sp_f16(0, 128, BN)
                                   : ((1u << 4) | (1u << 16) | ((BN >> 3) << 17) | ((128 >> 4) << 24));
    for (int it = 0; it < iters; ++it) {
      for (int kb = 0; kb < 4; ++kb) {
        const uint64_t ad = smem_desc(sA + kb * 32, 16, 1024, 2);
        const uint64_t bd = smem_desc(sB + kb * (kSparse ? 4096 : 2048), 16384, 1024, 2);
        if (kSparse) {
          const uint32_t e = tb + 504 + kb;
          tc_mma_sp_f16(tb, ad, bd, idesc | (e & 1), e & ~1u, 1);
        } else {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tb),
                       "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
        }
      }
    }
    tc_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 32) cycles[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tb);
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int dev = 0;
  CK(cudaSetDevice(dev));
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncFn enc = reinterpret_cast<EncFn>(fp);
  unsigned long long* d_cyc;
  CK(cudaMalloc(&d_cyc, sizeof(unsigned long long) * 1024));
  std::vector<unsigned long long> cyc(1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);

  // ---------------- gather: B is K x T fp16
  for (int big = 0; big < 2; ++big) {
    const long K = big ? 49152 : 4096, T = big ? 8192 : 4096;
    void* B;
    CK(cudaMalloc(&B, 2 * K * T));
    CK(cudaMemset(B, 0, 2 * K * T));
    CUtensorMap tm1, tm4, tm32;
    cuuint64_t dims[2] = {(cuuint64_t)T, (cuuint64_t)K};
    cuuint64_t str[1] = {(cuuint64_t)(2 * T)};
    cuuint32_t es[2] = {1, 1};
    cuuint32_t b1[2] = {64, 1}, b4[2] = {64, 4}, b32[2] = {64, 32};
    enc(&tm1, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, B, dims, str, b1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&tm4, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, B, dims, str, b4, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&tm32, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, B, dims, str, b32, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const char* names[8] = {"gather4-random", "gather4-seq", "tile-64x4", "tile-64x32", "cpasync-random", "mixed-tma+cpa", "ldg128+sts", "mixed-3tma:1cpa"};
    // stages, ops/stage, issuers, issuing warps
    int cfgs[][4] = {{4, 64, 32, 1}, {2, 64, 32, 2}, {2, 32, 32, 4}, {2, 16, 32, 8}, {3, 32, 32, 4}, {3, 16, 32, 8}, {6, 8, 32, 8}};
    for (int mode = 0; mode < 8; ++mode) {
      if (mode == 1 || mode == 2 || mode == 3) continue;
      if (big == 1 && mode != 0 && mode != 5) continue;
      for (auto& c : cfgs) {
        const int stages = c[0], ops = c[1], issuers = c[2], nw = c[3];
        if ((mode >= 3) && issuers != 32) continue;
        const int iters = 2000;
        const int smem = nw * stages * ops * 512 + 1024 + 1024;
        CK(cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        gather_kernel<<<sms, 256, smem>>>(tm1, tm4, tm32, (const uint16_t*)B, mode, stages, ops, 10, K, T, issuers, nw, d_cyc);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        gather_kernel<<<sms, 256, smem>>>(tm1, tm4, tm32, (const uint16_t*)B, mode, stages, ops, iters, K, T, issuers, nw, d_cyc);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        CK(cudaMemcpy(cyc.data(), d_cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost));
        double avgc = 0;
        for (int i = 0; i < sms; ++i) avgc += cyc[i];
        avgc /= sms;
        const double bytes = double(sms) * nw * iters * ops * 512;
        printf("%-15s K=%-6ld warps=%d stages=%d ops/stage=%3d issuers=%2d: %8.1f GB/s chip, %6.1f B/cycle/SM\n",
               names[mode], K, nw, stages, ops, issuers, bytes / ms / 1e6, double(nw) * iters * ops * 512 / avgc);
      }
    }
    CK(cudaFree(B));
  }

  // ---------------- mma
  auto run_mma = [&](auto kern, const char* name, double flop_per_iter) {
    const int smem = 16384 + 65536 + 2048 + 1024;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int iters = 20000;
    kern<<<sms, 128, smem>>>(100, d_cyc);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    kern<<<sms, 128, smem>>>(iters, d_cyc);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    CK(cudaMemcpy(cyc.data(), d_cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost));
    double avgc = 0;
    for (int i = 0; i < sms; ++i) avgc += cyc[i];
    avgc /= sms;
    printf("%-28s: %8.1f TFLOP/s (issued, dense-equivalent), %7.1f cycles per 4-MMA stage\n", name,
           flop_per_iter * iters * sms / ms / 1e9, avgc / iters);
  };
  run_mma(mma_kernel<true, 256>, "sparse M128 N256 K32 x4", 2.0 * 128 * 256 * 32 * 4);
  run_mma(mma_kernel<true, 128>, "sparse M128 N128 K32 x4", 2.0 * 128 * 128 * 32 * 4);
  run_mma(mma_kernel<false, 256>, "dense  M128 N256 K16 x4", 2.0 * 128 * 256 * 16 * 4);
  run_mma(mma_kernel<false, 128>, "dense  M128 N128 K16 x4", 2.0 * 128 * 128 * 16 * 4);
  return 0;
}
