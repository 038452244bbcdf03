// microbench_mma.cu — sparse tcgen05 MMA rate vs concurrent shared-memory traffic (SURVEY §7a
// step 6). Operands stay resident in SMEM (no loads):
//   CG = 1: tcgen05.mma.sp.cta_group::1, M = 128, N = 256, K = 32 (× 4 per stage)
//   CG = 2: tcgen05.mma.sp.cta_group::2, M = 256 (128 per CTA), N = 256 (128 columns per CTA)
// while `nsts` other warps stream STS.128 into a scratch region (optionally with a
// fence.proxy.async after every 8 stores, the pattern the dense-K expanders use).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/microbench_mma tools/microbench_mma.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2310_02065_b200/csrc/ptx_sm100.cuh"

using namespace venom::ptx;

struct Out {
  unsigned long long mma_cycles, sts_bytes, fences, sts_cycles;
};

// side-warp traffic kinds: 0 STS.128, 1 LDS.128, 2 LDG.128 (L1-resident buffer), 3 tcgen05.st
// (16 columns), 4 tcgen05.ld (16 columns)
template <int CG, bool kFence, int KIND = 0>
__global__ void __launch_bounds__(384, 1) mma_sts_kernel(int iters, int nsts, Out* out,
                                                         const uint4* __restrict__ gbuf) {
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int BBYTES = 65536 / CG;
  const uint32_t sA = smem_u32(smem), sB = sA + 16384, sE = sB + BBYTES, sS = sE + 2048;
  for (int i = threadIdx.x; i < (16384 + BBYTES + 2048) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0x44444444u);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    done = 0;
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) {
    if constexpr (CG == 2) tmem_alloc_2sm<512>(smem_u32(&tbase));
    else tmem_alloc<512>(smem_u32(&tbase));
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  tc_fence_after();
  const uint32_t tb = tbase;
  const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0u;
  if (warp == 1) {
    if (rank == 0 && lane == 0) {
      const unsigned long long t0 = clock64();
      const uint32_t idesc = idesc_sp_f16(0, 128 * CG, 256);
      if constexpr (CG == 2) tc_cp_128x128b_2sm(tb + 504, smem_desc(sE, 16, 128, 0));
      else tc_cp_128x128b(tb + 504, smem_desc(sE, 16, 128, 0));
      for (int it = 0; it < iters; ++it) {
        for (int kb = 0; kb < 4; ++kb) {
          const uint64_t ad = smem_desc(sA + kb * 32, 16, 1024, 2);
          const uint64_t bd = smem_desc(sB + kb * 4096, 16384, 1024, 2);
          const uint32_t e = tb + 504 + kb;
          if constexpr (CG == 2) tc_mma_sp_f16_2sm(tb, ad, bd, idesc | (e & 1), e & ~1u, 1);
          else tc_mma_sp_f16(tb, ad, bd, idesc | (e & 1), e & ~1u, 1);
        }
      }
      if constexpr (CG == 2) tc_commit_2sm_mc(smem_u32(&bar), 0x3);
      else tc_commit(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), 0);
      out[blockIdx.x].mma_cycles = clock64() - t0;
      done = 1;
    }
    if (rank != 0 && lane == 0) {
      mbar_wait(smem_u32(&bar), 0);  // multicast commit arrives here too
      done = 1;
    }
  } else if (warp >= 2 && warp < 2 + nsts) {
    // STS.128 stream into a 32 KB scratch region (row = lane, 16 chunks)
    unsigned long long bytes = 0, fences = 0;
    const unsigned long long t0 = clock64();
    uint8_t* scr = smem + (sS - sA) + (warp - 2) * 4096;
    uint4 v = make_uint4(lane, warp, 0, 0);
    uint32_t acc = 0;
    const uint32_t tl = tb + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + 256 + 16 * ((warp - 2) >> 2);
    while (!done) {
      if constexpr (KIND == 0) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(scr + ((lane * 8 + c) % 256) * 16)),
                       "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
          v.x += 1;
        }
      } else if constexpr (KIND == 1) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint4 w;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                       : "r"(smem_u32(scr + ((lane * 8 + c) % 256) * 16)) : "memory");
          acc += w.x ^ w.w;
        }
      } else if constexpr (KIND == 2) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 w = __ldg(gbuf + ((lane * 8 + c + acc) & 1023));
          acc += w.x ^ w.w;
        }
      } else if constexpr (KIND == 3) {
        uint32_t r16[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) r16[c] = v.x + c;
        tmem_st_32x32b_x16(tl, r16);
        tmem_st_32x32b_x16(tl, r16);
        tmem_st_wait();
        v.x += 1;
      } else {
        uint32_t r32[32];
        tmem_ld_32x32b_x32(tl, r32);
        tmem_ld_wait();
        acc += r32[0] ^ r32[31];
      }
      bytes += 8 * 16 * 32;
      if (kFence) {
        fence_proxy_async_smem();
        ++fences;
      }
    }
    if (acc == 0x12345678u) bytes += 1;  // keep the loads alive
    if (lane == 0) {
      atomicAdd(&out[blockIdx.x].sts_bytes, bytes);
      atomicAdd(&out[blockIdx.x].fences, fences);
      atomicMax(&out[blockIdx.x].sts_cycles, clock64() - t0);
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_2sm<512>(tb);
    else tmem_dealloc<512>(tb);
  }
}

template <int CG, bool kFence, int KIND = 0>
void run(int sms, int nsts, const char* name, const uint4* gbuf = nullptr, int miters = 4000) {
  auto kern = mma_sts_kernel<CG, kFence, KIND>;
  const int smem = 16384 + 65536 / CG + 2048 + 8 * 4096 + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  Out* d;
  cudaMalloc(&d, sizeof(Out) * 256);
  const int iters = miters;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(d, 0, sizeof(Out) * 256);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms - sms % CG);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, iters, nsts, d, gbuf);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: error %s\n", name, cudaGetErrorString(e));
      exit(1);
    }
  }
  std::vector<Out> h(256);
  cudaMemcpy(h.data(), d, sizeof(Out) * 256, cudaMemcpyDeviceToHost);
  double mc = 0, sb = 0, sc = 0, fe = 0;
  int n = 0;
  for (int i = 0; i < sms; i += CG) {
    mc += h[i].mma_cycles;
    ++n;
  }
  for (int i = 0; i < sms; ++i) {
    sb += h[i].sts_bytes;
    sc += h[i].sts_cycles;
    fe += h[i].fences;
  }
  mc /= n;
  sb /= sms;
  sc /= sms;
  fe /= sms;
  printf("%-34s nsts=%d: %7.1f cycles per 4-MMA stage; per-SM STS %6.1f B/cycle; %s%.0f cycles/fence\n",
         name, nsts, mc / iters, sc > 0 ? sb / sc : 0.0, kFence ? "" : "(no fence) ",
         (kFence && fe > 0) ? sc / (fe / (nsts > 0 ? nsts : 1)) : 0.0);
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4* g;
  cudaMalloc(&g, 1024 * 16);
  cudaMemset(g, 0, 1024 * 16);
  for (int nsts : {0, 1, 2, 4, 8}) {
    run<1, false>(sms, nsts, "1-CTA sparse M128 N256");
    if (nsts) run<1, true>(sms, nsts, "1-CTA sparse M128 N256 + fence");
    run<2, false>(sms, nsts, "2-CTA sparse M256 N256");
    if (nsts) run<2, true>(sms, nsts, "2-CTA sparse M256 N256 + fence");
  }
  // side traffic of other kinds against the 2-CTA MMA (and with the MMA idle: iters = 1)
  for (int nsts : {2, 8}) {
    run<2, false, 1>(sms, nsts, "2-CTA MMA + LDS.128", g);
    run<2, false, 2>(sms, nsts, "2-CTA MMA + LDG.128 (L1 hit)", g);
    run<2, false, 3>(sms, nsts, "2-CTA MMA + tcgen05.st x16", g);
    run<2, false, 4>(sms, nsts, "2-CTA MMA + tcgen05.ld x32", g);
    run<2, false, 0>(sms, nsts, "idle MMA + STS.128", g, 1);
    run<2, false, 1>(sms, nsts, "idle MMA + LDS.128", g, 1);
    run<2, false, 2>(sms, nsts, "idle MMA + LDG.128 (L1 hit)", g, 1);
  }
  return 0;
}
