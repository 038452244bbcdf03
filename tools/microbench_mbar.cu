// microbench_mbar.cu — mbarrier hand-off cost on B200.
// Two roles ping-pong over S stages: producer waits empty[s], arrives full[s]; consumer waits
// full[s], arrives empty[s] (plain arrive, or tcgen05.commit with no MMA in flight). Reports cycles
// per stage iteration for: S, lanes spinning (1 or 32), try_wait vs test_wait, and extra idle
// spinning warps on other barriers.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/microbench_mbar tools/microbench_mbar.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2310_02065_b200/csrc/ptx_sm100.cuh"

using namespace venom::ptx;

__device__ __forceinline__ uint32_t test_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok;
}

template <bool kTest>
__device__ __forceinline__ void wait(uint32_t bar, uint32_t parity) {
  if constexpr (kTest) {
    while (!test_wait(bar, parity)) {
    }
  } else {
    while (!mbar_try_wait(bar, parity)) {
    }
  }
}

// mode bit 0: consumer uses tcgen05.commit instead of arrive; bit 1: only lane 0 waits
template <bool kTest>
__global__ void __launch_bounds__(512, 1) pingpong(int iters, int S, int mode, int idle_warps,
                                                   unsigned long long* out) {
  __shared__ uint64_t full[8], empty[8], dummy;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    mbar_init(smem_u32(&dummy), 1);
    fence_mbar_init();
  }
  if (warp == 1 && (mode & 1)) tmem_alloc<32>(smem_u32(&tslot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const bool one = mode & 2;
  const unsigned long long t0 = clock64();
  if (warp == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      if (!one || lane == 0) wait<kTest>(smem_u32(&empty[s]), ((it / S) & 1) ^ 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&full[s]));
    }
  } else if (warp == 1) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      if (!one || lane == 0) wait<kTest>(smem_u32(&full[s]), (it / S) & 1);
      __syncwarp();
      if (lane == 0) {
        if (mode & 1) tc_commit(smem_u32(&empty[s]));
        else mbar_arrive(smem_u32(&empty[s]));
      }
    }
    if (lane == 0) {
      out[blockIdx.x] = clock64() - t0;
      mbar_arrive(smem_u32(&dummy));
    }
  } else if (warp - 2 < idle_warps) {
    wait<kTest>(smem_u32(&dummy), 0);  // spins until the consumer is done
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1 && (mode & 1)) {
    tc_fence_after();
    tmem_dealloc<32>(tslot);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 1024);
  const int iters = 20000;
  for (int test = 0; test < 2; ++test)
    for (int mode = 0; mode < 4; ++mode)
      for (int idle : {0, 14})
        for (int S : {1, 2, 4}) {
          auto k = test ? pingpong<true> : pingpong<false>;
          k<<<148, 512>>>(iters, S, mode, idle, d);
          k<<<148, 512>>>(iters, S, mode, idle, d);
          cudaError_t e = cudaDeviceSynchronize();
          unsigned long long h = 0;
          cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
          printf("%s %-7s %-9s idle=%2d S=%d: %7.1f cycles/iter %s\n", test ? "test_wait" : "try_wait ",
                 (mode & 1) ? "commit" : "arrive", (mode & 2) ? "lane0" : "32lanes", idle, S,
                 double(h) / iters, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
  return 0;
}
