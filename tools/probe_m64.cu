// probe_m64.cu — TMEM layouts of the M = 64 sparse MMA (tcgen05.mma.sp.cta_group::1.kind::f16,
// M = 64, N = 64, K = 32), measured on the hardware: where the accumulator rows land (and whether a
// lane offset of 16 in the D address places a second 64-row accumulator on the other half of each
// lane quarter), and which TMEM lane / nibble of the metadata column serves which (row, group).
// Used to lay out the V = 64 path of spmm_kernel.cuh (two 64-row V-blocks per 128-lane accumulator).
//
//   mode 0: D layout. A[r][*] = r + 1, metadata all (0,1), B[k] = 1 at k % 4 in {0,1}
//           -> D[r] = 16 (r + 1); prints the TMEM lane of every row (D at lane offset `doff`).
//   mode 1: metadata layout. A = 1, B[4g+2] = 2^g (else 0), metadata all (0,1) except one nibble
//           (lane L, nibble n) = (2,3) -> exactly one row gains 2^g; prints (L, n) -> (D lane, g).
//           `eoff` adds a lane offset to the metadata address.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probe_m64 tools/probe_m64.cu
// Run:   tools/probe_m64 MODE DOFF EOFF
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../paper_2310_02065_b200/csrc/ptx_sm100.cuh"

using namespace venom::ptx;

__device__ __forceinline__ uint16_t f2h(float f) { return __half_as_ushort(__float2half_rn(f)); }

__global__ void __launch_bounds__(128, 1) probe(int mode, uint32_t doff, uint32_t eoff, float* out) {
  __shared__ __align__(1024) uint8_t a_s[64 * 128];
  __shared__ __align__(1024) uint8_t b_s[32 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // A: 64 rows × 64 compressed values (K-major SW128); only values 0..15 feed the K = 32 MMA
  for (int i = threadIdx.x; i < 64 * 64; i += 128) {
    const int r = i / 64, j = i % 64;
    const float v = (mode == 0) ? static_cast<float>(r + 1) : 1.0f;
    const int byte = r * 128 + ((((j * 2) >> 4) ^ (r & 7)) << 4) + (j * 2) % 16;
    *reinterpret_cast<uint16_t*>(a_s + byte) = f2h(j < 16 ? v : 0.0f);
  }
  // B: 32 K-rows × 64 columns (MN-major SW128)
  for (int i = threadIdx.x; i < 32 * 64; i += 128) {
    const int k = i / 64, n = i % 64;
    float v = 0.0f;
    if (mode == 0) v = (k % 4 < 2) ? 1.0f : 0.0f;
    else v = (k % 4 == 2) ? static_cast<float>(1 << (k / 4)) : 0.0f;
    const int byte = k * 128 + ((((n * 2) >> 4) ^ (k & 7)) << 4) + (n * 2) % 16;
    *reinterpret_cast<uint16_t*>(b_s + byte) = f2h(v);
  }
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
  const uint32_t E = 256;  // metadata column
  const uint64_t adesc = smem_desc(smem_u32(a_s), 16, 1024, 2);
  const uint64_t bdesc = smem_desc(smem_u32(b_s), 16384, 1024, 2);
  const uint32_t idesc = idesc_sp_f16(0, 64, 64);
  const int nprobe = (mode == 0) ? 1 : 128 * 8;
  for (int pi = 0; pi < nprobe; ++pi) {
    // metadata: every nibble (0,1) = 0x4, except (lane pi / 8, nibble pi % 8) = (2,3) = 0xE in mode 1
    const int myl = 32 * warp + lane;
    uint32_t m = 0x44444444u;
    if (mode == 1 && myl == pi / 8) m = (m & ~(0xFu << (4 * (pi % 8)))) | (0xEu << (4 * (pi % 8)));
    tmem_st_32x32b_x2(tb + (static_cast<uint32_t>(32 * warp) << 16) + E, m, m);
    // clear the accumulator region (both lane halves) so stale values cannot masquerade
    uint32_t z[16] = {};
    tmem_st_32x32b_x16(tb + (static_cast<uint32_t>(32 * warp) << 16), z);
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      tc_mma_sp_f16(tb + (doff << 16), adesc, bdesc, idesc, tb + (eoff << 16) + E, 0u);
      tc_commit(smem_u32(&bar));
    }
    mbar_wait(smem_u32(&bar), pi & 1);
    tc_fence_after();
    uint32_t v[16];
    tmem_ld_32x32b_x16(tb + (static_cast<uint32_t>(32 * warp) << 16), v);
    tmem_ld_wait();
    out[pi * 128 + myl] = __uint_as_float(v[0]);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (warp == 0) tmem_dealloc<512>(tb);
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const uint32_t doff = argc > 2 ? atoi(argv[2]) : 0, eoff = argc > 3 ? atoi(argv[3]) : 0;
  const int nprobe = (mode == 0) ? 1 : 1024;
  float* d;
  cudaMalloc(&d, nprobe * 128 * 4);
  cudaMemset(d, 0, nprobe * 128 * 4);
  probe<<<1, 128>>>(mode, doff, eoff, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("mode %d doff %u eoff %u: CUDA error %s\n", mode, doff, eoff, cudaGetErrorString(e));
    return 1;
  }
  float* h = static_cast<float*>(malloc(nprobe * 128 * 4));
  cudaMemcpy(h, d, nprobe * 128 * 4, cudaMemcpyDeviceToHost);
  printf("mode %d doff %u eoff %u\n", mode, doff, eoff);
  if (mode == 0) {
    // row r -> lanes holding 16 (r + 1)
    for (int l = 0; l < 128; ++l) {
      const float v = h[l];
      if (v != 0.0f) printf("lane %3d: %g -> row %g\n", l, v, v / 16.0f - 1.0f);
    }
  } else {
    for (int pi = 0; pi < nprobe; ++pi) {
      printf("meta lane %3d nibble %d ->", pi / 8, pi % 8);
      int hits = 0;
      for (int l = 0; l < 128; ++l) {
        const float v = h[pi * 128 + l];
        if (v != 0.0f) {
          printf(" Dlane %d val %g;", l, v);
          ++hits;
        }
      }
      printf(hits ? "\n" : " none\n");
    }
  }
  return 0;
}
