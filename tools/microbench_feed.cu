// microbench_feed.cu — the per-SM L2 -> SMEM feed of the gathered SpMM, measured independently of
// the kernel (VERDICT r1 "establish the landing ceiling independently").
//
// One persistent CTA per SM runs a ring of S stages shaped like the SpMM's (spmm_kernel.cuh):
// per stage an optional A tile (16 KB TMA box, K-major SW128) plus RT rows × 256 columns of B'
// (the 4 selected rows of each 16-row group, MN-major SW128, 64-column chunks), fetched by
//   - `ntw` TMA warps issuing tile::gather4 (4 rows × 128 B per op; one op per lane), and/or
//   - `nlw` LDG warps: one 512-byte B row per warp instruction (ld.global.v4), stored with
//     st.shared.v4 into the same swizzled layout, fence.proxy.async, one mbarrier arrive per warp;
//   - or contiguous 16 KB tile boxes (mode "tile": the dense-B feed of the 2:4 form).
// The consumer either releases the stage at once (no MMA), or issues the stage's 4 sparse MMAs
// (tcgen05.mma.sp M = 128, N = 256, K = 32; metadata 0x4 codes in TMEM) and commits the release —
// the real shared-memory contention between landing and the tensor core.
// B is [K = 49152][1024] fp16 (100 MB, L2-resident after warm-up); each CTA reads one of 4
// 256-column bands. Reported: bytes landed per cycle per SM (clock64 over the CTA's loop) and the
// chip-wide rate (CUDA events).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/microbench_feed tools/microbench_feed.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2310_02065_b200/csrc/ptx_sm100.cuh"

using namespace venom::ptx;

struct Cfg {
  int S;        // stages
  int rows;     // B' rows per stage (K' per stage: 128 or 64)
  int rt;       // rows fetched by TMA gather4 (the rest, rows - rt, by the LDG warps)
  int ntw;      // TMA-issuing warps
  int nlw;      // LDG warps
  int with_a;   // 16 KB A box per stage (8 KB when rows == 64)
  int tile;     // B' by contiguous tile boxes of `tile` rows × 64 columns instead of gathers
  int mma;      // consumer issues the stage's sparse MMAs
  int cpa;      // the non-TMA warps use cp.async (16 B per lane, completion via
                // cp.async.mbarrier.arrive.noinc; no register staging, several stages in flight)
  int iters;
};

constexpr int KROWS = 49152, TCOLS = 1024;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

// row of B for B' row j (0..rows-1) of stage iteration `it`: group g = it*rows/4 + j/4, 4 distinct
// rows of the 16-row group, ascending
__device__ __forceinline__ int brow(int it, int j, int rows, uint32_t salt) {
  const int g = static_cast<int>((static_cast<long long>(it) * (rows / 4) + j / 4) % (KROWS / 16));
  const uint32_t h = hash32(static_cast<uint32_t>(g) * 2654435761u ^ salt) & 3u;
  return g * 16 + static_cast<int>(h) + 4 * (j & 3);
}

__global__ void __launch_bounds__(512, 1) feed_kernel(const __grid_constant__ CUtensorMap tm_g,
                                                       const __grid_constant__ CUtensorMap tm_t,
                                                       const __grid_constant__ CUtensorMap tm_a,
                                                       const __grid_constant__ CUtensorMap tm_a64,
                                                       const uint16_t* __restrict__ Bp, Cfg c,
                                                       unsigned long long* cycles) {
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[8], empty[8], drain;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a_bytes = c.with_a ? (c.rows == 128 ? 16384 : 8192) : 0;
  const int b_bytes = c.rows * 512;                  // rows × 256 columns × 2 B
  const int chunk = c.rows * 128;                    // one 64-column chunk of B'
  const int stage_bytes = a_bytes + b_bytes;
  const int W_MMA = c.ntw + c.nlw;                   // consumer warp
  const uint32_t band = (blockIdx.x & 3) * 256;
  const uint32_t salt = blockIdx.x * 7919u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < c.S; ++s) {
      mbar_init(smem_u32(&full[s]), 1 + (c.cpa ? 32 * c.nlw : c.nlw));
      mbar_init(smem_u32(&empty[s]), 1);
    }
    mbar_init(smem_u32(&drain), 1);
    fence_mbar_init();
  }
  // metadata block for tcgen05.cp: 128 lanes x 16 B of the all-zero-value code 0x4 (m-indices 0, 1)
  uint8_t* meta = smem + 220 * 1024;
  for (int i = threadIdx.x; i < 128; i += blockDim.x)
    reinterpret_cast<uint4*>(meta)[i] = make_uint4(0x44444444u, 0x44444444u, 0x44444444u, 0x44444444u);
  fence_proxy_async_smem();
  if (c.mma && warp == W_MMA) tmem_alloc<512>(smem_u32(&tbase));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t s0 = smem_u32(smem);
  const uint64_t pol = policy_evict_last();
  const unsigned long long t0 = clock64();
  if (warp < c.ntw) {
    // ------------------------------------------------ TMA warps (warp 0 lane 0 also: expect_tx, A)
    // tile: boxes of c.tile rows × 64 columns; gather: (rows/4) × 4 chunks of gather4
    const int ops = c.tile ? 4 * (c.rows / c.tile) : (c.rt / 4) * 4;
    for (int it = 0; it < c.iters; ++it) {
      const int s = it % c.S;
      mbar_wait(smem_u32(&empty[s]), ((it / c.S) & 1) ^ 1);
      const uint32_t sb = s0 + s * stage_bytes;
      const uint32_t fb = smem_u32(&full[s]);
      if (warp == 0 && lane == 0) {
        const uint32_t tx = a_bytes + (c.tile ? b_bytes : c.rt * 512);
        mbar_arrive_expect_tx(fb, tx);
        if (c.with_a) tma_load_2d(sb, c.rows == 128 ? &tm_a : &tm_a64, fb, 0, (blockIdx.x * 128 + it * 128) % 8192, pol);
      }
      __syncwarp();
      // op o -> warp o % ntw, lane o / ntw: the ops of a stage are spread evenly over the warps
      // (TMA instructions issue serially within a warp)
      for (int o = lane * c.ntw + warp; o < ops; o += 32 * c.ntw) {
        if (c.tile) {
          // boxes of [tile rows][64 columns]: chunk o % 4, row slice o / 4 of consecutive rows
          const int r0 = (it * c.rows) % (KROWS - c.rows) + (o / 4) * c.tile;
          tma_load_2d(sb + a_bytes + (o % 4) * chunk + (o / 4) * c.tile * 128, &tm_t, fb, band + 64 * (o % 4), r0, pol);
        } else {
          const int q = o % (c.rt / 4), ch = o / (c.rt / 4);  // group-of-4-rows, chunk
          int r[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) r[t] = brow(it, 4 * q + t, c.rows, salt);
          tma_gather4(sb + a_bytes + ch * chunk + q * 512, &tm_g, fb, band + 64 * ch, r[0], r[1], r[2], r[3], pol);
        }
      }
    }
  } else if (warp < c.ntw + c.nlw && c.cpa) {
    // ------------------------------------------------ cp.async warps: rows [rt, rows), one 512-byte
    // row per warp instruction; the stage's completion is signalled asynchronously, so a warp moves
    // on to the next stage without waiting for its copies (in flight: up to S stages)
    const int lw = warp - c.ntw;
    const int chn = lane >> 3, unit = lane & 7;
    for (int it = 0; it < c.iters; ++it) {
      const int s = it % c.S;
      mbar_wait(smem_u32(&empty[s]), ((it / c.S) & 1) ^ 1);
      const uint32_t sb = s0 + s * stage_bytes + a_bytes;
      for (int j = c.rt + lw; j < c.rows; j += c.nlw) {
        const int row = brow(it, j, c.rows, salt);
        const uint16_t* src = Bp + static_cast<size_t>(row) * TCOLS + band + chn * 64 + unit * 8;
        const uint32_t dst = sb + chn * chunk + j * 128 + ((unit ^ (j & 7)) << 4);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp < c.ntw + c.nlw) {
    // ------------------------------------------------ LDG warps: rows [rt, rows) of every stage
    const int lw = warp - c.ntw;
    const int chn = lane >> 3, unit = lane & 7;  // 64-column chunk and 16-byte unit of this lane
    for (int it = 0; it < c.iters; ++it) {
      const int s = it % c.S;
      mbar_wait(smem_u32(&empty[s]), ((it / c.S) & 1) ^ 1);
      uint8_t* sb = smem + s * stage_bytes + a_bytes;
      constexpr int U = 8;
      for (int j0 = c.rt + lw * U; j0 < c.rows; j0 += U * c.nlw) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + u;
          if (j < c.rows) {
            const int row = brow(it, j, c.rows, salt);
            v[u] = __ldcg(reinterpret_cast<const uint4*>(Bp + static_cast<size_t>(row) * TCOLS + band + chn * 64 + unit * 8));
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + u;
          if (j < c.rows)
            *reinterpret_cast<uint4*>(sb + chn * chunk + j * 128 + ((unit ^ (j & 7)) << 4)) = v[u];
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&full[s]));
    }
  } else if (warp == W_MMA && lane == 0) {
    // ------------------------------------------------ consumer
    const uint32_t tb = tbase;
    if (c.mma) tc_cp_128x128b(tb + 508, smem_desc(smem_u32(meta), 16, 128, 0));  // metadata -> TMEM
    const uint32_t idesc = idesc_sp_f16(0, 128, 256);
    const int kbs = c.rows / 32;
    for (int it = 0; it < c.iters; ++it) {
      const int s = it % c.S;
      mbar_wait(smem_u32(&full[s]), (it / c.S) & 1);
      if (c.cpa) fence_proxy_async_smem();  // cp.async wrote through the generic proxy
      tc_fence_after();
      if (c.mma) {
        const uint32_t sb = s0 + s * stage_bytes;
        for (int kb = 0; kb < kbs; ++kb) {
          const uint64_t ad = smem_desc(sb + kb * 32, 16, 1024, 2);
          const uint64_t bd = smem_desc(sb + a_bytes + kb * 4096, chunk, 1024, 2);
          const uint32_t e = tb + 508 + (kb & 3);
          tc_mma_sp_f16(tb, ad, bd, idesc | (e & 1u), e & ~1u, (it | kb) ? 1u : 0u);
        }
        tc_commit(smem_u32(&empty[s]));
      } else {
        mbar_arrive(smem_u32(&empty[s]));
      }
    }
    if (c.mma) {
      tc_commit(smem_u32(&drain));  // wait for the last MMAs
      mbar_wait(smem_u32(&drain), 0);
    }
    cycles[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (c.mma && warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  // argv[1]: L2 promotion of the gather map (0 none, 1 64B, 2 128B, 3 256B); argv[2] = 1: gather cases only
  const int promo = argc > 1 ? atoi(argv[1]) : 3;
  const bool only_gather = argc > 2 && atoi(argv[2]) == 1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncFn enc = reinterpret_cast<EncFn>(fn);
  uint16_t *B, *A;
  cudaMalloc(&B, size_t(KROWS) * TCOLS * 2);
  cudaMemset(B, 0, size_t(KROWS) * TCOLS * 2);
  cudaMalloc(&A, size_t(8192) * 64 * 2);
  cudaMemset(A, 0, size_t(8192) * 64 * 2);
  CUtensorMap tg, tt, ta, ta64, tt64;
  cuuint64_t dims[2] = {cuuint64_t(TCOLS), cuuint64_t(KROWS)};
  cuuint64_t strides[1] = {cuuint64_t(TCOLS) * 2};
  cuuint32_t es[2] = {1, 1};
  cuuint32_t box1[2] = {64, 1}, box128[2] = {64, 128}, box64[2] = {64, 64}, box32[2] = {64, 32}, box8[2] = {64, 8};
  CUtensorMap tt32, tt8;
  enc(&tt32, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, B, dims, strides, box32, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tt8, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, B, dims, strides, box8, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tg, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, B, dims, strides, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, static_cast<CUtensorMapL2promotion>(promo), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("gather map L2 promotion %d\n", promo);
  enc(&tt, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, B, dims, strides, box128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tt64, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, B, dims, strides, box64, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t adims[2] = {64, 8192};
  cuuint64_t astr[1] = {128};
  cuuint32_t abox[2] = {64, 128};
  enc(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, A, adims, astr, abox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint32_t abox64[2] = {64, 64};
  enc(&ta64, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, A, adims, astr, abox64, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* d;
  cudaMalloc(&d, 8 * 1024);
  cudaFuncSetAttribute(feed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
  // {S, rows, rt, ntw, nlw, with_a, tile, mma, cpa}
  std::vector<Cfg> cases = {
      // gather4 with and without the 16 KB A box (what multicasting A across a 2-CTA cluster saves)
      {2, 128, 128, 11, 0, 0, 0, 1, 0}, {2, 128, 128, 15, 0, 0, 0, 1, 0}, {2, 128, 128, 15, 0, 1, 0, 1, 0},
      {2, 128, 128, 15, 0, 0, 0, 0, 0},
      // cp.async only, and cp.async beside gather4 (round 2b)
      {2, 128, 0, 1, 8, 1, 0, 0, 1}, {2, 128, 0, 1, 14, 1, 0, 0, 1}, {5, 64, 0, 1, 14, 1, 0, 0, 1},
      {3, 96, 0, 1, 14, 1, 0, 0, 1},
      {2, 128, 96, 8, 6, 1, 0, 0, 1}, {2, 128, 80, 8, 6, 1, 0, 0, 1}, {2, 128, 64, 8, 6, 1, 0, 0, 1},
      {2, 128, 96, 11, 4, 1, 0, 0, 1}, {2, 128, 64, 11, 4, 1, 0, 0, 1},
      {2, 128, 96, 8, 6, 1, 0, 1, 1}, {2, 128, 80, 8, 6, 1, 0, 1, 1}, {2, 128, 64, 8, 6, 1, 0, 1, 1},
      {2, 128, 128, 11, 0, 1, 0, 1, 0},
      // gather4 only (80 KB stages as the GPT-3 kernel: A + 64 KB B'; 40 KB at K' = 64)
      {2, 128, 128, 4, 0, 1, 0, 0}, {2, 128, 128, 8, 0, 1, 0, 0}, {2, 128, 128, 15, 0, 1, 0, 0},
      {5, 64, 64, 4, 0, 1, 0, 0}, {5, 64, 64, 8, 0, 1, 0, 0}, {5, 64, 64, 15, 0, 1, 0, 0},
      // LDG only; both paths at once
      {5, 64, 0, 1, 14, 1, 0, 0}, {2, 128, 96, 8, 6, 1, 0, 0}, {5, 64, 48, 8, 6, 1, 0, 0},
      // contiguous tile boxes: 128 / 64 / 32 / 8 rows per box (16 / 8 / 4 / 1 KB)
      {2, 128, 0, 1, 0, 1, 128, 0}, {2, 128, 0, 4, 0, 1, 128, 0}, {2, 128, 0, 4, 0, 1, 32, 0},
      {2, 128, 0, 8, 0, 1, 8, 0}, {2, 128, 0, 15, 0, 1, 8, 0},
      {5, 64, 0, 1, 0, 1, 64, 0}, {5, 64, 0, 4, 0, 1, 64, 0}, {5, 64, 0, 4, 0, 1, 32, 0}, {5, 64, 0, 8, 0, 1, 8, 0},
      // with the sparse MMA consuming every stage
      {2, 128, 128, 8, 0, 1, 0, 1}, {2, 128, 128, 15, 0, 1, 0, 1}, {5, 64, 64, 8, 0, 1, 0, 1},
      {5, 64, 64, 15, 0, 1, 0, 1}, {2, 128, 96, 8, 6, 1, 0, 1},
      {2, 128, 0, 4, 0, 1, 128, 1}, {5, 64, 0, 4, 0, 1, 64, 1}, {5, 64, 0, 4, 0, 1, 32, 1},
  };
  const int grids[2] = {sms, 16};
  for (int gi = 0; gi < 2; ++gi)
    for (Cfg c : cases) {
      if (gi == 1 && c.mma) continue;
      const int grid = grids[gi];
      const int a_bytes = c.with_a ? (c.rows == 128 ? 16384 : 8192) : 0;
      const int stage = a_bytes + c.rows * 512;
      if (c.S * stage > 220 * 1024 || c.S > 7 || c.ntw + c.nlw + 1 > 16) continue;
      if (gi == 1 && (c.tile == 8 || c.nlw > 0)) continue;
      if (only_gather && (c.tile || c.nlw || gi == 1)) continue;
      c.iters = 20;
      const CUtensorMap& tile_map = c.tile == 128 ? tt : c.tile == 64 ? tt64 : c.tile == 32 ? tt32 : tt8;
      feed_kernel<<<grid, 512, 226 * 1024>>>(tg, tile_map, ta, ta64, B, c, d);  // warm-up (L2 fill)
      c.iters = 2000;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      feed_kernel<<<grid, 512, 226 * 1024>>>(tg, tile_map, ta, ta64, B, c, d);
      cudaEventRecord(e1);
      cudaError_t err = cudaGetLastError();
      if (err == cudaSuccess) err = cudaDeviceSynchronize();
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<unsigned long long> cyc(grid);
      cudaMemcpy(cyc.data(), d, 8 * grid, cudaMemcpyDeviceToHost);
      double avgc = 0;
      for (int i = 0; i < grid; ++i) avgc += double(cyc[i]) / grid;
      const double bytes = double(c.iters) * stage;  // per CTA
      printf("grid=%3d S=%d rows=%3d gather_rows=%3d tma_warps=%2d %s_warps=%2d A=%d tile=%d mma=%d: "
             "%6.1f B/cycle/SM  %6.1f B/ns/SM  %6.2f TB/s chip  stage %6.0f cycles %s\n",
             grid, c.S, c.rows, c.tile ? 0 : c.rt, c.ntw, c.cpa ? "cpa" : "ldg", c.nlw, c.with_a, c.tile, c.mma, bytes / avgc,
             bytes * grid / (ms * 1e6) / grid, bytes * grid / (ms * 1e9), avgc / c.iters,
             err == cudaSuccess ? "" : cudaGetErrorString(err));
      if (err != cudaSuccess) return 1;
    }
  return 0;
}
