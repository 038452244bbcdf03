// densek_kernel.cuh — "dense-K" execution of the V:N:M SpMM for small V·M on B200.
//
// Why a second strategy: the gathered kernel (spmm_kernel.cuh) follows the paper's Fig 4 mapping
// (PAPER.md:207-209): per V-block it fetches only the 4 selected rows of B per group and runs a
// 2:4 product over K' = 4K/M. Each gathered B' byte feeds only V/2 useful FLOPs, and on B200 every
// 128-byte-row gather path (TMA gather4, cp.async, LDG) tops out near 33 B/cycle/SM
// (tools/microbench.cu, profiles/r01_microbench_gather_mma.txt), while the sparse tensor cores
// consume ~100 B/cycle of B'. For small V·M the gather feed, not the tensor core, binds.
//
// When M % 4 == 0 every V:N:M row is also a valid 2:4 row over the ORIGINAL K: a group of M
// columns holds 2 kept values, so each aligned 4-column subgroup holds at most 2 (DESIGN.md
// "dense-K"). This kernel therefore expands the compressed operand on the fly — values, m-indices
// and column_idx (the paper's column-loc resolves which subgroup and position each kept value
// occupies) — into the 2:4 form over K, and multiplies it with dense B tiles fetched by large TMA
// boxes (~60 B/cycle/SM). Tensor work is M/4 × the gathered kernel's, B is shared by every row of
// the tile (any V), and no B row gathers are needed. The cost model in venom_api.cu picks the
// faster strategy per problem; both produce the same fp32-accumulated product.
//
// Roles: warp 0 TMA producer (B tiles), warp 1 MMA (shared with the gathered kernel), warps 2-5
// epilogue (shared), warps 6-13 expanders (one row-half per thread per stage).
#pragma once
#include "spmm_kernel.cuh"

namespace venom {

template <int BN_, int STAGES_, int M_>
struct DenseKCfg {
  static constexpr int NB = 1;
  static constexpr int BN = BN_;
  static constexpr int STAGES = STAGES_;
  static constexpr int MM = M_;                 // V:N:M block width (compile-time for the expander)
  static constexpr int KT = 128;                // original K columns per stage (4 MMAs of K = 32)
  static constexpr int A_BYTES = 128 * 128;     // 128 rows × 64 expanded 2:4 values × 2 B (SW128)
  static constexpr int B_CHUNK = 128 * 128;     // 128 K-rows × 64 columns × 2 B
  static constexpr int B_BYTES = (BN / 64) * B_CHUNK;
  static constexpr int E_BYTES = 128 * 16;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES + E_BYTES;
  static constexpr int TX_BYTES = B_BYTES;
  static constexpr int ACC_COLS = BN;
  static constexpr int E_COLS = 8;
  static constexpr int ACC_BUFS = (2 * ACC_COLS + E_COLS <= 512) ? 2 : 1;
  static constexpr int E_COL = 512 - E_COLS;
  static constexpr int NGH = 64 / M_;           // groups touched by one row-half (64 columns)
  // compressed values of one stage: 128 rows × (128/M groups × 2) values, TMA-staged in a ring
  static constexpr int VE = 256 / M_;           // value elements per row per stage
  static constexpr int RAW_BYTES = 128 * VE * 2;
  static constexpr int AVAIL = 227 * 1024 - 1536 - STAGES * STAGE_BYTES;  // for the side rings
  static constexpr int RS_FIT = (AVAIL - 2 * 128 * 4 * (M_ == 4 ? 4 : (128 / M_ + (128 / M_ + 7) / 8))) / RAW_BYTES;
  static constexpr int RS = RS_FIT < 4 ? RS_FIT : 4;
  // column_idx words and metadata nibbles of one stage, staged by loader warps (global loads are
  // kept out of the expander warps: their proxy fence would wait for outstanding loads)
  static constexpr int GS = 128 / M_;           // groups per row per stage
  static constexpr int NMW = (GS + 7) / 8;      // metadata words per row per stage
  static constexpr int CW = (M_ == 4) ? 0 : GS; // column_idx words per row per stage
  static constexpr int PITCH = 4 * (CW + NMW);  // side-ring bytes per row
  static constexpr int SIDE_BYTES = 128 * PITCH;
  static constexpr int SS = (AVAIL - RS * RAW_BYTES) / SIDE_BYTES < 4
                                ? (AVAIL - RS * RAW_BYTES) / SIDE_BYTES : 4;  // side-ring slots
  static constexpr int W_MMA = 1, W_EPI = 2, W_EXP = 6, N_EXP = 8, W_RAW = W_EXP + N_EXP;
  static constexpr int W_LD = W_RAW + 1, N_LD = 4;
  static constexpr int NUM_THREADS = 32 * (W_LD + N_LD);
  static constexpr int SMEM_BYTES =
      1024 + STAGES * STAGE_BYTES + RS * RAW_BYTES + SS * SIDE_BYTES + 512;
  static_assert(M_ % 4 == 0 && M_ <= 32, "dense-K: M in {4, 8, 16, 32}");
  static_assert(ACC_BUFS * ACC_COLS + E_COLS <= 512, "TMEM budget");
  static_assert(SMEM_BYTES <= 227 * 1024, "smem budget");
  static_assert(RS >= 2 && SS >= 2, "ring depth");
};

// Column_idx words and metadata nibbles of one row-half (NGH groups), read from the side ring.
template <int NGH>
struct ExpRaw {
  uint32_t cidx[NGH];
  uint32_t nib[(NGH + 7) / 8];
};

// Loader: the column_idx words (GS) and metadata nibbles (GS, packed 8 per word) of one row for
// one k-stage, from global memory. Groups past G read as the all-zero pattern 0x4.
template <class Cfg>
__device__ __forceinline__ void side_fetch(const SpmmParams& p, int64_t row, int ks,
                                           uint32_t (&cw)[Cfg::CW > 0 ? Cfg::CW : 1],
                                           uint32_t (&mw)[Cfg::NMW]) {
  constexpr int GS = Cfg::GS, CW = Cfg::CW, NMW = Cfg::NMW;
  const int64_t g0 = static_cast<int64_t>(ks) * GS;
#pragma unroll
  for (int q = 0; q < (CW > 0 ? CW : 1); ++q) cw[q] = 0x03020100u;
#pragma unroll
  for (int q = 0; q < NMW; ++q) mw[q] = 0x44444444u;
  if (row >= p.R) return;
  if constexpr (CW > 0) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(p.column_idx) + (row / p.V) * p.G + g0;
    if (g0 + GS <= p.G) {
#pragma unroll
      for (int q = 0; q < CW / 4; ++q) {  // (rb·G + g0) % 4 == 0: G % 4 == 0 and GS >= 4
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(src) + q);
        cw[4 * q] = v.x; cw[4 * q + 1] = v.y; cw[4 * q + 2] = v.z; cw[4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < CW; ++q)
        if (g0 + q < p.G) cw[q] = __ldg(src + q);
    }
  }
  const uint8_t* mb = p.metadata + row * p.meta_row + (g0 >> 1);
  constexpr int NBY = GS / 2;  // metadata bytes per row per stage (2, 4, 8 or 16)
  uint32_t w[NMW];
#pragma unroll
  for (int q = 0; q < NMW; ++q) w[q] = 0u;
  if (g0 + GS <= p.G && (reinterpret_cast<uintptr_t>(mb) % NBY) == 0) {
    if constexpr (NBY == 16) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(mb));
      w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    } else if constexpr (NBY == 8) {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(mb));
      w[0] = v.x; w[1] = v.y;
    } else if constexpr (NBY == 4) {
      w[0] = __ldg(reinterpret_cast<const uint32_t*>(mb));
    } else {
      w[0] = __ldg(reinterpret_cast<const uint16_t*>(mb));
    }
  } else {
#pragma unroll
    for (int q = 0; q < NBY; ++q)
      if (g0 + 2 * q < p.G) w[q >> 2] |= static_cast<uint32_t>(__ldg(mb + q)) << (8 * (q & 3));
  }
#pragma unroll
  for (int gi = 0; gi < GS; ++gi) {
    if (g0 + gi >= p.G) {
      w[gi >> 3] &= ~(0xFu << (4 * (gi & 7)));
      w[gi >> 3] |= 0x4u << (4 * (gi & 7));
    }
  }
#pragma unroll
  for (int q = 0; q < NMW; ++q) mw[q] = w[q];
}

// Expand one row-half (64 original columns = 16 subgroups of 4 = 2 MMAs of K = 32) into 2:4 form:
// 16 value words (one per subgroup: two 16-bit values) and 2 metadata words (8 nibbles each).
// Per group: the two kept values sit at block columns c0 < c1 (column_idx through the m-indices);
// subgroup s = c >> 2, position i = c & 3. A subgroup holding both gets (v0, v1) at (i0, i1); one
// holding a single value v at i gets (v, 0) at (0, 1) if i == 0 else (0, v) at (0, i); an empty
// subgroup gets zeros at (0, 1). M = 4 is plain 2:4: the group IS the subgroup (pass-through).
template <class Cfg>
__device__ __forceinline__ void exp_build(const ExpRaw<Cfg::NGH>& raw, const uint32_t (&val)[Cfg::NGH],
                                          uint32_t (&vw)[16], uint32_t (&mw)[2]) {
  constexpr int M = Cfg::MM, NGH = Cfg::NGH, SUB = M / 4;  // subgroups per group
  if constexpr (M == 4) {
#pragma unroll
    for (int j = 0; j < 16; ++j) vw[j] = val[j];
    mw[0] = raw.nib[0];
    mw[1] = raw.nib[1];
    return;
  }
  mw[0] = 0u;
  mw[1] = 0u;
#pragma unroll
  for (int gi = 0; gi < NGH; ++gi) {
    const uint32_t n4 = (raw.nib[gi >> 3] >> (4 * (gi & 7))) & 0xFu;
    const uint32_t cw = raw.cidx[gi];
    const uint32_t c0 = __byte_perm(cw, 0u, 0x4440u | (n4 & 3u)) ;          // byte p0 of cw
    const uint32_t c1 = __byte_perm(cw, 0u, 0x4440u | (n4 >> 2));           // byte p1 of cw
    const uint32_t v = val[gi];
    const uint32_t s0 = c0 >> 2, s1 = c1 >> 2, i0 = c0 & 3u, i1 = c1 & 3u;
    const uint32_t one0w = i0 ? (v << 16) : (v & 0xFFFFu);
    const uint32_t one0n = i0 ? (i0 << 2) : 0x4u;
    const uint32_t one1w = i1 ? (v & 0xFFFF0000u) : (v >> 16);
    const uint32_t one1n = i1 ? (i1 << 2) : 0x4u;
    const bool same = (s0 == s1);
    const uint32_t w0 = same ? v : one0w;
    const uint32_t n0 = same ? (i0 | (i1 << 2)) : one0n;
#pragma unroll
    for (int u = 0; u < SUB; ++u) {
      const int j = gi * SUB + u;  // subgroup index within the half
      const uint32_t w = (s0 == uint32_t(u)) ? w0 : ((s1 == uint32_t(u)) ? one1w : 0u);
      const uint32_t n = (s0 == uint32_t(u)) ? n0 : ((s1 == uint32_t(u)) ? one1n : 0x4u);
      vw[j] = w;
      mw[j >> 3] |= n << (4 * (j & 7));
    }
  }
}

template <class Cfg, bool kBF16>
__global__ void __launch_bounds__(Cfg::NUM_THREADS, 1)
    vnm_spmm_densek_kernel(const __grid_constant__ CUtensorMap tm_b,
                           const __grid_constant__ CUtensorMap tm_v, const SpmmParams p) {
  using namespace ptx;
  constexpr int STAGES = Cfg::STAGES, BN = Cfg::BN;

  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) &
                                             ~uintptr_t(1023));
  constexpr int RS = Cfg::RS;
  uint8_t* raw_smem = smem + STAGES * Cfg::STAGE_BYTES;  // RS slots of TMA-staged values
  uint8_t* side_smem = raw_smem + RS * Cfg::RAW_BYTES;   // SS slots of column_idx + metadata
  uint64_t* bars = reinterpret_cast<uint64_t*>(side_smem + Cfg::SS * Cfg::SIDE_BYTES);
  const uint32_t full0 = smem_u32(bars);
  const uint32_t empty0 = full0 + 8 * STAGES;
  const uint32_t accf0 = empty0 + 8 * STAGES;
  const uint32_t acce0 = accf0 + 16;
  const uint32_t rfull0 = acce0 + 16;
  const uint32_t rempty0 = rfull0 + 8 * RS;
  const uint32_t sfull0 = rempty0 + 8 * RS;
  const uint32_t sempty0 = sfull0 + 8 * Cfg::SS;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4 + 2 * RS + 2 * Cfg::SS);
  const uint32_t smem0 = smem_u32(smem);
  const uint32_t raw0 = smem_u32(raw_smem);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1 + Cfg::N_EXP);  // producer expect_tx + expander warps
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(accf0 + 8 * b, 1);
      mbar_init(acce0 + 8 * b, 4);
    }
    for (int s = 0; s < RS; ++s) {
      mbar_init(rfull0 + 8 * s, 1);               // producer expect_tx
      mbar_init(rempty0 + 8 * s, Cfg::N_EXP);     // expander warps done reading
    }
    for (int s = 0; s < Cfg::SS; ++s) {
      mbar_init(sfull0 + 8 * s, Cfg::N_LD);       // loader warps stored the slot
      mbar_init(sempty0 + 8 * s, Cfg::N_EXP);     // expander warps done reading
    }
    fence_mbar_init();
    prefetch_tmap(&tm_b);
    prefetch_tmap(&tm_v);
  }
  if (warp == Cfg::W_MMA) tmem_alloc<512>(smem_u32(tmem_base_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  const int my_tiles =
      (static_cast<int>(blockIdx.x) < p.num_tiles)
          ? (p.num_tiles - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                static_cast<int>(gridDim.x)
          : 0;
  const int total = my_tiles * p.num_ks;

  if (warp == 0) {
    // ======================= producer: dense B tiles (128 K-rows × 64 columns per box) ==========
    const uint64_t pol_b = policy_evict_last();
    for (int it = 0; it < total; ++it) {
      const int stage = it % STAGES;
      int m_tile, n_tile;
      tile_coords(p, it / p.num_ks, m_tile, n_tile);
      const int ks = it % p.num_ks;
      mbar_wait(empty0 + 8 * stage, ((it / STAGES) & 1) ^ 1);
      if (lane == 0) {
        VENOM_TRACE_EVENT(0, it);
        const uint32_t bdst = smem0 + stage * Cfg::STAGE_BYTES + Cfg::A_BYTES;
        mbar_arrive_expect_tx(full0 + 8 * stage, Cfg::TX_BYTES);
#pragma unroll
        for (int c = 0; c < BN / 64; ++c)
          tma_load_2d(bdst + c * Cfg::B_CHUNK, &tm_b, full0 + 8 * stage, n_tile * BN + 64 * c,
                      ks * Cfg::KT, pol_b);
      }
      __syncwarp();
    }
  } else if (warp == Cfg::W_MMA) {
    mma_role<Cfg, kBF16>(p, my_tiles, tmem_base, smem0, full0, empty0, accf0, acce0, lane);
  } else if (warp >= Cfg::W_EPI && warp < Cfg::W_EPI + 4) {
    epilogue_role<Cfg, kBF16>(p, my_tiles, tmem_base, accf0, acce0, warp, lane);
  } else if (warp == Cfg::W_RAW) {
    // ======================= raw ring: the stage's compressed values (128 rows × VE) ============
    // runs up to RS stages ahead of the expanders, independently of the B ring
    const uint64_t pol_v = policy_evict_first();
    for (int j = 0; j < total; ++j) {
      const int slot = j % RS;
      int m_tile, n_tile;
      tile_coords(p, j / p.num_ks, m_tile, n_tile);
      mbar_wait(rempty0 + 8 * slot, ((j / RS) & 1) ^ 1);
      if (lane == 0) {
        mbar_arrive_expect_tx(rfull0 + 8 * slot, Cfg::RAW_BYTES);
        tma_load_2d(raw0 + slot * Cfg::RAW_BYTES, &tm_v, rfull0 + 8 * slot, (j % p.num_ks) * Cfg::VE,
                    m_tile * 128, pol_v);
      }
      __syncwarp();
    }
  } else if (warp >= Cfg::W_LD) {
    // ======================= loaders: column_idx + metadata of each stage -> side ring ==========
    const int r = 32 * (warp - Cfg::W_LD) + lane;  // tile row
    constexpr int PL = 3;                          // register prefetch depth (k-stages)
    constexpr int CWN = Cfg::CW > 0 ? Cfg::CW : 1;
    uint32_t cw[PL][CWN], mw[PL][Cfg::NMW];
    auto fetch = [&](int it, uint32_t (&c)[CWN], uint32_t (&m)[Cfg::NMW]) {
      if (it >= total) return;
      int m_tile, n_tile;
      tile_coords(p, it / p.num_ks, m_tile, n_tile);
      side_fetch<Cfg>(p, static_cast<int64_t>(m_tile) * 128 + r, it % p.num_ks, c, m);
    };
#pragma unroll
    for (int j = 0; j < PL; ++j) fetch(j, cw[j], mw[j]);
    for (int it0 = 0; it0 < total; it0 += PL) {
#pragma unroll
      for (int j = 0; j < PL; ++j) {
        const int it = it0 + j;
        if (it < total) {
          const int slot = it % Cfg::SS;
          mbar_wait(sempty0 + 8 * slot, ((it / Cfg::SS) & 1) ^ 1);
          uint32_t* dst = reinterpret_cast<uint32_t*>(side_smem + slot * Cfg::SIDE_BYTES + r * Cfg::PITCH);
#pragma unroll
          for (int q = 0; q < Cfg::CW; ++q) dst[q] = cw[j][q];
#pragma unroll
          for (int q = 0; q < Cfg::NMW; ++q) dst[Cfg::CW + q] = mw[j][q];
          __syncwarp();
          if (lane == 0) mbar_arrive(sfull0 + 8 * slot);
          fetch(it + PL, cw[j], mw[j]);
        }
      }
    }
  } else {
    // ======================= expanders: V:N:M -> 2:4 over the original K, in SMEM ===============
    const int e = warp - Cfg::W_EXP;
    const int r = 32 * (e & 3) + lane;  // tile row
    const int h = e >> 2;               // which 64-column half of the stage
    const int L0 = (r & 7) + 16 * (r >> 4);
    const int m1 = (r >> 3) & 1;
    constexpr int NGH = Cfg::NGH;
    for (int it = 0; it < total; ++it) {
      const int stage = it % STAGES;
      const int slot = it % RS;
      const int sslot = it % Cfg::SS;
      // this row-half's compressed values (TMA-staged) and column_idx / metadata (loader-staged)
      mbar_wait(rfull0 + 8 * slot, (it / RS) & 1);
      mbar_wait(sfull0 + 8 * sslot, (it / Cfg::SS) & 1);
      if (e == 0 && lane == 0) VENOM_TRACE_EVENT(3, it);
      uint32_t val[NGH];
      const uint8_t* vsrc = raw_smem + slot * Cfg::RAW_BYTES + r * (Cfg::VE * 2) + h * (NGH * 4);
      if constexpr (NGH >= 4) {
#pragma unroll
        for (int q = 0; q < NGH / 4; ++q) {
          const uint4 v = *reinterpret_cast<const uint4*>(vsrc + 16 * q);
          val[4 * q] = v.x; val[4 * q + 1] = v.y; val[4 * q + 2] = v.z; val[4 * q + 3] = v.w;
        }
      } else {
        const uint2 v = *reinterpret_cast<const uint2*>(vsrc);
        val[0] = v.x;
        val[1] = v.y;
      }
      ExpRaw<NGH> raw;
      const uint32_t* side = reinterpret_cast<const uint32_t*>(side_smem + sslot * Cfg::SIDE_BYTES + r * Cfg::PITCH);
#pragma unroll
      for (int gi = 0; gi < NGH; ++gi) raw.cidx[gi] = (Cfg::CW > 0) ? side[h * NGH + gi] : 0x03020100u;
      {
        // nibbles of groups h·NGH .. h·NGH + NGH - 1 of the stage
        constexpr int NW = (NGH + 7) / 8;
        if constexpr (NGH >= 8) {
#pragma unroll
          for (int q = 0; q < NW; ++q) raw.nib[q] = side[Cfg::CW + h * NW + q];
        } else {
          const uint32_t word = side[Cfg::CW];  // GS <= 8: one word holds the whole stage
          raw.nib[0] = word >> (4 * NGH * h);
        }
      }
      uint32_t vw[16], mw[2];
      exp_build<Cfg>(raw, val, vw, mw);
      mbar_wait(empty0 + 8 * stage, ((it / STAGES) & 1) ^ 1);
      if (e == 0 && lane == 0) VENOM_TRACE_EVENT(4, it);
      uint8_t* sbase = smem + stage * Cfg::STAGE_BYTES;
      // A': row r, 16-byte chunks 4h..4h+3, 128B-swizzled (chunk ^ (row & 7))
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int chunk = 4 * h + c;
        *reinterpret_cast<uint4*>(sbase + r * 128 + 16 * (chunk ^ (r & 7))) =
            make_uint4(vw[4 * c], vw[4 * c + 1], vw[4 * c + 2], vw[4 * c + 3]);
      }
      // metadata in the tensor-core lane layout: row r's word for MMA kb splits into its
      // K-halves, lanes L0 (k1 = 0) and L0 + 8 (k1 = 1), half-word m1
      uint8_t* e_smem = sbase + Cfg::A_BYTES + Cfg::B_BYTES;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int kb = 2 * h + u;
        *reinterpret_cast<uint16_t*>(e_smem + 16 * L0 + 4 * kb + 2 * m1) =
            static_cast<uint16_t>(mw[u] & 0xFFFFu);
        *reinterpret_cast<uint16_t*>(e_smem + 16 * (L0 + 8) + 4 * kb + 2 * m1) =
            static_cast<uint16_t>(mw[u] >> 16);
      }
      fence_proxy_async_smem();
      __syncwarp();
      // Release the raw and side slots only now: the stores above consume every value loaded from
      // them, so those shared loads have returned. (An arrive placed right after the loads can
      // overtake them — ptxas may schedule it first — and let the next TMA overwrite the slot
      // under the reads: observed as data from k-stage it + RS.)
      if (lane == 0) {
        mbar_arrive(rempty0 + 8 * slot);
        mbar_arrive(sempty0 + 8 * sslot);
        mbar_arrive(full0 + 8 * stage);
      }
      if (e == 0 && lane == 0) VENOM_TRACE_EVENT(5, it);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == Cfg::W_MMA) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace venom
