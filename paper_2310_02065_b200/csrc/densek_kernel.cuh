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
// "dense-K"). This kernel expands the compressed operand on the fly — values, m-indices and
// column_idx (the paper's column-loc decides which subgroup and position each kept value occupies)
// — into the 2:4 form over K and multiplies it with dense B tiles fetched by large TMA boxes. B is
// shared by every row of the tile (any V), so CTA pairs (cta_group::2, 256-row tiles) split B
// between their shared memories. Tensor work is M/4 × the gathered kernel's.
//
// Measured constraints that shape it (tools/microbench_mma.cu): while the tensor core streams
// operands, generic st.shared crawls (~6-14 B/cycle/SM) and every fence.proxy.async costs ~650
// cycles, serialised across warps. So the expanded operand never touches shared memory: the
// expander warps write A' and its metadata straight into TMEM (tcgen05.st) and the sparse MMA
// reads A from TMEM; only B (TMA) and the compressed values (TMA ring) use shared memory.
//
// Roles (16 warps): 0 B producer (TMA), 1 MMA (pair leader), 2 values ring (TMA), 3 idle,
// 4-7 epilogue (shared with the gathered kernel), 8-15 expanders (row-half per thread).
#pragma once
#include "spmm_kernel.cuh"

namespace venom {

template <int BN_, int STAGES_, int M_, int CG_ = 1>
struct DenseKCfg {
  static constexpr int NB = 1;
  static constexpr bool M64 = false;            // (shares spmm_kernel.cuh's epilogue)
  static constexpr int CG = CG_;                // 2: CTA pair (cta_group::2), M = 256 per MMA
  static constexpr int BN = BN_;
  static constexpr int STAGES = STAGES_;
  static constexpr int MM = M_;                 // V:N:M block width (compile-time for the expander)
  static constexpr int KT = 128;                // original K columns per stage (4 MMAs of K = 32)
  static constexpr int B_CHUNK = 128 * 128;     // 128 K-rows × 64 columns × 2 B
  static constexpr int BNH = BN / CG_;          // B columns held by one CTA (pair: half of N)
  static constexpr int B_BYTES = (BNH / 64) * B_CHUNK;
  static constexpr int STAGE_BYTES = B_BYTES;
  static constexpr int TX_BYTES = B_BYTES;      // per CTA; the pair leader expects CG × this
  // TMEM columns: accumulators, then per stage the expanded A (32 columns: 128 rows × 64 values)
  // and its metadata (4 columns, one per K = 32 MMA)
  static constexpr int ACC_COLS = BN;
  static constexpr int ACC_BUFS = (2 * BN + STAGES_ * 36 <= 512) ? 2 : 1;
  static constexpr int A_COL = ACC_BUFS * BN;
  static constexpr int E_COL = A_COL + 32 * STAGES_;
  static constexpr int NGH = 64 / M_;           // groups touched by one row-half (64 columns)
  // compressed values of one stage: 128 rows × (128/M groups × 2) values, TMA-staged in a ring
  static constexpr int VE = 256 / M_;           // value elements per row per stage
  static constexpr int RAW_BYTES = 128 * VE * 2;
  static constexpr int RS = 4;
  // expanders load the values straight from global memory (true) or from the TMA values ring
  static constexpr bool DIRECT = true;
  static constexpr int W_MMA = 1, W_RAW = 2, W_EPI = 4, W_EXP = 8, N_EXP = 8, EPI_WARPS = 4;
  static constexpr int EPI_SLOT = 2048, EPI_BUFS = 1;  // (the shared epilogue's TMA-store path is unused here)
  static constexpr int NUM_THREADS = 32 * (W_EXP + N_EXP);
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + RS * RAW_BYTES + 512;
  static_assert(M_ % 4 == 0 && M_ <= 32, "dense-K: M in {4, 8, 16, 32}");
  static_assert(BNH % 64 == 0, "B half must be whole 64-column chunks");
  static_assert(E_COL + 4 * STAGES_ <= 512, "TMEM budget");
  static_assert(SMEM_BYTES <= 227 * 1024, "smem budget");
  static_assert(W_EPI % 4 == 0 && W_EXP % 4 == 0, "TMEM lane quarters follow warp % 4");
};

// Column_idx words and metadata nibbles of one row-half (NGH groups).
template <int NGH>
struct ExpRaw {
  uint32_t cidx[NGH];
  uint32_t nib[(NGH + 7) / 8];
  uint32_t val[NGH];  // the two kept values of each group (direct-load path)
};

// Global loads for one row-half of one k-stage: the block's column_idx words (broadcast across
// the block's rows) and the row's metadata nibbles. Groups past G read as the zero pattern 0x4.
template <class Cfg, bool kDirectValues>
__device__ __forceinline__ void exp_fetch(const SpmmParams& p, int64_t row, int ks, int h,
                                          ExpRaw<Cfg::NGH>& raw) {
  constexpr int M = Cfg::MM, NGH = Cfg::NGH, NW = (NGH + 7) / 8;
  const int64_t g0 = (static_cast<int64_t>(ks) * 128 + 64 * h) / M;
#pragma unroll
  for (int gi = 0; gi < NGH; ++gi) raw.cidx[gi] = 0x03020100u;
#pragma unroll
  for (int w = 0; w < NW; ++w) raw.nib[w] = 0x44444444u;
#pragma unroll
  for (int gi = 0; gi < NGH; ++gi) raw.val[gi] = 0u;
  if (row >= p.R) return;
  if (kDirectValues) {
    const uint32_t* vp = reinterpret_cast<const uint32_t*>(p.values) + row * p.G + g0;
    if (g0 + NGH <= p.G && (reinterpret_cast<uintptr_t>(vp) % (4 * (NGH >= 4 ? 4 : NGH))) == 0) {
      if constexpr (NGH >= 4) {
#pragma unroll
        for (int q = 0; q < NGH / 4; ++q) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(vp) + q);
          raw.val[4 * q] = v.x; raw.val[4 * q + 1] = v.y; raw.val[4 * q + 2] = v.z; raw.val[4 * q + 3] = v.w;
        }
      } else {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(vp));
        raw.val[0] = v.x;
        raw.val[1] = v.y;
      }
    } else {
#pragma unroll
      for (int gi = 0; gi < NGH; ++gi)
        if (g0 + gi < p.G) raw.val[gi] = __ldg(vp + gi);
    }
  }
  if constexpr (M != 4) {
    const uint32_t* cw = reinterpret_cast<const uint32_t*>(p.column_idx) + (row / p.V) * p.G + g0;
    if (g0 + NGH <= p.G) {
      if constexpr (NGH >= 4) {
#pragma unroll
        for (int q = 0; q < NGH / 4; ++q) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(cw) + q);  // (rb·G + g0) % 4 == 0
          raw.cidx[4 * q] = v.x; raw.cidx[4 * q + 1] = v.y;
          raw.cidx[4 * q + 2] = v.z; raw.cidx[4 * q + 3] = v.w;
        }
      } else {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(cw));  // NGH == 2, g0 even
        raw.cidx[0] = v.x;
        raw.cidx[1] = v.y;
      }
    } else {
#pragma unroll
      for (int gi = 0; gi < NGH; ++gi)
        if (g0 + gi < p.G) raw.cidx[gi] = __ldg(cw + gi);
    }
  }
  // metadata: NGH/2 bytes starting at byte g0/2 of the row (g0 is even)
  const uint8_t* mb = p.metadata + row * p.meta_row + (g0 >> 1);
  constexpr int NBY = NGH / 2;
  uint32_t w[NW];
#pragma unroll
  for (int q = 0; q < NW; ++q) w[q] = 0u;
  if (g0 + NGH <= p.G && (reinterpret_cast<uintptr_t>(mb) % NBY) == 0) {
    if constexpr (NBY == 8) {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(mb));
      w[0] = v.x;
      w[1] = v.y;
    } else if constexpr (NBY == 4) {
      w[0] = __ldg(reinterpret_cast<const uint32_t*>(mb));
    } else if constexpr (NBY == 2) {
      w[0] = __ldg(reinterpret_cast<const uint16_t*>(mb));
    } else {
      w[0] = __ldg(mb);
    }
  } else {
#pragma unroll
    for (int q = 0; q < NBY; ++q)
      if (g0 + 2 * q < p.G) w[q >> 2] |= static_cast<uint32_t>(__ldg(mb + q)) << (8 * (q & 3));
  }
#pragma unroll
  for (int gi = 0; gi < NGH; ++gi) {
    if (g0 + gi >= p.G) {
      w[gi >> 3] &= ~(0xFu << (4 * (gi & 7)));
      w[gi >> 3] |= 0x4u << (4 * (gi & 7));
    }
  }
#pragma unroll
  for (int q = 0; q < NW; ++q) raw.nib[q] = w[q];
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
    const uint32_t c0 = __byte_perm(cw, 0u, 0x4440u | (n4 & 3u));  // byte p0 of cw
    const uint32_t c1 = __byte_perm(cw, 0u, 0x4440u | (n4 >> 2));  // byte p1 of cw
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
  constexpr int STAGES = Cfg::STAGES, BN = Cfg::BN, CG = Cfg::CG, RS = Cfg::RS;

  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* raw_smem = smem + STAGES * Cfg::STAGE_BYTES;  // RS slots of TMA-staged values
  uint64_t* bars = reinterpret_cast<uint64_t*>(raw_smem + RS * Cfg::RAW_BYTES);
  const uint32_t full0 = smem_u32(bars);
  const uint32_t empty0 = full0 + 8 * STAGES;
  const uint32_t accf0 = empty0 + 8 * STAGES;
  const uint32_t acce0 = accf0 + 16;
  const uint32_t rfull0 = acce0 + 16;
  const uint32_t rempty0 = rfull0 + 8 * RS;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4 + 2 * RS);
  const uint32_t smem0 = smem_u32(smem);
  const uint32_t raw0 = smem_u32(raw_smem);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0u;  // position in the CTA pair

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      // leader's expect_tx + the expander warps of every CTA of the pair (only the leader's counts)
      mbar_init(full0 + 8 * s, 1 + CG * Cfg::N_EXP);
      mbar_init(empty0 + 8 * s, 1);  // (multicast) MMA commit: B smem and A'/E TMEM slot free
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(accf0 + 8 * b, 1);
      mbar_init(acce0 + 8 * b, 4 * CG);  // epilogue warps of every CTA of the pair
    }
    for (int s = 0; s < RS; ++s) {
      mbar_init(rfull0 + 8 * s, 1);             // values TMA (expect_tx)
      mbar_init(rempty0 + 8 * s, Cfg::N_EXP);   // expander warps done reading
    }
    fence_mbar_init();
    prefetch_tmap(&tm_b);
    prefetch_tmap(&tm_v);
  }
  if (warp == Cfg::W_MMA) {
    if constexpr (CG == 2) tmem_alloc_2sm<512>(smem_u32(tmem_base_slot));
    else tmem_alloc<512>(smem_u32(tmem_base_slot));
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();  // peer barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  const int my_tiles = my_tile_count<CG>(p);
  const int total = my_tiles * p.num_ks;
  const int row_off = 128 * static_cast<int>(rank);  // this CTA's rows within the pair tile

  if (warp == 0) {
    // ======================= producer: dense B tiles (128 K-rows × 64 columns per box) ==========
    const uint64_t pol_b = policy_evict_last();
    for (int it = 0; it < total; ++it) {
      const int stage = it % STAGES;
      int m_tile, n_tile;
      tile_coords<CG>(p, it / p.num_ks, m_tile, n_tile);
      const int ks = it % p.num_ks;
      mbar_wait(empty0 + 8 * stage, ((it / STAGES) & 1) ^ 1);
      if (lane == 0) {
        VENOM_TRACE_EVENT(0, it);
        const uint32_t bdst = smem0 + stage * Cfg::STAGE_BYTES;
        const int col0 = n_tile * BN + static_cast<int>(rank) * Cfg::BNH;
        if constexpr (CG == 2) {
          // both CTAs load their half of B; the bytes are counted on the leader's barrier
          const uint32_t lbar = mapa_shared(full0 + 8 * stage, 0);
          if (rank == 0) mbar_arrive_expect_tx(full0 + 8 * stage, CG * Cfg::TX_BYTES);
#pragma unroll
          for (int c = 0; c < Cfg::BNH / 64; ++c)
            tma_load_2d_2sm(bdst + c * Cfg::B_CHUNK, &tm_b, lbar, col0 + 64 * c, ks * Cfg::KT, pol_b);
        } else {
          mbar_arrive_expect_tx(full0 + 8 * stage, Cfg::TX_BYTES);
#pragma unroll
          for (int c = 0; c < BN / 64; ++c)
            tma_load_2d(bdst + c * Cfg::B_CHUNK, &tm_b, full0 + 8 * stage, col0 + 64 * c,
                        ks * Cfg::KT, pol_b);
        }
      }
      __syncwarp();
    }
  } else if (warp == Cfg::W_MMA) {
    // ======================= MMA issuer (pair leader): A' and metadata from TMEM ==============
    if (rank == 0) {
      constexpr uint32_t idesc = idesc_sp_f16(kBF16 ? 1u : 0u, 128 * CG, BN);
      for (int tl = 0; tl < my_tiles; ++tl) {
        const int ab = tl % Cfg::ACC_BUFS;
        mbar_wait(acce0 + 8 * ab, ((tl / Cfg::ACC_BUFS) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tile = tmem_base + ab * Cfg::ACC_COLS;
        for (int ks = 0; ks < p.num_ks; ++ks) {
          const int it = tl * p.num_ks + ks;
          const int stage = it % STAGES;
          mbar_wait(full0 + 8 * stage, (it / STAGES) & 1);
          tc_fence_after();
          if (lane == 0) {
            VENOM_TRACE_EVENT(1, it);
            const uint32_t sbase = smem0 + stage * Cfg::STAGE_BYTES;
            const uint32_t a_t = tmem_base + Cfg::A_COL + 32 * stage;
            const uint32_t e_t = tmem_base + Cfg::E_COL + 4 * stage;
#pragma unroll
            for (int kb = 0; kb < 4; ++kb) {
              const uint32_t e_addr = e_t + kb;
              const uint32_t id2 = e_addr & 1u;  // odd metadata column -> selector id2
              // B: MN-major SW128, 64-column chunks B_CHUNK apart, 8 K-rows 1024 B apart
              const uint64_t bdesc = smem_desc(sbase + kb * 4096, Cfg::B_CHUNK, 1024, 2);
              if constexpr (CG == 2)
                tc_mma_sp_f16_ts_2sm(d_tile, a_t + 8 * kb, bdesc, idesc | id2, e_addr & ~1u,
                                     (ks | kb) != 0 ? 1u : 0u);
              else
                tc_mma_sp_f16_ts(d_tile, a_t + 8 * kb, bdesc, idesc | id2, e_addr & ~1u,
                                 (ks | kb) != 0 ? 1u : 0u);
            }
            if constexpr (CG == 2) {
              tc_commit_2sm_mc(empty0 + 8 * stage, 0x3);
              if (ks == p.num_ks - 1) tc_commit_2sm_mc(accf0 + 8 * ab, 0x3);
            } else {
              tc_commit(empty0 + 8 * stage);
              if (ks == p.num_ks - 1) tc_commit(accf0 + 8 * ab);
            }
            VENOM_TRACE_EVENT(2, it);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == Cfg::W_RAW && !Cfg::DIRECT) {
    // ======================= values ring: the stage's compressed values (128 rows × VE) =========
    const uint64_t pol_v = policy_evict_first();
    for (int j = 0; j < total; ++j) {
      const int slot = j % RS;
      int m_tile, n_tile;
      tile_coords<CG>(p, j / p.num_ks, m_tile, n_tile);
      mbar_wait(rempty0 + 8 * slot, ((j / RS) & 1) ^ 1);
      if (lane == 0) {
        mbar_arrive_expect_tx(rfull0 + 8 * slot, Cfg::RAW_BYTES);
        tma_load_2d(raw0 + slot * Cfg::RAW_BYTES, &tm_v, rfull0 + 8 * slot, (j % p.num_ks) * Cfg::VE,
                    m_tile * (128 * CG) + row_off, pol_v);
      }
      __syncwarp();
    }
  } else if (warp >= Cfg::W_EPI && warp < Cfg::W_EPI + 4) {
    epilogue_role<Cfg, kBF16, CG>(p, my_tiles, tmem_base, accf0, acce0, warp, lane);
  } else if (warp >= Cfg::W_EXP) {  // (warps 2-3 idle with the direct values path)
    // ======================= expanders: V:N:M -> 2:4 over the original K, into TMEM =============
    const int e = warp - Cfg::W_EXP;
    const int q = e & 3;                // TMEM lane quarter (== warp % 4)
    const int h = e >> 2;               // which 64-column half of the stage
    const int r = 32 * q + lane;        // tile row == TMEM lane
    constexpr int NGH = Cfg::NGH;
    // metadata lane layout of one K = 32 MMA: lane L holds rows (L&7) + 16(L>>4) (low half-word)
    // and that + 8 (high half-word), each for the K-half k1 = (L>>3)&1 (4 groups of 4)
    const int src_a = (lane & 7) + 16 * (lane >> 4);
    const int src_b = src_a + 8;
    const int k1 = (lane >> 3) & 1;
    constexpr int PD = 4;
    ExpRaw<NGH> raw[PD];
    auto fetch = [&](int it, ExpRaw<NGH>& x) {
      if (it >= total) return;
      int m_tile, n_tile;
      tile_coords<CG>(p, it / p.num_ks, m_tile, n_tile);
      exp_fetch<Cfg, Cfg::DIRECT>(p, static_cast<int64_t>(m_tile) * (128 * CG) + row_off + r, it % p.num_ks, h, x);
    };
#pragma unroll
    for (int j = 0; j < PD; ++j) fetch(j, raw[j]);
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
    for (int it0 = 0; it0 < total; it0 += PD) {
#pragma unroll
      for (int j = 0; j < PD; ++j) {
        const int it = it0 + j;
        if (it < total) {
          const int stage = it % STAGES;
          const int slot = it % RS;
          if (!Cfg::DIRECT) mbar_wait(rfull0 + 8 * slot, (it / RS) & 1);
          if (e == 0 && lane == 0) VENOM_TRACE_EVENT(3, it);
          uint32_t val[NGH];
          const uint8_t* vsrc = raw_smem + slot * Cfg::RAW_BYTES + r * (Cfg::VE * 2) + h * (NGH * 4);
          if constexpr (Cfg::DIRECT) {
#pragma unroll
            for (int u = 0; u < NGH; ++u) val[u] = raw[j].val[u];
          } else if constexpr (NGH >= 4) {
#pragma unroll
            for (int u = 0; u < NGH / 4; ++u) {
              const uint4 v = *reinterpret_cast<const uint4*>(vsrc + 16 * u);
              val[4 * u] = v.x; val[4 * u + 1] = v.y; val[4 * u + 2] = v.z; val[4 * u + 3] = v.w;
            }
          } else {
            const uint2 v = *reinterpret_cast<const uint2*>(vsrc);
            val[0] = v.x;
            val[1] = v.y;
          }
          uint32_t vw[16], mw[2];
          exp_build<Cfg>(raw[j], val, vw, mw);
          fetch(it + PD, raw[j]);
          // metadata words of this warp's 32 lanes for its two MMAs (kb = 2h, 2h+1)
          uint32_t ew[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const uint32_t wa = __shfl_sync(0xffffffffu, mw[u], src_a);
            const uint32_t wb = __shfl_sync(0xffffffffu, mw[u], src_b);
            ew[u] = ((wa >> (16 * k1)) & 0xFFFFu) | (((wb >> (16 * k1)) & 0xFFFFu) << 16);
          }
          mbar_wait(empty0 + 8 * stage, ((it / STAGES) & 1) ^ 1);
          if (e == 0 && lane == 0) VENOM_TRACE_EVENT(4, it);
          tmem_st_32x32b_x16(lane_base + Cfg::A_COL + 32 * stage + 16 * h, vw);
          tmem_st_32x32b_x2(lane_base + Cfg::E_COL + 4 * stage + 2 * h, ew[0], ew[1]);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (!Cfg::DIRECT) mbar_arrive(rempty0 + 8 * slot);  // values consumed (stores used them)
            if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(full0 + 8 * stage, 0));
            else mbar_arrive(full0 + 8 * stage);
          }
          if (e == 0 && lane == 0) VENOM_TRACE_EVENT(5, it);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();  // the leader's MMAs use the peer's TMEM until here
  if (warp == Cfg::W_MMA) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_2sm<512>(tmem_base);
    else tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace venom
