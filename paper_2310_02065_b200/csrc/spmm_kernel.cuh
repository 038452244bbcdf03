// spmm_kernel.cuh — V:N:M SpMM  C = A_vnm · B (+ bias)  for sm_100a.
//
// The paper's Spatha kernel (§4.1) is an Ampere design: cp.async staging,
// mma.sp m16n8k32 from registers, padded SMEM epilogue. What carries over to Blackwell is the
// mapping (Fig 4): per V-block, gather only the 4 selected rows of B for every
// group of M columns (through column-loc), so the block becomes a plain 2:4 sparse product over
// the condensed dimension K' = 4·K/M that the sparse tensor cores execute natively.
//
// B200 design:
//   * persistent CTAs (one per SM), static round-robin tile schedule, tiles of 128 rows × BN cols;
//   * warps 0..P-1 producers: column_idx words -> 4 B-row coordinates per group, TMA
//             tile::gather4 of the selected rows (the paper's stage 1₂ "only the rows of B selected
//             by column-loc") plus a TMA tile load of the compressed values; column_idx is
//             register-prefetched several stages ahead (stage 1₁ "two-level pre-fetching"). TMA
//             issue is serial per warp (~70 cycles per op, tools/microbench.cu), so P warps issue;
//   * warp P  MMA: tcgen05.cp metadata SMEM->TMEM, tcgen05.mma.sp (M=128, N=BN, K=32) with fp32
//             accumulation in TMEM (the paper's stage 2 on 5th-gen sparse tensor cores);
//   * warps P+1..P+8 epilogue: tcgen05.ld -> +bias -> round into registers, release the
//             accumulator, then 16-byte global stores (stage 3) overlapping the next tile;
//   * warps P+9..P+12 metadata (only without pre-ordered metadata): canonical per-row nibbles ->
//             the tensor-core metadata layout in
//             SMEM ("we also load directly ... the m-indices"), prefetched ahead.
// V = 128·k uses one V-block per tile; V ∈ {32, 64} packs NB = 128/V blocks into one 128-row A
// tile and issues one MMA per block (each block has its own gathered B' and accumulator).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "ptx_sm100.cuh"

namespace venom {

constexpr int kMaxPeers = 8;  // fused all-gather fan-out (one 8-GPU NVSwitch node)

struct SpmmParams {
  const uint16_t* values;   // read directly by the dense-K expanders (the gathered kernel uses TMA)
  const uint8_t* metadata;
  const uint8_t* column_idx;
  const uint16_t* bias;
  uint16_t* C;
  int64_t R, K, T, ldc;
  int V, M, G, meta_row;
  int num_ks;    // k-stages per tile: ceil(G / 32) gathered, ceil(K / 128) dense-K
  int last_kb;   // gathered: K = 32 MMAs of the last k-stage that hold real groups (1..4)
  int m_tiles;   // ceil(R / 128)
  int n_tiles;   // ceil(T / BN)
  int num_tiles;
  int group_n;   // tile order: groups of group_n column tiles, row tiles outer within a group
                 // (L2 reuse of both A and B across the CTAs running at the same time; 1 = T-band order)
  int is_bf16;
  int b3d;  // M = 4: B map is 3-D [T/64][K][64] (one box per stage) instead of 2-D
  int c_t;  // C stored transposed (token-major): element (r, t) at C[t * ldc + r]
  int bk;   // B given K-major (token-major activations, dtype[T][ldb]); M = 4 operand only
  int act;  // 1: GELU after the bias (row-major C only)
  int tma_c;  // row-major C stored by TMA boxes (tm_c encoded by the host)
  int e4d;    // M64 + pre-ordered metadata: tm_e is the 4-D lane-permuting map (else 8 row loads)
  // fused all-gather: every C element is also stored at the same offset
  // relative to each of n_peers other buffers (e.g. the other ranks' full-output buffers, mapped
  // peer-to-peer over NVLink, each pointer already offset to this rank's slice)
  int n_peers;
  uint16_t* c_peers[kMaxPeers];
  int dbg;  // debug/ablation flags (0 in production)
};

template <int NB_, int BN_, int STAGES_, int PRODUCERS_ = 8, int CG_ = 1, bool PRE_ = false, int MB_ = 1>
struct SpmmCfg {
  static constexpr int MB = MB_;              // 128-row blocks per CTA (2: two accumulators, one
                                              // B tile serves both; CTA pair + 2:4 form only)
  static constexpr bool PRE = PRE_;           // metadata pre-ordered for the tensor core (TMA-loaded,
                                              // tcgen05.cp to TMEM by the MMA thread): no metadata warps
  static constexpr int NB = NB_;              // V-blocks per 128-row tile
  static constexpr int CG = CG_;              // 2: CTA pair (cta_group::2, 256-row tiles): needs
                                              // one column_idx per pair tile (V % 256 == 0 or M == 4)
  static constexpr int BN = BN_;              // output columns per tile (MMA N)
  static constexpr int BNH = BN / CG_;        // B' columns staged by one CTA
  static constexpr int STAGES = STAGES_;
  static constexpr int P = PRODUCERS_;        // gather-issuing warps (TMA issue is per-warp serial)
  static constexpr int BM = 128;              // rows per CTA
  static constexpr int KG = 32;               // groups per k-stage: K' = 128, 4 MMAs of K = 32
  static constexpr int A_BLOCK = BM * 128;    // 128 rows × 64 compressed values × 2 B (SW128)
  static constexpr int A_BYTES = MB_ * A_BLOCK;
  static constexpr int B_CHUNK = 128 * 128;   // 128 K'-rows × 64 columns × 2 B (SW128, MN-major)
  static constexpr int NCH = (BNH + 63) / 64; // 64-column chunks of B' per block (last may be partial)
  static constexpr int B_BYTES = NCH * B_CHUNK;
  static constexpr int E_BLOCK = 128 * 16;    // 128 lanes × 4 metadata words
  static constexpr int E_BYTES = PRE_ ? MB_ * E_BLOCK : 0;
  static constexpr int STAGE_BYTES = A_BYTES + NB * B_BYTES + E_BYTES;
  static constexpr int TX_BYTES = STAGE_BYTES;  // per CTA
  // M64 (V = 64, two V-blocks per 128-row tile): each block is one M = 64 MMA on its own 64 A rows,
  // its accumulator on one half of every TMEM lane quarter (block b: lanes 32q + 16b .. +15, the
  // D and metadata addresses both offset by 16b lanes; probed in tools/probe_m64.cu). Both blocks
  // share one BN-column accumulator: no wasted tensor work or TMEM, so the accumulator is
  // double-buffered. V = 32 (NB = 4) keeps one M = 128 MMA per block into its own columns.
  // V = 32 (NB = 4) uses the same lane halves: M = 64 MMAs over rows 0-63 (lane offset 0) and
  // 64-127 (offset 16), each half run once per V-block of B' with the block's result kept: blocks
  // 0 / 2 write columns [0, BN), blocks 1 / 3 columns [BN, 2·BN) (half the wasted tensor work and
  // TMEM of one M = 128 MMA per block, so the accumulator is double-buffered at BN = 64).
  static constexpr bool M64 = (NB_ == 2 || NB_ == 4);
  static constexpr int ACC_COLS = (M64 ? NB / 2 : NB) * MB_ * BN;
  // TMEM: accumulators, then 4 metadata columns per row block and stage
  static constexpr int E_PER_STAGE = 4 * MB_;
  static constexpr int ACC_BUFS = (2 * ACC_COLS + E_PER_STAGE * STAGES_ <= 512) ? 2 : 1;
  static constexpr int E_COL = ACC_BUFS * ACC_COLS;
  static constexpr int NOPS = NB * NCH * 32;  // gather4 ops per stage (one per group × chunk × block)
  static constexpr int OPS_PER_WARP = (NOPS + P - 1) / P;  // the last warp may get fewer
  static constexpr int LANE_OPS = (OPS_PER_WARP + 31) / 32;
  // warp roles: [0,P) producers, P MMA, P+1..P+8 epilogue, P+9..P+12 metadata; epilogue and
  // metadata warps address TMEM lane quarter (warp % 4)
  // MB = 2: 16 epilogue warps (row block × column half × lane quarter) so that the whole
  // accumulator pair fits in registers and is released before the stores
  static constexpr int EPI_WARPS = (MB_ == 2) ? 16 : 8;
  static constexpr int W_MMA = P, W_EPI = P + 1, W_META = P + 1 + EPI_WARPS;
  static constexpr int NUM_THREADS = 32 * (P + 1 + EPI_WARPS + (PRE_ ? 0 : 4));
  static_assert(CG_ == 1 || NB_ == 1, "CTA pairs need one V-block per CTA tile");
  static constexpr int BAR_BYTES = 1024;  // keeps the epilogue slots 1 KB aligned (TMA-store swizzle)
  // per epilogue warp: one 32-row output chunk (64 B rows; 32 B rows for MB = 2); MB = 1 stages its
  // chunks for TMA stores, double-buffered when the shared memory allows
  static constexpr int EPI_SLOT = (MB_ == 2) ? 1024 : 2048;
  static constexpr int EPI_BUFS =
      (MB_ == 1 && 1024 + STAGES_ * STAGE_BYTES + BAR_BYTES + EPI_WARPS * 2 * EPI_SLOT <= 227 * 1024) ? 2 : 1;
  static constexpr int EPI_STAGE_BYTES = EPI_SLOT * EPI_BUFS;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + BAR_BYTES + EPI_WARPS * EPI_STAGE_BYTES;
  static_assert((BNH % 64 == 0 || MB_ == 2) && BNH % 8 == 0 && BN <= 256, "BN");
  static_assert(MB_ == 1 || (CG_ == 2 && NB_ == 1 && PRE_), "two row blocks: CTA pair, pre-ordered metadata");
  static_assert(E_COL + E_PER_STAGE * STAGES_ <= 512, "TMEM budget");
  static_assert(STAGE_BYTES % 1024 == 0, "stage alignment");
  static_assert(SMEM_BYTES <= 227 * 1024, "smem budget");
};

constexpr int kPrefetch = 4;  // register prefetch depth of column_idx / metadata (k-stages)

template <bool kBF16>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  if constexpr (kBF16) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}

// Canonical metadata of one row for one k-stage (32 groups = 16 bytes): the four 32-bit words
// (one per K=32 MMA; group 8·kb+q in bits 4q..4q+3). Groups past G and rows past R read as the
// valid all-zero-value pattern 0x4 (m-indices 0,1).
__device__ __forceinline__ void load_meta_stage(const SpmmParams& p, int64_t row, int ks,
                                                uint32_t (&w)[4]) {
  if (row >= p.R) {
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) w[kb] = 0x44444444u;
    return;
  }
  const uint8_t* base = p.metadata + row * p.meta_row + ks * 16;
  const int g_left = p.G - ks * 32;  // groups of this stage that exist (multiple of 4)
  if (g_left >= 32 && (p.meta_row & 15) == 0) {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(base));
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    return;
  }
  // halfword granularity (meta_row is even because G % 4 == 0); tail halfwords -> 0x4444
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    uint32_t lo = 0x4444u, hi = 0x4444u;
    if (8 * kb + 4 <= g_left) lo = __ldg(reinterpret_cast<const uint16_t*>(base) + 2 * kb);
    if (8 * kb + 8 <= g_left) hi = __ldg(reinterpret_cast<const uint16_t*>(base) + 2 * kb + 1);
    w[kb] = lo | (hi << 16);
  }
}

// Persistent static schedule: CTA b runs tiles b, b + grid, b + 2·grid, ... With CTA pairs (CG = 2)
// the unit of scheduling is the cluster: pair b runs tiles b, b + pairs, ...
// Tile order: the column tiles are cut into groups of group_n; within a group the row tiles are
// outer and the group's column tiles inner, so the grid's concurrently running tiles cover about
// grid / group_n row tiles × group_n column tiles — each A row tile and each B column slab is then
// streamed from HBM by several CTAs at once (group_n = 1, the default, is the T-band order: all row
// tiles of one column band first; spmm_launch.cuh).
template <int CG = 1>
__device__ __forceinline__ void tile_coords(const SpmmParams& p, int tl, int& m_tile, int& n_tile) {
  const int t = static_cast<int>(blockIdx.x) / CG + tl * (static_cast<int>(gridDim.x) / CG);
  const int per_group = p.m_tiles * p.group_n;
  const int grp = t / per_group;
  const int rem = t - grp * per_group;
  const int n0 = grp * p.group_n;
  const int gw = min(p.group_n, p.n_tiles - n0);  // the last group may be narrower
  m_tile = rem / gw;
  n_tile = n0 + (rem - m_tile * gw);
}
template <int CG = 1>
__device__ __forceinline__ int my_tile_count(const SpmmParams& p) {
  const int gid = static_cast<int>(blockIdx.x) / CG, ng = static_cast<int>(gridDim.x) / CG;
  return gid < p.num_tiles ? (p.num_tiles - gid + ng - 1) / ng : 0;
}

// MMA issuer (one elected lane of the pair leader): per k-stage, 4 sparse MMAs (K = 32) per
// V-block. Stage layout: [A 16 KB K-major SW128][NB × B' (BNH/64 chunks × 16 KB, MN-major SW128)];
// the stage's metadata sits in TMEM columns E_COL + 4·stage (written by the metadata warps).
template <class Cfg, bool kBF16, int CG = 1, bool kBK = false>
__device__ __forceinline__ void mma_role(const SpmmParams& p, int my_tiles, uint32_t tmem_base,
                                         uint32_t smem0, uint32_t full0, uint32_t empty0,
                                         uint32_t accf0, uint32_t acce0, int lane) {
  using namespace ptx;
  constexpr int STAGES = Cfg::STAGES, NB = Cfg::NB, BN = Cfg::BN;
  // kBK: B' is K-major (bit 16 clear), else MN-major
  constexpr uint32_t idesc =
      idesc_sp_f16(kBF16 ? 1u : 0u, Cfg::M64 ? 64 : 128 * CG, BN) & (kBK ? ~(1u << 16) : ~0u);
  for (int tl = 0; tl < my_tiles; ++tl) {
    const int ab = tl % Cfg::ACC_BUFS;
    const uint32_t aphase = (tl / Cfg::ACC_BUFS) & 1;
    mbar_wait(acce0 + 8 * ab, aphase ^ 1);
    tc_fence_after();
    const uint32_t d_tile = tmem_base + ab * Cfg::ACC_COLS;
    for (int ks = 0; ks < p.num_ks; ++ks) {
      const int it = tl * p.num_ks + ks;
      const int stage = it % STAGES;
      mbar_wait(full0 + 8 * stage, (it / STAGES) & 1);
      tc_fence_after();
      if (lane == 0) VENOM_TRACE_EVENT(1, it);
      if (lane == 0 && !(p.dbg & 2)) {  // ablation 2: no MMAs (commits only)
        const uint32_t sbase = smem0 + stage * Cfg::STAGE_BYTES;
        const uint32_t e_tmem = tmem_base + Cfg::E_COL + Cfg::E_PER_STAGE * stage;
        if constexpr (Cfg::PRE) {
          // pre-ordered metadata block(s) of this stage: SMEM [128 lanes][16 B] -> 4 TMEM columns
          // per row block; tcgen05.cp and the MMAs below execute in issue order
#pragma unroll
          for (int mb = 0; mb < Cfg::MB; ++mb) {
            const uint64_t edesc =
                smem_desc(sbase + Cfg::A_BYTES + NB * Cfg::B_BYTES + mb * Cfg::E_BLOCK, 16, 128, 0);
            if constexpr (CG == 2) tc_cp_128x128b_2sm(e_tmem + 4 * mb, edesc);
            else tc_cp_128x128b(e_tmem + 4 * mb, edesc);
          }
        }
        const int n_kb = (ks == p.num_ks - 1) ? p.last_kb : 4;
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
          if (kb >= n_kb) break;
#pragma unroll
          for (int b = 0; b < NB * Cfg::MB; ++b) {
            // MB = 2: row block b has its own A tile and metadata, the B tile is shared;
            // NB > 1: V-block b has its own gathered B', the A tile is shared
            // M64: block b's accumulator and metadata sit 16·h lanes into every lane quarter, h the
            // 64-row half of the tile holding the block (NB = 2: h = b; NB = 4: h = b / 2, and the
            // odd block of a half writes the second BN columns)
            const int half = (NB == 4) ? (b >> 1) : b;
            const uint32_t lane_off = Cfg::M64 ? (static_cast<uint32_t>(16 * half) << 16) : 0u;
            const uint32_t col_off = (Cfg::M64 && NB == 4) ? static_cast<uint32_t>((b & 1) * BN) : 0u;
            const uint32_t e_addr = e_tmem + (Cfg::MB > 1 ? 4 * b : 0) + kb + lane_off;
            const uint32_t id2 = e_addr & 1u;  // odd metadata column -> selector id2
            // A: K-major SW128, 8-row groups 1024 B apart; K advance 32 B per K=32 MMA
            // (M64: block b's 64 rows start 8 KB into the tile)
            const uint64_t adesc =
                smem_desc(sbase + (Cfg::MB > 1 ? b * Cfg::A_BLOCK : 0) + (Cfg::M64 ? half * 8192 : 0) + kb * 32,
                          16, 1024, 2);
            // B': MN-major SW128, 64-column chunks B_CHUNK apart, 8 K-rows 1024 B apart;
            // K advance 32 rows = 4096 B per MMA
            // kBK: two K-major SW128 regions of BNH rows × 64 K-elements; K = 32 per MMA = 64 B
            const uint64_t bdesc =
                kBK ? smem_desc(sbase + Cfg::A_BYTES + (kb >> 1) * (Cfg::BNH * 128) + (kb & 1) * 64, 16, 1024, 2)
                    : smem_desc(sbase + Cfg::A_BYTES + (NB > 1 ? b * Cfg::B_BYTES : 0) + kb * 4096,
                                Cfg::B_CHUNK, 1024, 2);
            if constexpr (CG == 2)
              tc_mma_sp_f16_2sm(d_tile + b * BN, adesc, bdesc, idesc | id2, e_addr & ~1u,
                                (ks | kb) != 0 ? 1u : 0u);
            else
              tc_mma_sp_f16(Cfg::M64 ? d_tile + lane_off + col_off : d_tile + b * BN, adesc, bdesc, idesc | id2,
                            e_addr & ~1u, (ks | kb) != 0 ? 1u : 0u);
          }
        }
      }
      if (lane == 0) {
        VENOM_TRACE_EVENT(8, it);
        if constexpr (CG == 2) {
          tc_commit_2sm_mc(empty0 + 8 * stage, 0x3);
          if (ks == p.num_ks - 1) tc_commit_2sm_mc(accf0 + 8 * ab, 0x3);
        } else if (p.dbg & 512) {  // ablation 512 (with 2): plain arrives instead of commits
          mbar_arrive(empty0 + 8 * stage);
          if (ks == p.num_ks - 1) mbar_arrive(accf0 + 8 * ab);
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

// Epilogue (8 warps: each TMEM lane quarter twice, one half of the tile's columns per warp):
// TMEM -> +bias (fp32) -> RNE to fp16/bf16 packed in registers; the accumulator buffer is released
// to the MMA warp as soon as it has been read, and the 16-byte global stores overlap the next
// tile's main loop (a single TMEM accumulator no longer serialises the epilogue).
// kACT: the activation after the bias, in fp32 before the rounding — a separate instantiation per
// activation (a runtime activation branch slowed every SpMM):
//   1 GELU, erf form (torch.nn.functional.gelu): erff is ~20 FMA-pipe instructions per element,
//     which makes the epilogue pace the kernel (+23% on the encoder's FFN1; a Chebyshev erfc with
//     a MUFU reciprocal and exp measured no faster);
//   2 GELU, tanh form (F.gelu(approximate="tanh"), the original BERT's and GPT-2/3's): one MUFU
//     tanh.approx (max relative error 2^-11, below the fp16 output's rounding) and 4 FMAs.
__device__ __forceinline__ float gelu_f(float v) { return 0.5f * v * (1.0f + erff(v * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_tanh_f(float v) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.7978845608028654f * fmaf(0.044715f * v, v * v, v)));
  return 0.5f * v * (1.0f + t);
}
template <int kACT>
__device__ __forceinline__ float act_f(float v) {
  if constexpr (kACT == 1) return gelu_f(v);
  else if constexpr (kACT == 2) return gelu_tanh_f(v);
  else return v;
}

template <class Cfg, bool kBF16, int CG = 1, bool kCT = false, int kACT = 0>
__device__ __forceinline__ void epilogue_role(const SpmmParams& p, int my_tiles, uint32_t tmem_base,
                                              uint32_t accf0, uint32_t acce0, int warp, int lane,
                                              uint32_t stage_smem = 0, const CUtensorMap* tm_c = nullptr) {
  using namespace ptx;
  constexpr int NB = Cfg::NB, BN = Cfg::BN;
  constexpr int HC = BN / (Cfg::EPI_WARPS / 4);  // columns per warp
  constexpr int NCH = (HC + 31) / 32;   // 32-column TMEM loads per warp
  const int q = warp & 3;               // TMEM lane quarter this warp may access
  const int h = (warp - Cfg::W_EPI) >> 2;  // column half
  const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0u;
  // row of this lane within the (pair) tile; M64: the lane half (lane >> 4) is the V-block
  const int r_local = Cfg::M64 ? 64 * (lane >> 4) + 16 * q + (lane & 15)
                               : 128 * static_cast<int>(rank) + 32 * q + lane;
  // row of slot row r (0..31) of this warp's 32-row staging chunk, relative to the tile's row 0
  auto slot_row = [&](int r) -> int {
    return Cfg::M64 ? 64 * (r >> 4) + 16 * q + (r & 15) : 128 * static_cast<int>(rank) + 32 * q + r;
  };
  for (int tl = 0; tl < my_tiles; ++tl) {
    int m_tile, n_tile;
    tile_coords<CG>(p, tl, m_tile, n_tile);
    const int ab = tl % Cfg::ACC_BUFS;
    mbar_wait_sleep(accf0 + 8 * ab, (tl / Cfg::ACC_BUFS) & 1);  // a whole tile: sleep, do not poll
    tc_fence_after();
    if (warp == Cfg::W_EPI && lane == 0) VENOM_TRACE_EVENT(9, tl);
    const int64_t row = static_cast<int64_t>(m_tile) * (128 * CG) + r_local;
    // warp-uniform accumulator column block of this lane quarter (M64 with NB = 4: quarters 2, 3
    // hold the odd blocks, written at columns [BN, 2·BN))
    const int b = (NB == 1 || (Cfg::M64 && NB == 2)) ? 0 : (Cfg::M64 ? (q >> 1) : (32 * q) / p.V);
    const float bv = (p.bias != nullptr && row < p.R)
                         ? (kBF16 ? __uint_as_float(static_cast<uint32_t>(p.bias[row]) << 16)
                                  : __half2float(__ushort_as_half(p.bias[row])))
                         : 0.0f;
    const uint32_t t_row = tmem_base + (static_cast<uint32_t>(32 * q) << 16) +
                           ab * Cfg::ACC_COLS + b * BN + h * HC;
    uint32_t pk[NCH][16];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      uint32_t v[32];
      if (p.dbg & 64) {  // ablation 64: no accumulator reads
#pragma unroll
        for (int u = 0; u < 32; ++u) v[u] = 0u;
      } else {
        tmem_ld_32x32b_x32(t_row + 32 * c, v);
        tmem_ld_wait();
      }
#pragma unroll
      for (int j = 0; j < 16; ++j)
        pk[c][j] = pack2<kBF16>(act_f<kACT>(__uint_as_float(v[2 * j]) + bv),
                                act_f<kACT>(__uint_as_float(v[2 * j + 1]) + bv));
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(acce0 + 8 * ab, 0));  // pair leader
      else mbar_arrive(acce0 + 8 * ab);
    }
    const int64_t col_base = static_cast<int64_t>(n_tile) * BN + h * HC;
    if (kCT && tm_c != nullptr && !(p.dbg & 4)) {
      // token-major C through the TMA-store epilogue: lane pairs swap halves with one shuffle (the
      // even lane then holds rows (r, r+1) of column t, the odd lane rows (r-1, r) of column t+1),
      // each 32-bit word goes to its place in a shared-memory slot laid out as the C^T box
      // [32 columns t][32 rows r] (64-byte rows, 64-byte swizzle; M64: two [32 t][16 r] halves of
      // 32-byte rows, 32-byte swizzle), and one lane stores the box(es) with cp.async.bulk.tensor.
      // (The direct path below issued a bounds-checked store per word and per peer: the epilogue
      // then paced the V = 64 kernel, 0.19 vs 0.11 ms for row-major C at the encoder's QKV layer.)
      const bool odd = lane & 1;
      const int rb0 = m_tile * (128 * CG);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        if (32 * c >= HC) break;
        const uint32_t slot = stage_smem + (c % Cfg::EPI_BUFS) * Cfg::EPI_SLOT;
        if (lane == 0) {
          if (Cfg::EPI_BUFS == 2) bulk_wait_group_read<1>();
          else bulk_wait_group_read<0>();
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t w = pk[c][j];
          const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, w, 1);
          const uint32_t v = odd ? ((o >> 16) | (w & 0xFFFF0000u)) : ((w & 0xFFFFu) | (o << 16));
          const int t = 2 * j + (odd ? 1 : 0);  // column within the chunk = slot row
          uint32_t a;
          if constexpr (Cfg::M64) {
            const int wd = (lane & 15) >> 1;  // word of the 16-row half: rows 2·wd, 2·wd + 1
            a = slot + (lane >> 4) * 1024 + t * 32 + ((((wd >> 2) ^ (t >> 2)) & 1) << 4) + (wd & 3) * 4;
          } else {
            const int wd = lane >> 1;
            a = slot + t * 64 + ((((wd >> 2) ^ (t >> 1)) & 3) << 4) + (wd & 3) * 4;
          }
          asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
        }
        fence_proxy_async_smem();
        __syncwarp();
        const int tcol = static_cast<int>(col_base) + 32 * c;
        if (lane == 0) {
          tma_store_2d(tm_c, slot, rb0 + slot_row(0), tcol);
          if constexpr (Cfg::M64) tma_store_2d(tm_c, slot + 1024, rb0 + slot_row(16), tcol);
          bulk_commit_group();
        }
        if (p.n_peers > 0) {
          // fused all-gather: the chunk from the slot to every peer buffer, 16-byte row segments
          constexpr int HALVES = Cfg::M64 ? 2 : 1, RB = Cfg::M64 ? 32 : 64;  // row bytes per half
#pragma unroll
          for (int hh = 0; hh < HALVES; ++hh)
#pragma unroll
            for (int jj = 0; jj < 4 / HALVES; ++jj) {
              const int spr = RB / 16;  // 16-byte segments per slot row
              const int t = (32 / spr) * jj + lane / spr, sgm = lane % spr;
              const int swz = Cfg::M64 ? ((t >> 2) & 1) : ((t >> 1) & 3);
              uint4 o;
              const uint32_t a = slot + hh * 1024 + t * RB + ((sgm ^ swz) << 4);
              asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(o.x), "=r"(o.y), "=r"(o.z), "=r"(o.w) : "r"(a) : "memory");
              const int64_t r = rb0 + slot_row(16 * hh) + 8 * sgm;
              const int64_t tt = tcol + t;
              if (tt < p.T && r < p.R)
                for (int pp = 0; pp < p.n_peers; ++pp) {
                  uint16_t* dst = p.c_peers[pp] + tt * p.ldc + r;
                  if (r + 8 <= p.R) {
                    *reinterpret_cast<uint4*>(dst) = o;
                  } else {
                    const uint16_t* e = reinterpret_cast<const uint16_t*>(&o);
                    for (int u = 0; u < p.R - r; ++u) dst[u] = e[u];
                  }
                }
            }
        }
      }
      if (warp == Cfg::W_EPI && lane == 0) VENOM_TRACE_EVENT(10, tl);
    } else if constexpr (kCT) {
      // token-major C (C^T[t][r]): the warp's 32 lanes hold 32 consecutive rows of columns t, t+1
      // (one packed word). Lane pairs swap halves with one shuffle so the even lane stores rows
      // (r, r+1) of column t and the odd lane rows (r-1, r) of column t+1 as 32-bit words: every
      // store instruction writes 64 contiguous bytes to each of two C^T rows
      const bool odd = lane & 1;
      const int64_t r0 = row - (odd ? 1 : 0);  // even row of the pair
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t w = pk[c][j];
          const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, w, 1);
          const uint32_t v = odd ? ((o >> 16) | (w & 0xFFFF0000u)) : ((w & 0xFFFFu) | (o << 16));
          const int jj = 32 * c + 2 * j + (odd ? 1 : 0);  // column within the warp's slice
          const int64_t t = col_base + jj;
          if (jj < HC && t < p.T && r0 < p.R) {
            const int64_t off = t * p.ldc + r0;
            const bool pair = r0 + 1 < p.R;
            for (int pp = -1; pp < p.n_peers; ++pp) {  // this rank's C, then the fused all-gather
              uint16_t* dst = (pp < 0 ? p.C : p.c_peers[pp]) + off;
              if (pair) *reinterpret_cast<uint32_t*>(dst) = v;
              else *dst = static_cast<uint16_t>(v & 0xFFFFu);
            }
          }
        }
    } else if (p.dbg & 4) {  // ablation 4: no C stores
    } else if (tm_c != nullptr && !(p.dbg & 16384)) {
      // TMA-store epilogue (the paper's stage 3 output staging, on the bulk-copy
      // engine): each 32-row × 32-column chunk is written to a shared-memory slot in the 64-byte
      // swizzled layout of the C tensor map (16-byte segment s of row r at segment s ^ ((r >> 1) & 3),
      // conflict-free), then one lane stores the box with cp.async.bulk.tensor; the TMA unit
      // clips the ragged R / T edges. Slots are double-buffered when shared memory allows: a slot
      // is rewritten only once the store issued from it has read it.
      const int row_base = m_tile * (128 * CG);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        if (32 * c >= HC) break;
        const uint32_t slot = stage_smem + (c % Cfg::EPI_BUFS) * Cfg::EPI_SLOT;
        if (lane == 0) {
          if (Cfg::EPI_BUFS == 2) bulk_wait_group_read<1>();
          else bulk_wait_group_read<0>();
        }
        __syncwarp();
#pragma unroll
        for (int sgm = 0; sgm < 4; ++sgm) {
          const uint32_t a = slot + lane * 64 + ((sgm ^ ((lane >> 1) & 3)) * 16);
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(pk[c][4 * sgm]),
                       "r"(pk[c][4 * sgm + 1]), "r"(pk[c][4 * sgm + 2]), "r"(pk[c][4 * sgm + 3]) : "memory");
        }
        fence_proxy_async_smem();  // the generic-proxy writes, visible to the bulk-copy engine
        __syncwarp();
        if (lane == 0) {
          if constexpr (Cfg::M64) {
            // the two V-blocks' 16-row halves (the C map's box is 16 rows for M64)
            tma_store_2d(tm_c, slot, static_cast<int32_t>(col_base + 32 * c), row_base + slot_row(0));
            tma_store_2d(tm_c, slot + 1024, static_cast<int32_t>(col_base + 32 * c), row_base + slot_row(16));
          } else {
            tma_store_2d(tm_c, slot, static_cast<int32_t>(col_base + 32 * c), row_base + slot_row(0));
          }
          bulk_commit_group();
        }
        if (p.n_peers > 0) {
          // fused all-gather: the same chunk from the slot to every peer buffer, 8 rows × 64
          // contiguous bytes per store instruction (the slot stays valid: it is rewritten only
          // after this warp's next pass)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = 8 * j + (lane >> 2), sgm = lane & 3;
            uint4 o;
            const uint32_t a = slot + r * 64 + ((sgm ^ ((r >> 1) & 3)) * 16);
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(o.x), "=r"(o.y), "=r"(o.z), "=r"(o.w) : "r"(a) : "memory");
            const int64_t orow = row_base + slot_row(r);
            const int64_t ocol = col_base + 32 * c + 8 * sgm;
            if (orow < p.R && ocol < p.T)
              for (int pp = 0; pp < p.n_peers; ++pp)
                *reinterpret_cast<uint4*>(p.c_peers[pp] + orow * p.ldc + ocol) = o;
          }
        }
      }
      if (warp == Cfg::W_EPI && lane == 0) VENOM_TRACE_EVENT(10, tl);
    } else if (stage_smem != 0 && !(p.dbg & 16384)) {  // ablation 16384: direct stores below
      // transpose each 32-row × 32-column chunk through a 2 KB shared-memory slot so that every
      // store instruction writes 8 rows × 64 contiguous bytes (full sectors) instead of 32 rows ×
      // 16 bytes; 16-byte segments XOR-swizzled by row to keep both passes bank-conflict free
      const int64_t row_base = static_cast<int64_t>(m_tile) * (128 * CG);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        if (32 * c >= HC) break;
#pragma unroll
        for (int sgm = 0; sgm < 4; ++sgm) {
          const uint32_t a = stage_smem + lane * 64 + ((sgm ^ ((lane >> 1) & 3)) * 16);
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(pk[c][4 * sgm]),
                       "r"(pk[c][4 * sgm + 1]), "r"(pk[c][4 * sgm + 2]), "r"(pk[c][4 * sgm + 3]) : "memory");
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = 8 * j + (lane >> 2), sgm = lane & 3;
          uint4 o;
          const uint32_t a = stage_smem + r * 64 + ((sgm ^ ((r >> 1) & 3)) * 16);
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(o.x), "=r"(o.y), "=r"(o.z), "=r"(o.w) : "r"(a) : "memory");
          const int64_t orow = row_base + slot_row(r);
          const int64_t ocol = col_base + 32 * c + 8 * sgm;
          // ablation 8192: the shared-memory transposes without the global stores
          if (orow < p.R && ocol < p.T && !(p.dbg & 8192)) *reinterpret_cast<uint4*>(p.C + orow * p.ldc + ocol) = o;
        }
        __syncwarp();
      }
      if (warp == Cfg::W_EPI && lane == 0) VENOM_TRACE_EVENT(10, tl);
    } else if (row < p.R) {
      uint16_t* dst = p.C + row * p.ldc + col_base;
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (32 * c + 8 * u < HC && col_base + 32 * c + 8 * u < p.T)
            *reinterpret_cast<uint4*>(dst + 32 * c + 8 * u) =
                make_uint4(pk[c][4 * u], pk[c][4 * u + 1], pk[c][4 * u + 2], pk[c][4 * u + 3]);
    }
  }
  // the CTA's shared memory must outlive the stores that read it
  if (tm_c != nullptr && lane == 0) bulk_wait_group_all();
}

// Epilogue for MB = 2 (two 128-row accumulators per CTA, BN = 240): 16 warps, warp e = w - W_EPI
// takes row block e / 8, column half (e / 4) % 2 and TMEM lane quarter w % 4; its 32 × 120 slice
// goes to registers (packed), the accumulator pair is released, then each 16-column chunk is
// transposed through a 1 KB swizzled SMEM slot so a store writes 16 rows × 32 contiguous bytes.
template <class Cfg, bool kBF16, int CG>
__device__ __forceinline__ void epilogue_role_mb2(const SpmmParams& p, int my_tiles, uint32_t tmem_base,
                                                  uint32_t accf0, uint32_t acce0, int warp, int lane,
                                                  uint32_t stage_smem) {
  using namespace ptx;
  constexpr int BN = Cfg::BN;
  constexpr int HALF = BN / 2;            // valid columns per half
  constexpr int NCH = 2 * ((HALF + 31) / 32);  // 16-column TMEM loads per half (even)
  const int e = warp - Cfg::W_EPI;
  const int q = warp & 3;
  const int b = e >> 3;
  const int h = (e >> 2) & 1;
  const uint32_t rank = cluster_ctarank();
  for (int tl = 0; tl < my_tiles; ++tl) {
    int m_tile, n_tile;
    tile_coords<CG>(p, tl, m_tile, n_tile);
    mbar_wait_sleep(accf0, tl & 1);
    tc_fence_after();
    if (warp == Cfg::W_EPI && lane == 0) VENOM_TRACE_EVENT(9, tl);
    const int64_t row_base = static_cast<int64_t>(m_tile) * (128 * CG * 2) + b * (128 * CG) +
                             128 * static_cast<int>(rank) + 32 * q;
    const int64_t row = row_base + lane;
    const float bv = (p.bias != nullptr && row < p.R)
                         ? (kBF16 ? __uint_as_float(static_cast<uint32_t>(p.bias[row]) << 16)
                                  : __half2float(__ushort_as_half(p.bias[row])))
                         : 0.0f;
    const uint32_t t_row = tmem_base + (static_cast<uint32_t>(32 * q) << 16) + b * BN + h * HALF;
    uint32_t pk[NCH][8];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      uint32_t v[16];
      tmem_ld_32x32b_x16(t_row + 16 * c, v);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 8; ++j)
        pk[c][j] = pack2<kBF16>(__uint_as_float(v[2 * j]) + bv, __uint_as_float(v[2 * j + 1]) + bv);
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive_cluster(mapa_shared(acce0, 0));  // pair leader
    if (warp == Cfg::W_EPI && lane == 0) VENOM_TRACE_EVENT(12, tl);
    if (p.dbg & 4) continue;  // ablation 4: no C stores
    const int64_t col_base = static_cast<int64_t>(n_tile) * BN + h * HALF;
    // 32-column chunks (64 B per row), 16 rows at a time through the 1 KB slot: every store
    // instruction writes 8 rows × 64 contiguous bytes
#pragma unroll
    for (int c = 0; c < NCH / 2; ++c) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        if ((lane >> 4) == hh) {
          const int rr = lane & 15;
#pragma unroll
          for (int sgm = 0; sgm < 4; ++sgm) {
            const uint32_t* src = pk[2 * c + (sgm >> 1)] + 4 * (sgm & 1);
            const uint32_t a = stage_smem + rr * 64 + ((sgm ^ ((rr >> 1) & 3)) * 16);
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(src[0]), "r"(src[1]),
                         "r"(src[2]), "r"(src[3]) : "memory");
          }
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int r = 8 * j + (lane >> 2), sgm = lane & 3;
          uint4 o;
          const uint32_t a = stage_smem + r * 64 + ((sgm ^ ((r >> 1) & 3)) * 16);
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(o.x), "=r"(o.y), "=r"(o.z), "=r"(o.w) : "r"(a) : "memory");
          const int64_t orow = row_base + 16 * hh + r;
          const int cc = 32 * c + 8 * sgm;  // column within the half
          if (orow < p.R && cc < HALF && col_base + cc < p.T)
            *reinterpret_cast<uint4*>(p.C + orow * p.ldc + col_base + cc) = o;
        }
        __syncwarp();
      }
    }
    if (warp == Cfg::W_EPI && lane == 0) VENOM_TRACE_EVENT(10, tl);
  }
}

// M = 4 producer (the 2:4 operand and the #18 re-encoding): B' is a plain K-slice of B, so a stage
// is three TMA ops. Lane 0 of warp 0 issues expect_tx, the A box(es) and the metadata block(s);
// lane 0 of warp 1 the B' box (one 3-D box, or one 2-D box per 64-column chunk on warps 1..NCH).
// Tile coordinates advance incrementally: the whole per-stage cost is a barrier wait and a few
// instructions (the generic per-stage coordinate computation took longer than the stage's MMAs).
template <class Cfg, bool kBK = false>
__device__ __forceinline__ void producer_contiguous(const SpmmParams& p, const CUtensorMap* tm_values,
                                                    const CUtensorMap* tm_b, const CUtensorMap* tm_e,
                                                    int my_tiles, uint32_t smem0, uint32_t full0,
                                                    uint32_t empty0, uint32_t rank, int warp) {
  using namespace ptx;
  constexpr int STAGES = Cfg::STAGES, CG = Cfg::CG, MB = Cfg::MB;
  const bool b3d = p.b3d != 0;
  const int role = warp == 0 ? 0 : (((b3d || kBK) ? warp == 1 : warp <= Cfg::NCH) ? 1 : -1);
  if (role < 0 || my_tiles == 0) return;
  const uint64_t pol_a = policy_evict_first();
  const uint64_t pol_b = policy_evict_last();
  // ablation flags (p.dbg, tools only): 1 no B loads, 16 no A load, 2048 no metadata load
  const bool do_a = !(p.dbg & 16), do_b = !(p.dbg & 1), do_e = Cfg::PRE && !(p.dbg & 2048);
  const uint32_t tx = CG * ((do_a ? Cfg::A_BYTES : 0) + (do_b ? Cfg::B_BYTES : 0) + (do_e ? Cfg::E_BYTES : 0));
  const uint32_t fbar0 = (CG == 2) ? mapa_shared(full0, 0) : full0;
  const int row_off = 128 * static_cast<int>(rank);
  int m_tile, n_tile, arow = 0, col0 = 0, eblk0 = 0;
  auto set_tile = [&](int tl) {
    tile_coords<CG>(p, tl, m_tile, n_tile);
    arow = m_tile * 128 * CG * MB + row_off;
    col0 = n_tile * Cfg::BN + static_cast<int>(rank) * Cfg::BNH;
    eblk0 = (m_tile * MB * CG + static_cast<int>(rank)) * p.num_ks;
  };
  set_tile(0);
  int tl = 0, ks = 0, stage = 0;
  uint32_t phase = 0;
  const int total = my_tiles * p.num_ks;
  for (int it = 0; it < total; ++it) {
    mbar_wait(empty0 + 8 * stage, phase ^ 1);
    const uint32_t sbase = smem0 + stage * Cfg::STAGE_BYTES;
    const uint32_t fbar = fbar0 + 8 * stage;
    if (role == 0) {
      VENOM_TRACE_EVENT(0, it);
      if (rank == 0) mbar_arrive_expect_tx(full0 + 8 * stage, tx);
      if (do_a)
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
          if constexpr (CG == 2) tma_load_2d_2sm(sbase + mb * Cfg::A_BLOCK, tm_values, fbar, ks * 64, arow + mb * 128 * CG, pol_a);
          else tma_load_2d(sbase + mb * Cfg::A_BLOCK, tm_values, fbar, ks * 64, arow + mb * 128 * CG, pol_a);
        }
      if (do_e)
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
          const uint32_t edst = sbase + Cfg::A_BYTES + Cfg::B_BYTES + mb * Cfg::E_BLOCK;
          const int eblk = eblk0 + mb * CG * p.num_ks + ks;
          if constexpr (CG == 2) tma_load_2d_2sm(edst, tm_e, fbar, 0, eblk, pol_a);
          else tma_load_2d(edst, tm_e, fbar, 0, eblk, pol_a);
        }
      VENOM_TRACE_EVENT(4, it);
    } else if (do_b) {
      if constexpr (kBK) {
        // K-major B ([T][K]): two boxes of BNH token rows × 64 K-elements (K-major SW128)
#pragma unroll
        for (int kc = 0; kc < 2; ++kc) {
          const uint32_t bdst = sbase + Cfg::A_BYTES + kc * (Cfg::BNH * 128);
          if constexpr (CG == 2) tma_load_2d_2sm(bdst, tm_b, fbar, ks * 128 + 64 * kc, col0, pol_b);
          else tma_load_2d(bdst, tm_b, fbar, ks * 128 + 64 * kc, col0, pol_b);
        }
      } else if (b3d) {
        if constexpr (CG == 2) tma_load_3d_2sm(sbase + Cfg::A_BYTES, tm_b, fbar, 0, ks * 128, col0 / 64, pol_b);
        else tma_load_3d(sbase + Cfg::A_BYTES, tm_b, fbar, 0, ks * 128, col0 / 64, pol_b);
      } else {
        const int c = warp - 1;
        if constexpr (CG == 2) tma_load_2d_2sm(sbase + Cfg::A_BYTES + c * Cfg::B_CHUNK, tm_b, fbar, col0 + 64 * c, ks * 128, pol_b);
        else tma_load_2d(sbase + Cfg::A_BYTES + c * Cfg::B_CHUNK, tm_b, fbar, col0 + 64 * c, ks * 128, pol_b);
      }
      VENOM_TRACE_EVENT(7, it);
    }
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1;
    }
    if (++ks == p.num_ks) {
      ks = 0;
      if (++tl < my_tiles) set_tile(tl);
    }
  }
}

template <class Cfg, bool kBF16, bool kContig, bool kCT, bool kBK = false, int kACT = 0>
__global__ void __launch_bounds__(Cfg::NUM_THREADS, 1)
    vnm_spmm_kernel(const __grid_constant__ CUtensorMap tm_values,
                    const __grid_constant__ CUtensorMap tm_b,
                    const __grid_constant__ CUtensorMap tm_e,
                    const __grid_constant__ CUtensorMap tm_c, const SpmmParams p) {
  using namespace ptx;
  constexpr int STAGES = Cfg::STAGES, NB = Cfg::NB, BN = Cfg::BN, CG = Cfg::CG;

  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  // bars: full[STAGES], empty[STAGES], acc_full[2], acc_empty[2]; then the TMEM base word
  const uint32_t full0 = smem_u32(bars);
  const uint32_t empty0 = full0 + 8 * STAGES;
  const uint32_t accf0 = empty0 + 8 * STAGES;
  const uint32_t acce0 = accf0 + 16;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);
  const uint32_t smem0 = smem_u32(smem);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0u;  // position in the CTA pair
  if (threadIdx.x == 0) VENOM_TRACE_EVENT(11, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      // leader's expect_tx + metadata warps of the pair (ablation 256: metadata warps idle)
      mbar_init(full0 + 8 * s, (Cfg::PRE || (p.dbg & 256)) ? 1 : 1 + 4 * CG);
      mbar_init(empty0 + 8 * s, 1);          // (multicast) MMA commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(accf0 + 8 * b, 1);           // (multicast) MMA commit
      mbar_init(acce0 + 8 * b, Cfg::EPI_WARPS * CG);  // epilogue warps of the pair
    }
    fence_mbar_init();
    prefetch_tmap(&tm_values);
    prefetch_tmap(&tm_b);
    if constexpr (Cfg::PRE) prefetch_tmap(&tm_e);
    if (p.tma_c) prefetch_tmap(&tm_c);
  }
  if (warp == Cfg::W_MMA) {
    if constexpr (CG == 2) tmem_alloc_2sm<512>(smem_u32(tmem_base_slot));
    else tmem_alloc<512>(smem_u32(tmem_base_slot));
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  if (threadIdx.x == 0) VENOM_TRACE_EVENT(11, 1);

  const int my_tiles = my_tile_count<CG>(p);
  const int total = my_tiles * p.num_ks;  // k-stage iterations this CTA runs
  const int nrb = static_cast<int>(p.R / p.V);
  const int row_off = 128 * static_cast<int>(rank);

  auto tile_of = [&](int tl, int& m_tile, int& n_tile) { tile_coords<CG>(p, tl, m_tile, n_tile); };
  auto block_of = [&](int m_tile, int b) -> int {
    const int rb = (NB == 1) ? (m_tile * 128 * CG + row_off) / p.V : m_tile * NB + b;
    return rb < nrb ? rb : nrb - 1;  // padding block of a ragged last tile: any valid block
  };

  if (warp < Cfg::P && kContig) {
    if (lane == 0)
      producer_contiguous<Cfg, kBK>(p, &tm_values, &tm_b, &tm_e, my_tiles, smem0, full0, empty0, rank, warp);
  } else if (warp < Cfg::P) {
    // ======================= producers: values tile + gathered B' rows =======================
    // (M > 4; M = 4 runs producer_contiguous.) Stage ops are (block b, chunk c, group q); warp w
    // issues ops [w·OPS_PER_WARP, ...), one per lane: TMA issue is serial within a warp, so the
    // gathers are spread over P warps. A lane's op (b, c, q) is the same in every stage, and the
    // tile / k-stage cursors advance incrementally (no per-stage divisions: the producer's own
    // instruction count sets how fast it refills the ring). With a CTA pair every TMA signals the
    // leader's barrier (cta_group::2 forms).
    const uint64_t pol_a = policy_evict_first();
    const uint64_t pol_b = policy_evict_last();
    int ob[Cfg::LANE_OPS], oc[Cfg::LANE_OPS], oq[Cfg::LANE_OPS];
    bool olive[Cfg::LANE_OPS];
#pragma unroll
    for (int j = 0; j < Cfg::LANE_OPS; ++j) {
      const int o_local = lane + 32 * j;
      const int o = warp * Cfg::OPS_PER_WARP + o_local;
      // the last warp's share is short when P does not divide NOPS
      olive[j] = o_local < Cfg::OPS_PER_WARP && o < Cfg::NOPS;
      ob[j] = olive[j] ? o / (Cfg::NCH * 32) : 0;
      oc[j] = olive[j] ? (o / 32) % Cfg::NCH : 0;
      oq[j] = olive[j] ? o % 32 : 0;
    }
    const uint32_t* cidx = reinterpret_cast<const uint32_t*>(p.column_idx);
    // column_idx words of this lane's ops for the tile the prefetch cursor is in
    auto tile_cptr = [&](int tl, const uint32_t* (&cp)[Cfg::LANE_OPS]) {
      int m_tile, n_tile;
      tile_of(tl, m_tile, n_tile);
#pragma unroll
      for (int j = 0; j < Cfg::LANE_OPS; ++j) cp[j] = cidx + static_cast<int64_t>(block_of(m_tile, ob[j])) * p.G + oq[j];
    };
    // prefetch cursor: kPrefetch k-stages ahead of the issue cursor (the paper's two-level
    // pre-fetching of column-loc)
    int ftl = 0, fks = 0;
    const uint32_t* fcp[Cfg::LANE_OPS];
    if (my_tiles > 0) tile_cptr(0, fcp);
    auto fetch_next = [&](uint32_t (&w)[Cfg::LANE_OPS]) {
      if (ftl >= my_tiles) return;
#pragma unroll
      for (int j = 0; j < Cfg::LANE_OPS; ++j)
        w[j] = (olive[j] && fks * Cfg::KG + oq[j] < p.G) ? __ldg(fcp[j] + fks * Cfg::KG) : 0u;
      if (++fks == p.num_ks) {
        fks = 0;
        if (++ftl < my_tiles) tile_cptr(ftl, fcp);
      }
    };
    uint32_t cw[kPrefetch][Cfg::LANE_OPS];
#pragma unroll
    for (int j = 0; j < kPrefetch; ++j) fetch_next(cw[j]);
    // issue cursor
    int tl = 0, ks = 0, stage = 0;
    uint32_t phase = 0;
    int m_tile = 0, n_tile = 0, col0 = 0, arow = 0;
    auto set_tile = [&]() {
      tile_of(tl, m_tile, n_tile);
      col0 = n_tile * BN + static_cast<int>(rank) * Cfg::BNH;
      arow = m_tile * 128 * CG * Cfg::MB + row_off;
    };
    if (my_tiles > 0) set_tile();
    // ablation flags (p.dbg, tools only): 1 no B loads, 16 no A load, 2048 no metadata load
    const uint32_t tx = CG * ((p.dbg & 16 ? 0 : Cfg::A_BYTES) + (p.dbg & 1 ? 0 : NB * Cfg::B_BYTES) +
                              (p.dbg & 2048 ? 0 : Cfg::E_BYTES));
    // the last k-stage gathers only the groups its MMAs read (8·last_kb of 32)
    const uint32_t tx_last = tx - CG * (p.dbg & 1 ? 0u : static_cast<uint32_t>(NB * Cfg::NCH * 512 * (32 - 8 * p.last_kb)));
    for (int it0 = 0; it0 < total; it0 += kPrefetch) {
#pragma unroll
      for (int jj = 0; jj < kPrefetch; ++jj) {
        const int it = it0 + jj;
        if (it < total) {
          mbar_wait(empty0 + 8 * stage, phase ^ 1);
          const uint32_t sbase = smem0 + stage * Cfg::STAGE_BYTES;
          const uint32_t fbar = (CG == 2) ? mapa_shared(full0 + 8 * stage, 0) : full0 + 8 * stage;
          if (warp == 0 && lane == 0) {
            VENOM_TRACE_EVENT(0, it);
            if (rank == 0) mbar_arrive_expect_tx(full0 + 8 * stage, ks == p.num_ks - 1 ? tx_last : tx);
            if (!(p.dbg & 16)) {
#pragma unroll
              for (int mb = 0; mb < Cfg::MB; ++mb) {
                const int ar = arow + mb * 128 * CG;
                if constexpr (CG == 2) tma_load_2d_2sm(sbase + mb * Cfg::A_BLOCK, &tm_values, fbar, ks * 64, ar, pol_a);
                else tma_load_2d(sbase + mb * Cfg::A_BLOCK, &tm_values, fbar, ks * 64, ar, pol_a);
              }
            }
            if constexpr (Cfg::PRE) if (!(p.dbg & 2048)) {
              // this CTA's 128-row tile(s), k-stage ks: 2 KB block (tile·num_ks + ks) of the
              // pre-ordered metadata, one TMA row
#pragma unroll
              for (int mb = 0; mb < Cfg::MB; ++mb) {
                const uint32_t edst = sbase + Cfg::A_BYTES + NB * Cfg::B_BYTES + mb * Cfg::E_BLOCK;
                const int eblk = ((m_tile * Cfg::MB + mb) * CG + static_cast<int>(rank)) * p.num_ks + ks;
                if constexpr (CG == 2) {
                  tma_load_2d_2sm(edst, &tm_e, fbar, 0, eblk, pol_a);
                } else if constexpr (Cfg::M64) {
                  // the M = 64 lane order: 16-lane group x + 4y of the block lands at 2x + y (a
                  // 4-D map [block][x: 4, 256 B apart][y: 2, 1 KB apart][256 B], box order y, x)
                  if (p.e4d) {
                    tma_load_4d(edst, &tm_e, fbar, 0, 0, 0, eblk, pol_a);
                  } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                      tma_load_2d(edst + 256 * (2 * (j & 3) + (j >> 2)), &tm_e, fbar, 0, 8 * eblk + j, pol_a);
                  }
                } else {
                  tma_load_2d(edst, &tm_e, fbar, 0, eblk, pol_a);
                }
              }
            }
          }
          if (!(p.dbg & 1)) {
#pragma unroll
            for (int j = 0; j < Cfg::LANE_OPS; ++j) {
              if (!olive[j] || (ks == p.num_ks - 1 && oq[j] >= 8 * p.last_kb)) continue;
              const int gg = ks * Cfg::KG + oq[j];
              const uint32_t w = cw[jj][j];
              int r[4];
#pragma unroll
              for (int t = 0; t < 4; ++t)
                r[t] = (gg < p.G) ? gg * p.M + static_cast<int>((w >> (8 * t)) & 0xFF)
                                  : static_cast<int>(p.K);  // past the last row: zero fill
              const uint32_t bdst = sbase + Cfg::A_BYTES + ob[j] * Cfg::B_BYTES + oc[j] * Cfg::B_CHUNK + oq[j] * 512;
              if constexpr (CG == 2)
                tma_gather4_2sm(bdst, &tm_b, fbar, col0 + 64 * oc[j], r[0], r[1], r[2], r[3], pol_b);
              else
                tma_gather4(bdst, &tm_b, fbar, col0 + 64 * oc[j], r[0], r[1], r[2], r[3], pol_b);
            }
          }
          __syncwarp();
          if (warp == 0 && lane == 0) VENOM_TRACE_EVENT(4, it);
          fetch_next(cw[jj]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
          if (++ks == p.num_ks) {
            ks = 0;
            if (++tl < my_tiles) set_tile();
          }
        }
      }
    }
  } else if (warp == Cfg::W_MMA) {
    if (rank == 0) mma_role<Cfg, kBF16, CG, kBK>(p, my_tiles, tmem_base, smem0, full0, empty0, accf0, acce0, lane);
  } else if (warp >= Cfg::W_EPI && warp < Cfg::W_EPI + Cfg::EPI_WARPS) {
    const uint32_t slot = smem0 + STAGES * Cfg::STAGE_BYTES + Cfg::BAR_BYTES + (warp - Cfg::W_EPI) * Cfg::EPI_STAGE_BYTES;
    if constexpr (Cfg::MB == 2) epilogue_role_mb2<Cfg, kBF16, CG>(p, my_tiles, tmem_base, accf0, acce0, warp, lane, slot);
    else epilogue_role<Cfg, kBF16, CG, kCT, kACT>(p, my_tiles, tmem_base, accf0, acce0, warp, lane, slot,
                                                   p.tma_c ? &tm_c : nullptr);
  } else if constexpr (!Cfg::PRE) {
    // ======================= metadata: canonical nibbles -> TMEM (tensor-core layout) ==========
    // TMEM lane L of one K=32 MMA holds rows m = (L&7) + 16(L>>4) (low half-word) and m+8 (high
    // half-word), each for K-half k1 = (L>>3)&1: the 16 bits of groups 4·k1 .. 4·k1+3. The warp
    // writes its lane quarter (warp % 4) with tcgen05.st: no shared memory, no proxy fence.
    const int qd = warp & 3;
    // TMEM lane 32·qd + lane holds the M = 128 order's lane L; M64 interleaves the two 64-row
    // blocks' halves (physical lane bits [6:5] = L bits [5:4], bit 4 = L bit 6)
    const int Pl = 32 * qd + lane;
    const int L = Cfg::M64 ? (Pl & 15) + 16 * ((Pl >> 5) & 3) + 64 * ((Pl >> 4) & 1) : Pl;
    const int total_meta = (p.dbg & 256) ? 0 : total;
    const int m_a = (L & 7) + 16 * (L >> 4);
    const int k1 = (L >> 3) & 1;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(32 * qd) << 16);
    uint32_t wa[kPrefetch][4], wb[kPrefetch][4];
    auto fetch = [&](int it, uint32_t (&xa)[4], uint32_t (&xb)[4]) {
      if (it >= total) return;
      int m_tile, n_tile;
      tile_of(it / p.num_ks, m_tile, n_tile);
      const int ks = it % p.num_ks;
      const int64_t ra = static_cast<int64_t>(m_tile) * 128 * CG + row_off + m_a;
      if (p.dbg & 32) {  // ablation 32: no metadata global loads
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) xa[kb] = xb[kb] = 0x44444444u;
        return;
      }
      load_meta_stage(p, ra, ks, xa);
      load_meta_stage(p, ra + 8, ks, xb);
    };
#pragma unroll
    for (int j = 0; j < kPrefetch; ++j) fetch(j, wa[j], wb[j]);
    for (int it0 = 0; it0 < total_meta; it0 += kPrefetch) {
#pragma unroll
      for (int j = 0; j < kPrefetch; ++j) {
        const int it = it0 + j;
        if (it < total) {
          const int stage = it % STAGES;
          uint32_t o[4];
#pragma unroll
          for (int kb = 0; kb < 4; ++kb)
            o[kb] = ((wa[j][kb] >> (16 * k1)) & 0xFFFFu) | (((wb[j][kb] >> (16 * k1)) & 0xFFFFu) << 16);
          mbar_wait(empty0 + 8 * stage, ((it / STAGES) & 1) ^ 1);
          if (!(p.dbg & 8)) {  // ablation 8: no metadata stores
            tmem_st_32x32b_x4(lane_base + Cfg::E_COL + 4 * stage, o[0], o[1], o[2], o[3]);
            tmem_st_wait();
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (qd == 0) VENOM_TRACE_EVENT(3, it);
            if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(full0 + 8 * stage, 0));
            else mbar_arrive(full0 + 8 * stage);
          }
          fetch(it + kPrefetch, wa[j], wb[j]);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  if (threadIdx.x == 0) VENOM_TRACE_EVENT(11, 2);
  if (warp == Cfg::W_MMA) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_2sm<512>(tmem_base);
    else tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace venom
