/*
 * venom.h — C ABI of libvenom: the B200 (sm_100a) hot path of VENOM / Spatha (arXiv 2310.02065).
 *
 * The three calls are the operations the paper defines:
 *   venom_compress   dense weight -> V:N:M (values, metadata, column_idx)   PAPER.md:187-195 (§3)
 *   venom_spmm       C = A_vnm · B (+ bias) on the compressed operand       PAPER.md:197-263 (§4),
 *                    bias as in spatha.spmm(values, columns, metadata, input, bias)
 *   venom_decompress V:N:M -> dense (inverse of Fig 3; verification / dense-baseline operand)
 *
 * Notation: C[R×T] = A[R×K] · B[K×T]. A is cut into V-row × M-column blocks;
 * each block keeps 4 columns (column_idx) and each row keeps 2 of those 4 (values + 2-bit
 * m-indices packed as metadata nibbles). N is fixed at 2 (fp16/bf16 sparse tensor cores are 2:4,
 * PAPER.md:144). G = K/M groups per row.
 *
 * Canonical byte layouts (what "bit-exact" is checked on; readings #7-#10):
 *   values     dtype[R][G][2]            the two kept weights of (row, group), original bits,
 *                                        ordered by ascending m-index. Row-major R × (2G).
 *   metadata   uint8[R][ceil(G/2)]       nibble(r,g) = p0 | p1<<2 with p0 < p1 in [0,4) the
 *                                        m-indices; byte h of row r = nib(r,2h) | nib(r,2h+1)<<4;
 *                                        an odd G leaves the last high nibble 0.
 *   column_idx uint8[R/V][G][4]          the block's 4 selected columns, block-relative in [0,M),
 *                                        strictly ascending.
 *
 * Conventions
 *   - Every data pointer is a DEVICE pointer owned by the caller. The library never allocates,
 *     never synchronises `stream`, and keeps no mutable global state (thread-safe; the only
 *     process-wide state is the lazily resolved driver entry point cuTensorMapEncodeTiled).
 *   - Argument, shape and architecture errors are returned synchronously and nothing is launched.
 *   - Data-dependent errors (non-finite input, corrupt metadata) are reported on the device by
 *     atomicMax()-ing a venom_status_t into *dev_status (nullable: NULL skips those checks); the
 *     outputs are undefined when that word becomes non-zero. The caller zeroes it.
 *   - Buffers must stay valid until the stream work completes.
 */
#ifndef VENOM_H_
#define VENOM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  VENOM_OK = 0,
  VENOM_ERR_INVALID_ARGUMENT = 1,    /* null pointer, ld < cols, misalignment, bad sizes          */
  VENOM_ERR_NON_DIVISIBLE_ROWS = 2,  /* V does not divide R              */
  VENOM_ERR_NON_DIVISIBLE_COLS = 3,  /* M does not divide K              */
  VENOM_ERR_UNSUPPORTED_PATTERN = 4, /* N != 2, M < 4, M > 256; spmm: V not in {32,64} ∪ 128ℕ,
                                        G % 4 != 0 without the padded execution form            */
  VENOM_ERR_UNSUPPORTED_DTYPE = 5,
  VENOM_ERR_NON_FINITE = 6,          /* device-reported (finite inputs only)         */
  VENOM_ERR_CORRUPT_METADATA = 7,    /* device-reported: m-indices not ascending, column_idx not
                                        strictly ascending or >= M                  */
  VENOM_ERR_ARCH = 8,                /* current device is not sm_100                             */
  VENOM_ERR_CUDA = 9,                /* launch / driver error                                    */
  VENOM_ERR_INVALID_MASK = 10        /* device-reported by venom_compress_masked: the mask is not
                                        V:N:M (> 4 columns in a V×M block or > 2 kept entries in a
                                        row of a group)                                         */
} venom_status_t;

typedef enum { VENOM_F16 = 0, VENOM_BF16 = 1 } venom_dtype_t;

/* V:N:M pattern. n must be 2. */
typedef struct {
  int32_t v, n, m;
} venom_format_t;

/* Opaque CUDA stream (cudaStream_t); 0 = legacy default stream. */
typedef void* venom_stream_t;

/* Sizes of the three compressed arrays for an R×K matrix (PAPER.md:194-195:
 * values R×K/M×2, column-loc R/V×K/M×4). Host-only, no device access. */
venom_status_t venom_compressed_sizes(int64_t R, int64_t K, venom_format_t f,
                                      int64_t* values_elems,      /* R*(K/M)*2        */
                                      int64_t* metadata_bytes,    /* R*ceil((K/M)/2)  */
                                      int64_t* column_idx_bytes); /* (R/V)*(K/M)*4    */

/*
 * Magnitude V:N:M compression: per V×M block, the 4 columns with the largest
 * L1 mass over the block's V rows (fp64, ascending rows; ties -> lower index), then per row the 2
 * largest |w| among those 4 (ties -> lower m-index). Bit-identical to the CPU oracle.
 *   A          dtype[R][lda], row-major, lda >= K
 *   values, metadata, column_idx   outputs in the canonical layouts above
 * Requirements: any V >= 1 with V | R, 4 <= M <= 256 with M | K, n == 2. No alignment demands.
 */
venom_status_t venom_compress(const void* A, int64_t R, int64_t K, int64_t lda,
                              venom_dtype_t dt, venom_format_t f,
                              void* values, uint8_t* metadata, uint8_t* column_idx,
                              int32_t* dev_status, venom_stream_t stream);

/*
 * Masked V:N:M compression (reading #20): the kept entries come from
 * an external mask (e.g. a second-order pruner) instead of the magnitude rule.
 *   mask   uint8[R][ldm] row-major, ldm >= K; non-zero keeps A[i][k]. It must be V:N:M: at most 4
 *          columns of each V×M block hold kept entries and at most 2 per row of each group, else
 *          VENOM_ERR_INVALID_MASK is reported through dev_status (outputs undefined).
 *   column_idx: the block's kept columns, completed to 4 with the lowest-index free columns,
 *   ascending; per row the kept m-indices completed to 2 with the lowest free ones; kept entries
 *   store A's raw bits, filled ones +0.0 — so decompress(result) == A∘mask bit for bit.
 * Requirements: as venom_compress. Bit-identical to the CPU oracle. Offline (once per weight).
 */
venom_status_t venom_compress_masked(const void* A, int64_t R, int64_t K, int64_t lda,
                                     const uint8_t* mask, int64_t ldm, venom_dtype_t dt,
                                     venom_format_t f, void* values, uint8_t* metadata,
                                     uint8_t* column_idx, int32_t* dev_status, venom_stream_t stream);

/*
 * Energy of a pruned matrix: energy = Σ|kept| / Σ|dense|, both in fp64.
 *   A        dtype[R][lda], the dense matrix w*
 *   values   dtype[n_values], the kept values (e.g. a compressed operand's values array; filled
 *            +0.0 entries add nothing)
 *   out      DEVICE double[3]: {Σ|kept|, Σ|dense|, energy}; energy = 1 when Σ|dense| = 0.
 * The sums are fp64 over per-CTA partials (order differs from the oracle's: equal to ≤ 1e-12
 * relative). Writes `out` on the stream; no host synchronisation.
 */
venom_status_t venom_energy(const void* A, int64_t R, int64_t K, int64_t lda, const void* values,
                            int64_t n_values, venom_dtype_t dt, double* out, venom_stream_t stream);

/*
 * Inverse of the format: A_out[i][g*M + column_idx[i/V][g][p]] = value with
 * m-index p; every other element is +0.0. A_out is dtype[R][lda], lda >= K.
 */
venom_status_t venom_decompress(const void* values, const uint8_t* metadata,
                                const uint8_t* column_idx, int64_t R, int64_t K,
                                venom_dtype_t dt, venom_format_t f,
                                void* A_out, int64_t lda,
                                int32_t* dev_status, venom_stream_t stream);

/*
 * SpMM  C = decompress(A) · B (+ bias), fp32 accumulation, round-to-nearest-even to dtype
 * (PAPER.md:207-209 mapping onto 2:4 sparse tensor cores; reading #13).
 *   B     dtype[K][ldb] row-major (T contiguous; for a Linear layer, the feature-major activation)
 *   C     dtype[R][ldc] row-major
 *   bias  nullable dtype[R], added in fp32 before rounding
 * Requirements (else VENOM_ERR_UNSUPPORTED_PATTERN / INVALID_ARGUMENT):
 *   V | R; M in [4,256], M | K; T % 8 == 0, ldb % 8 == 0, ldc % 8 == 0, ldb >= T, ldc >= T;
 *   values/B/C 16-byte aligned, column_idx 4-byte aligned; metadata 16-byte aligned whenever it
 *   is read (no opts->metadata_tc); dense-K additionally needs column_idx 16-byte aligned (a
 *   misaligned view returns VENOM_ERR_INVALID_ARGUMENT instead of faulting on the device);
 *   and at least one strategy applies:
 *     gather : (V in {32, 64} or V % 128 == 0 or M == 4) and G = K/M with G % 4 == 0, or any G
 *              with opts->metadata_tc and opts->values_padded (venom_pad_values)
 *     dense-K: M in {4, 8, 16, 32} and G % 4 == 0 (any V)
 *   The library picks the faster applicable strategy (see venom_spmm_opts_t).
 * R == 0 or T == 0: nothing to compute, VENOM_OK with no launch (leading dimensions are not checked).
 * K == 0: C = bias broadcast (or 0).
 * metadata may be NULL when opts->metadata_tc is given; column_idx may be NULL when M == 4 (it is the
 * identity and never read).
 * Metadata validity is NOT checked here (use venom_decompress with dev_status to validate);
 * malformed metadata gives undefined values, never out-of-bounds accesses.
 */
venom_status_t venom_spmm(const void* values, const uint8_t* metadata, const uint8_t* column_idx,
                          int64_t R, int64_t K, venom_format_t f,
                          const void* B, int64_t T, int64_t ldb,
                          void* C, int64_t ldc,
                          const void* bias,
                          venom_dtype_t dt, venom_stream_t stream);

/*
 * Re-encode a V:N:M matrix with M % 4 == 0 as the SAME matrix in V:2:4 form over the original K
 * (reading #18 "dense-K"): a group of M columns keeps 2 values, so each aligned 4-column
 * subgroup holds at most 2 — the V:N:M pattern is a 2:4 pattern. Per row and 4-column subgroup:
 * two kept values -> (a, b) at their positions; one kept value v at position i -> (v, 0) at (0, 1)
 * if i == 0 else (0, v) at (0, i); none -> zeros at (0, 1) (inserted zeros are +0.0). Outputs are
 * the canonical arrays of format {v, 2, 4}: values_out dtype[R][K/4][2], metadata_out
 * uint8[R][ceil(K/8)], column_idx_out uint8[R/V][K/4][4] (all {0,1,2,3}). decompress(out) equals
 * decompress(in) bit for bit, so venom_spmm on the output computes the same product — on B200 the
 * M = 4 SpMM (dense B tiles, CTA pairs, no gathers) is the faster execution for small V·M.
 * Corrupt metadata is reported through *dev_status (nullable).
 */
venom_status_t venom_expand_2to4(const void* values, const uint8_t* metadata,
                                const uint8_t* column_idx, int64_t R, int64_t K,
                                venom_dtype_t dt, venom_format_t f,
                                void* values_out, uint8_t* metadata_out, uint8_t* column_idx_out,
                                int32_t* dev_status, venom_stream_t stream);

/*
 * Fused compression + execution-form preparation (one pass over A): writes everything
 * venom_compress writes (values, metadata, column_idx: the canonical V:N:M arrays, bit-identical to
 * venom_compress) and, for the same matrix, the V:2:4 re-encoding's values (as venom_expand_2to4:
 * values_2to4 dtype[R][K/4][2]) and its metadata in tensor-core order (as venom_order_metadata on
 * the re-encoding: metadata_2to4_tc, venom_metadata_tc_bytes(R, K, {v, 2, 4}) bytes). The pair
 * (values_2to4, metadata_2to4_tc) is a complete venom_spmm operand of format {v, 2, 4}: pass it with
 * opts.metadata_tc and NULL metadata / column_idx. Requires M % 8 == 0, M | 128, V % 16 == 0,
 * V <= 256, K % 16 == 0 (else VENOM_ERR_UNSUPPORTED_PATTERN); values_2to4 / metadata_2to4_tc
 * 16-byte aligned. Non-finite inputs are reported through *dev_status like venom_compress.
 */
venom_status_t venom_compress_2to4(const void* A, int64_t R, int64_t K, int64_t lda,
                                  venom_dtype_t dt, venom_format_t f,
                                  void* values, uint8_t* metadata, uint8_t* column_idx,
                                  void* values_2to4, uint8_t* metadata_2to4_tc,
                                  int32_t* dev_status, venom_stream_t stream);

/*
 * Planner hint: 1 when venom_spmm over venom_expand_2to4's output is expected to run faster on
 * B200 than venom_spmm on the V:N:M operand itself for this shape (R, K, T, f), and the fused
 * venom_compress_2to4 applies; 0 otherwise, including for any invalid format. Pure host function,
 * no device access.
 */
int32_t venom_prefer_2to4(int64_t R, int64_t K, int64_t T, venom_format_t f);

/* Optional overrides for venom_spmm (benchmarking / tuning / ablation). Zero = library default.
 *   tile_t    output columns per CTA tile (64, 128, 192 or 256; availability depends on strategy;
 *             240 = 512 × 240 CTA-pair tiles with two accumulators per CTA, M == 4 operands with
 *             metadata_tc only. 0 = the planner's choice)
 *   stages    reserved: must be 0 (the pipeline depth is fixed per tile configuration; any other
 *             value returns VENOM_ERR_INVALID_ARGUMENT)
 *   max_ctas  persistent grid cap (0 = #SMs)
 *   strategy  VENOM_STRATEGY_AUTO: the gathered/contiguous kernel wherever it applies, else
 *             DENSE_K; GATHER: the paper's mapping (gather the 4 selected
 *             B rows per group through column_idx, 2:4 MMA over K' = 4K/M); DENSE_K: expand the
 *             V:N:M operand on the fly to 2:4 over the original K and use dense B tiles (requires
 *             M in {4,8,16,32}, G % 4 == 0). Both return the same product. */
enum { VENOM_STRATEGY_AUTO = 0, VENOM_STRATEGY_GATHER = 1, VENOM_STRATEGY_DENSE_K = 2 };
typedef struct {
  int32_t tile_t;
  int32_t stages;
  int32_t max_ctas;
  int32_t strategy;
  int32_t cta_pair;  /* 1 = one CTA per 128-row tile, 2 = CTA pair (cta_group::2, 256-row tiles,
                        B split between the pair's shared memories); 0 = library default; any
                        other value returns VENOM_ERR_INVALID_ARGUMENT */
  const uint8_t* metadata_tc;  /* nullable DEVICE pointer: the operand's metadata in tensor-core
                        order (venom_order_metadata). When set, the gathered kernel loads it with
                        TMA and copies it to TMEM with tcgen05.cp instead of permuting `metadata`
                        on the fly; `metadata` is then not read. Must be 16-byte aligned. */
  int32_t c_transposed;  /* 1: C is written token-major, C^T = dtype[T][ldc] with ldc >= R
                        (element (r, t) at C[t*ldc + r]; ldc % 8 == 0) — the layout attention and
                        a PyTorch [tokens, features] activation use. Gathered / contiguous kernel
                        with one 128-row accumulator per CTA only (tile_t 240 and DENSE_K are
                        rejected with VENOM_ERR_INVALID_ARGUMENT). 0: row-major C (default). */
  int32_t b_kmajor;    /* 1: B is given K-major (token-major activations, the PyTorch [tokens,
                        features] layout): dtype[T][ldb] with ldb >= K, ldb % 8 == 0. M = 4 operands
                        (plain 2:4 or the V:2:4 form of venom_compress_2to4) read it natively, one
                        accumulator per CTA (tile_t 240 and DENSE_K rejected). M > 4 (gathered)
                        operands need b_scratch: B is first transposed into it (K % 8 == 0). With
                        c_transposed this is Y = X·Wᵀ on [T, K] activations. 0: B row-major
                        dtype[K][ldb] (default). */
  int32_t activation;  /* 1: GELU (erf form, x·Φ(x)) applied after the bias in fp32 before the
                        rounding; 2: GELU, tanh form (0.5·x·(1 + tanh(√(2/π)·(x + 0.044715·x³))), the
                        original BERT's and GPT-2/3's; hardware tanh.approx, max relative error 2^-11,
                        and 25% cheaper on FFN1-shaped layers than the erf form). Row-major B and C,
                        gathered / contiguous kernel with one accumulator per CTA (else
                        VENOM_ERR_INVALID_ARGUMENT). Not applied when K == 0. 0: none (default). */
  int32_t group_n;     /* tile order: column tiles are taken in groups of group_n, the row tiles
                        outer within a group (1 = all row tiles of one column band first). 0: the
                        library default (1). */
  void* const* c_peers;  /* fused all-gather: host array of n_peers
                        DEVICE pointers (e.g. the other ranks' full output buffers mapped peer-to-peer,
                        each already offset to where this rank's slice starts; 16-byte aligned, same
                        ldc as C). Every element of C is also stored there by the epilogue, so the
                        SpMM's output lands in all ranks' buffers without a separate collective. The
                        caller orders the ranks' kernels with the consumers (e.g. a barrier). Gathered
                        / contiguous kernel, one accumulator per CTA (dense-K and tile_t 240 return
                        VENOM_ERR_INVALID_ARGUMENT). NULL / 0: none. */
  int32_t n_peers;     /* 0..8 */
  const void* values_padded;  /* nullable DEVICE pointer: the operand's values with each row padded
                        to a multiple of 4 groups (venom_pad_values). Needed, with metadata_tc, when
                        G = K/M is not a multiple of 4: the values' TMA map needs a 16-byte row
                        pitch (4·G bytes otherwise). Ignored when G % 4 == 0. 16-byte aligned. */
  void* b_scratch;     /* nullable DEVICE pointer: dtype[K][T] caller-owned scratch (16-byte aligned)
                        for b_kmajor with an M > 4 operand (the transposed B the gathered path reads). */
} venom_spmm_opts_t;

venom_status_t venom_spmm_ex(const void* values, const uint8_t* metadata, const uint8_t* column_idx,
                             int64_t R, int64_t K, venom_format_t f,
                             const void* B, int64_t T, int64_t ldb,
                             void* C, int64_t ldc, const void* bias,
                             venom_dtype_t dt, const venom_spmm_opts_t* opts,
                             venom_stream_t stream);

/*
 * Tensor-core order of the metadata — the paper's "storage order" idea (§4.1:
 * m-indices are stored in the order the hardware consumes them) re-targeted to tcgen05: the same
 * nibbles as `metadata`, permuted so that the block for one 128-row tile and one k-stage of 32
 * groups is the 2 KB TMEM image the sparse MMA reads. Layout:
 * uint32[ceil(R/128)][ceil(G/32)][128 lanes][4 MMAs], G = K/M; lane L, MMA kb holds the 16 bits of
 * groups 32·ks + 8·kb + 4·((L>>3)&1) .. +3 of row (L&7) + 16·(L>>4) (low half) and of that row + 8
 * (high half); rows >= R and groups >= G are filled with the zero-value code 0x4 (m-indices 0,1).
 * venom_metadata_tc_bytes returns the size in bytes (-1 for an invalid format). Any G (a partial
 * last 4-group word is completed with 0x4 nibbles). metadata_tc: caller-owned device buffer,
 * 16-byte aligned. Metadata validity is not checked (use venom_decompress with dev_status).
 */
int64_t venom_metadata_tc_bytes(int64_t R, int64_t K, venom_format_t f);
venom_status_t venom_order_metadata(const uint8_t* metadata, int64_t R, int64_t K, venom_format_t f,
                                    uint8_t* metadata_tc, venom_stream_t stream);

/*
 * Values with a padded row pitch — the execution form for G = K/M not a multiple of 4 (the K'
 * tail the paper's K sweeps reach): values_padded = dtype[R][G4][2] with
 * G4 = ceil(G/4)·4; groups >= G are +0.0 (they meet the 0x4 metadata of venom_order_metadata and
 * zero-filled rows of B, so they add nothing). venom_values_padded_bytes returns R·G4·4 (-1 for
 * an invalid format). values: 4-byte aligned; values_padded: caller-owned, 16-byte aligned.
 */
int64_t venom_values_padded_bytes(int64_t R, int64_t K, venom_format_t f);
venom_status_t venom_pad_values(const void* values, int64_t R, int64_t K, venom_format_t f,
                                void* values_padded, venom_stream_t stream);

/* Number of kernels venom_spmm / venom_compress / venom_decompress launch per call (1 each). */
int32_t venom_kernels_per_call(void);

const char* venom_status_string(venom_status_t s);
const char* venom_version(void);

#ifdef __cplusplus
}
#endif
#endif /* VENOM_H_ */
