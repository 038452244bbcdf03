/*
 * venom_oracle.c — CPU ORACLE for the V:N:M hot path (VENOM / Spatha, arXiv 2310.02065).
 *
 * TEST INFRASTRUCTURE ONLY. This file is the plain, slow, obviously-correct reference that the
 * CUDA path is checked against. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The product library (paper_2310_02065_b200/csrc) shares no
 * code, header, table or constant with it, and never calls it.
 *
 * Everything here is scalar loops in the order the paper states, with fp64 arithmetic.
 * "PAPER.md:L" cites a line of the paper text; "§8(c)#n" cites a reading listed in DESIGN.md.
 *
 * Pins (tests/test_oracle_*.py, run with -m "not gpu"):
 *   - compress: worked examples P1-P4 (tests/golden/), brute force over all C(M,4) column subsets
 *     and all 6 row pairs, M=4 == textbook 2:4 magnitude pruning, shape identities PAPER.md:194-195.
 *   - decompress: worked example P5, roundtrip invariants.
 *   - spmm_compressed: == gemm_dense(decompress(.)) (independent formulation), B = I closed form,
 *     numpy float64 matmul on the decompressed matrix (library routine), linearity.
 *   - f16/bf16 decoding: exhaustive over all 65536 bit patterns vs numpy / torch.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Status codes (values chosen to match the DESIGN.md error table; defined here independently). */
enum {
  ORC_OK = 0,
  ORC_INVALID_ARGUMENT = 1,
  ORC_NON_DIVISIBLE_ROWS = 2,
  ORC_NON_DIVISIBLE_COLS = 3,
  ORC_UNSUPPORTED_PATTERN = 4,
  ORC_UNSUPPORTED_DTYPE = 5,
  ORC_NON_FINITE = 6,
  ORC_CORRUPT_METADATA = 7,
  ORC_INVALID_MASK = 10
};

/* dtype: 0 = IEEE binary16 (fp16, "half precision"), 1 = bfloat16. */

/* Decode one 16-bit pattern to a double, straight from the format definitions. */
double oracle_decode(uint16_t bits, int dtype) {
  int sign = (bits >> 15) & 1;
  double v;
  if (dtype == 0) {                 /* fp16: 1 sign, 5 exponent (bias 15), 10 fraction */
    int e = (bits >> 10) & 0x1F;
    int f = bits & 0x3FF;
    if (e == 0)        v = ldexp((double)f, -24);                 /* subnormal: f * 2^-14 * 2^-10 */
    else if (e == 31)  v = (f == 0) ? INFINITY : NAN;
    else               v = ldexp((double)(1024 + f), e - 25);     /* (1 + f/2^10) * 2^(e-15) */
  } else {                          /* bf16: 1 sign, 8 exponent (bias 127), 7 fraction */
    int e = (bits >> 7) & 0xFF;
    int f = bits & 0x7F;
    if (e == 0)        v = ldexp((double)f, -133);                /* f * 2^-126 * 2^-7 */
    else if (e == 255) v = (f == 0) ? INFINITY : NAN;
    else               v = ldexp((double)(128 + f), e - 134);     /* (1 + f/2^7) * 2^(e-127) */
  }
  return sign ? -v : v;
}

/* Validate (V, N, M) against (R, K). SPEC.md:58-66; M <= 256 because column_idx is u8 (§8(c)#10). */
int oracle_validate(int64_t R, int64_t K, int V, int N, int M) {
  if (R < 0 || K < 0 || V < 1) return ORC_INVALID_ARGUMENT;
  if (N != 2 || M < 4 || M > 256) return ORC_UNSUPPORTED_PATTERN;
  if (R % V != 0) return ORC_NON_DIVISIBLE_ROWS;
  if (K % M != 0) return ORC_NON_DIVISIBLE_COLS;
  return ORC_OK;
}

/*
 * Magnitude V:N:M compression, PAPER.md:187-189 (§3, Fig 2 ④) and PAPER.md:192-195 (Fig 3):
 *   "partitioning the original dense matrix in blocks of V×M elements. Then, the four most
 *    significant columns of each block are selected (vector-wise pruning), and for each row of
 *    four elements in a block, the two most meaningful weights are kept (2:4 pruning)."
 * Readings: column significance = L1 norm over the block's V rows, summed in fp64 in
 * ascending row order (#1, #2); two-stage greedy as written (#3); row weight significance = |w|
 * (#4); ties -> lower index (#5, #6); column_idx and m-indices stored ascending (#7); nibble
 * p0 | p1 << 2, two groups per byte, low nibble first, packed per row (#8).
 *
 * A:          R x K, row stride lda (elements), raw 16-bit patterns.
 * values:     R x (K/M) x 2 raw patterns (the kept weights, original bits; -0.0 stays -0.0).
 * metadata:   R x ceil((K/M)/2) bytes.
 * column_idx: (R/V) x (K/M) x 4 bytes, block-relative, strictly ascending.
 */
int oracle_compress(const uint16_t* A, int64_t R, int64_t K, int64_t lda, int dtype,
                    int V, int N, int M,
                    uint16_t* values, uint8_t* metadata, uint8_t* column_idx) {
  int st = oracle_validate(R, K, V, N, M);
  if (st != ORC_OK) return st;
  if (dtype != 0 && dtype != 1) return ORC_UNSUPPORTED_DTYPE;
  if (lda < K) return ORC_INVALID_ARGUMENT;

  /* Finite inputs only (§8(c)#15). */
  for (int64_t i = 0; i < R; ++i)
    for (int64_t k = 0; k < K; ++k)
      if (!isfinite(oracle_decode(A[i * lda + k], dtype))) return ORC_NON_FINITE;

  const int64_t G = K / M;                  /* groups (block columns) per row */
  const int64_t meta_row = (G + 1) / 2;     /* bytes of metadata per row */
  memset(metadata, 0, (size_t)(R * meta_row));

  double* s = (double*)malloc(sizeof(double) * (size_t)M);
  int* taken = (int*)malloc(sizeof(int) * (size_t)M);
  if (!s || !taken) { free(s); free(taken); return ORC_INVALID_ARGUMENT; }

  for (int64_t rb = 0; rb < R / V; ++rb) {
    for (int64_t g = 0; g < G; ++g) {
      /* Step 1: column scores s_j = sum_{i in block, ascending} |A[i][g*M + j]|, fp64. */
      for (int j = 0; j < M; ++j) {
        s[j] = 0.0;
        for (int64_t i = rb * V; i < rb * V + V; ++i)
          s[j] += fabs(oracle_decode(A[i * lda + g * M + j], dtype));
      }
      /* Step 2: the four most significant columns: repeatedly take the largest score not yet
       * taken; a strictly larger score is needed to displace a lower index (ties -> lower). */
      int c[4];
      for (int j = 0; j < M; ++j) taken[j] = 0;
      for (int t = 0; t < 4; ++t) {
        int best = -1;
        for (int j = 0; j < M; ++j) {
          if (taken[j]) continue;
          if (best < 0 || s[j] > s[best]) best = j;
        }
        taken[best] = 1;
        c[t] = best;
      }
      /* sort ascending (insertion sort of 4) */
      for (int a = 1; a < 4; ++a) {
        int x = c[a], b = a - 1;
        while (b >= 0 && c[b] > x) { c[b + 1] = c[b]; --b; }
        c[b + 1] = x;
      }
      for (int t = 0; t < 4; ++t) column_idx[(rb * G + g) * 4 + t] = (uint8_t)c[t];

      /* Step 3: per row, keep the two largest |w| among the 4 selected columns. */
      for (int64_t i = rb * V; i < rb * V + V; ++i) {
        double mag[4];
        for (int t = 0; t < 4; ++t) mag[t] = fabs(oracle_decode(A[i * lda + g * M + c[t]], dtype));
        int p[2];
        int used[4] = {0, 0, 0, 0};
        for (int q = 0; q < 2; ++q) {
          int best = -1;
          for (int t = 0; t < 4; ++t) {
            if (used[t]) continue;
            if (best < 0 || mag[t] > mag[best]) best = t;
          }
          used[best] = 1;
          p[q] = best;
        }
        if (p[0] > p[1]) { int x = p[0]; p[0] = p[1]; p[1] = x; }
        values[(i * G + g) * 2 + 0] = A[i * lda + g * M + c[p[0]]];
        values[(i * G + g) * 2 + 1] = A[i * lda + g * M + c[p[1]]];
        uint8_t nib = (uint8_t)(p[0] | (p[1] << 2));
        metadata[i * meta_row + g / 2] |= (uint8_t)(nib << (4 * (g % 2)));
      }
    }
  }
  free(s);
  free(taken);
  return ORC_OK;
}

/*
 * Masked compression (reading #20). The kept entries come from an
 * external mask (mask[i*ldm + k] != 0 keeps A[i][k]), e.g. one chosen by the paper's second-order
 * pruner, instead of the magnitude rule of PAPER.md:188. The mask must itself be
 * V:N:M: per V x M block at most 4 distinct columns hold kept entries ("4 columns
 * ... are selected"), and per row at most N = 2 kept entries per group.
 *   1. S = the block's columns with a kept entry in any of its V rows, in ascending order; if
 *      |S| < 4 it is completed with the lowest-index columns not in S (reading #6's fill rule) and
 *      the four are stored ascending as column_idx.
 *   2. Per row, P = the m-indices t with mask[i][g*M + c_t] != 0, ascending; if |P| < 2 it is
 *      completed with the lowest free m-indices. Kept entries store A's raw bits, filled ones +0.0
 *      (bits 0x0000): the operand is exactly A∘mask.
 * Returns ORC_INVALID_MASK if some block has |S| > 4 or some row-group |P| > 2.
 */
int oracle_compress_masked(const uint16_t* A, int64_t R, int64_t K, int64_t lda, int dtype,
                           const uint8_t* mask, int64_t ldm, int V, int N, int M,
                           uint16_t* values, uint8_t* metadata, uint8_t* column_idx) {
  int st = oracle_validate(R, K, V, N, M);
  if (st != ORC_OK) return st;
  if (dtype != 0 && dtype != 1) return ORC_UNSUPPORTED_DTYPE;
  if (lda < K || ldm < K) return ORC_INVALID_ARGUMENT;
  for (int64_t i = 0; i < R; ++i)
    for (int64_t k = 0; k < K; ++k)
      if (!isfinite(oracle_decode(A[i * lda + k], dtype))) return ORC_NON_FINITE;
  const int64_t G = K / M;
  const int64_t meta_row = (G + 1) / 2;
  memset(metadata, 0, (size_t)(R * meta_row));
  int* used = (int*)malloc(sizeof(int) * (size_t)M);
  if (!used) return ORC_INVALID_ARGUMENT;
  for (int64_t rb = 0; rb < R / V; ++rb) {
    for (int64_t g = 0; g < G; ++g) {
      /* step 1: columns of the block that hold a kept entry */
      int ns = 0;
      for (int j = 0; j < M; ++j) {
        used[j] = 0;
        for (int64_t i = rb * V; i < rb * V + V; ++i)
          if (mask[i * ldm + g * M + j]) used[j] = 1;
        ns += used[j];
      }
      if (ns > 4) { free(used); return ORC_INVALID_MASK; }
      for (int j = 0; j < M && ns < 4; ++j)
        if (!used[j]) { used[j] = 2; ++ns; }          /* fill: lowest free columns */
      int c[4], n = 0;
      for (int j = 0; j < M; ++j)
        if (used[j]) c[n++] = j;                       /* ascending by construction */
      for (int t = 0; t < 4; ++t) column_idx[(rb * G + g) * 4 + t] = (uint8_t)c[t];
      /* step 2: per row, the kept m-indices, completed to two */
      for (int64_t i = rb * V; i < rb * V + V; ++i) {
        int keep[4], np = 0;
        for (int t = 0; t < 4; ++t) {
          keep[t] = mask[i * ldm + g * M + c[t]] != 0;
          np += keep[t];
        }
        if (np > 2) { free(used); return ORC_INVALID_MASK; }
        int p[2], q = 0;
        /* the kept positions and the lowest free ones, merged in ascending order */
        int pick[4] = {0, 0, 0, 0};
        for (int t = 0; t < 4; ++t) pick[t] = keep[t];
        for (int t = 0; t < 4 && np < 2; ++t)
          if (!pick[t]) { pick[t] = 2; ++np; }
        for (int t = 0; t < 4; ++t)
          if (pick[t]) p[q++] = t;
        for (int s2 = 0; s2 < 2; ++s2)
          values[(i * G + g) * 2 + s2] = (pick[p[s2]] == 1) ? A[i * lda + g * M + c[p[s2]]] : (uint16_t)0x0000;
        uint8_t nib = (uint8_t)(p[0] | (p[1] << 2));
        metadata[i * meta_row + g / 2] |= (uint8_t)(nib << (4 * (g % 2)));
      }
    }
  }
  free(used);
  return ORC_OK;
}

/*
 * Energy of a pruned matrix: the kept magnitude over the dense magnitude,
 * energy = sum_kept |w_i| / sum_all |w*_i|, both summed in fp64 in ascending index order. The kept
 * entries are the stored values (n_values of them; filled +0.0 entries add nothing). out[0] = kept
 * sum, out[1] = dense sum, out[2] = energy, defined as 1 when the dense sum is 0 (reading #21).
 */
int oracle_energy(const uint16_t* A, int64_t R, int64_t K, int64_t lda, int dtype,
                  const uint16_t* values, int64_t n_values, double* out) {
  if (dtype != 0 && dtype != 1) return ORC_UNSUPPORTED_DTYPE;
  if (lda < K) return ORC_INVALID_ARGUMENT;
  double kept = 0.0, all = 0.0;
  for (int64_t v = 0; v < n_values; ++v) kept += fabs(oracle_decode(values[v], dtype));
  for (int64_t i = 0; i < R; ++i)
    for (int64_t k = 0; k < K; ++k) all += fabs(oracle_decode(A[i * lda + k], dtype));
  out[0] = kept;
  out[1] = all;
  out[2] = (all == 0.0) ? 1.0 : kept / all;
  return ORC_OK;
}

/* Read the nibble of (row i, group g) and its two 2-bit positions; 0 if well formed. */
static int nib_positions(const uint8_t* metadata, int64_t meta_row, int64_t i, int64_t g,
                         int* p0, int* p1) {
  uint8_t nib = (uint8_t)((metadata[i * meta_row + g / 2] >> (4 * (g % 2))) & 0xF);
  *p0 = nib & 3;
  *p1 = (nib >> 2) & 3;
  return (*p0 < *p1) ? 0 : 1;      /* m-indices strictly increasing */
}

static int column_idx_ok(const uint8_t* column_idx, int64_t R, int V, int64_t G, int M) {
  for (int64_t b = 0; b < (R / V) * G; ++b) {
    for (int t = 0; t < 4; ++t) {
      if (column_idx[b * 4 + t] >= M) return 0;
      if (t > 0 && column_idx[b * 4 + t] <= column_idx[b * 4 + t - 1]) return 0;
    }
  }
  return 1;
}

/*
 * Decompression: the inverse of Fig 3. Entry
 * (i, g*M + column_idx[i/V][g][p]) receives the stored value whose m-index is p; every other
 * entry is +0.0 (bits 0x0000). A_out is R x K with row stride lda.
 */
int oracle_decompress(const uint16_t* values, const uint8_t* metadata, const uint8_t* column_idx,
                      int64_t R, int64_t K, int dtype, int V, int N, int M,
                      uint16_t* A_out, int64_t lda) {
  int st = oracle_validate(R, K, V, N, M);
  if (st != ORC_OK) return st;
  if (dtype != 0 && dtype != 1) return ORC_UNSUPPORTED_DTYPE;
  if (lda < K) return ORC_INVALID_ARGUMENT;
  const int64_t G = K / M, meta_row = (G + 1) / 2;
  if (!column_idx_ok(column_idx, R, V, G, M)) return ORC_CORRUPT_METADATA;
  for (int64_t i = 0; i < R; ++i)
    for (int64_t g = 0; g < G; ++g) {
      int p0, p1;
      if (nib_positions(metadata, meta_row, i, g, &p0, &p1)) return ORC_CORRUPT_METADATA;
    }
  for (int64_t i = 0; i < R; ++i)
    for (int64_t k = 0; k < K; ++k) A_out[i * lda + k] = 0x0000;
  for (int64_t i = 0; i < R; ++i) {
    const int64_t rb = i / V;
    for (int64_t g = 0; g < G; ++g) {
      int p[2];
      nib_positions(metadata, meta_row, i, g, &p[0], &p[1]);
      for (int sidx = 0; sidx < 2; ++sidx) {
        int col = column_idx[(rb * G + g) * 4 + p[sidx]];
        A_out[i * lda + g * M + col] = values[(i * G + g) * 2 + sidx];
      }
    }
  }
  return ORC_OK;
}

/*
 * SpMM straight on the compressed operand (§4, Fig 4): for every row i and
 * group g, the two stored values multiply the rows of B named by column-loc through their
 * m-indices. fp64 accumulation, groups ascending.
 *   C[i][t] = bias[i] + sum_g sum_s values[i][g][s] * B[g*M + column_idx[i/V][g][p_s]][t]
 * B: K x T raw patterns with row stride ldb. bias: R patterns or NULL. C: R x T doubles (ldc).
 * Rows are independent; OpenMP (if enabled at build) splits rows only — each element's
 * summation order is unchanged.
 */
int oracle_spmm_compressed(const uint16_t* values, const uint8_t* metadata,
                           const uint8_t* column_idx, int64_t R, int64_t K, int dtype,
                           int V, int N, int M, const uint16_t* B, int64_t T, int64_t ldb,
                           const uint16_t* bias, double* C, int64_t ldc) {
  int st = oracle_validate(R, K, V, N, M);
  if (st != ORC_OK) return st;
  if (dtype != 0 && dtype != 1) return ORC_UNSUPPORTED_DTYPE;
  if (ldb < T || ldc < T) return ORC_INVALID_ARGUMENT;
  const int64_t G = K / M, meta_row = (G + 1) / 2;
  if (!column_idx_ok(column_idx, R, V, G, M)) return ORC_CORRUPT_METADATA;
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (int64_t i = 0; i < R; ++i) {
    const int64_t rb = i / V;
    double* acc = C + i * ldc;
    double b0 = bias ? oracle_decode(bias[i], dtype) : 0.0;
    for (int64_t t = 0; t < T; ++t) acc[t] = b0;
    for (int64_t g = 0; g < G; ++g) {
      int p[2];
      if (nib_positions(metadata, meta_row, i, g, &p[0], &p[1])) { bad = 1; break; }
      for (int sidx = 0; sidx < 2; ++sidx) {
        double v = oracle_decode(values[(i * G + g) * 2 + sidx], dtype);
        int64_t krow = g * M + column_idx[(rb * G + g) * 4 + p[sidx]];
        const uint16_t* brow = B + krow * ldb;
        for (int64_t t = 0; t < T; ++t) acc[t] += v * oracle_decode(brow[t], dtype);
      }
    }
  }
  return bad ? ORC_CORRUPT_METADATA : ORC_OK;
}

/*
 * Dense product on an uncompressed matrix (the "dense counterpart"):
 * C[i][t] = bias[i] + sum_{k ascending} A[i][k] * B[k][t], fp64. Used on decompress(.) as an
 * independent formulation of the SpMM.
 */
int oracle_gemm_dense(const uint16_t* A, int64_t R, int64_t K, int64_t lda, int dtype,
                      const uint16_t* B, int64_t T, int64_t ldb, const uint16_t* bias,
                      double* C, int64_t ldc) {
  if (dtype != 0 && dtype != 1) return ORC_UNSUPPORTED_DTYPE;
  if (lda < K || ldb < T || ldc < T) return ORC_INVALID_ARGUMENT;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < R; ++i) {
    for (int64_t t = 0; t < T; ++t) {
      double acc = bias ? oracle_decode(bias[i], dtype) : 0.0;
      for (int64_t k = 0; k < K; ++k)
        acc += oracle_decode(A[i * lda + k], dtype) * oracle_decode(B[k * ldb + t], dtype);
      C[i * ldc + t] = acc;
    }
  }
  return ORC_OK;
}

/*
 * Re-encoding of a V:N:M matrix (M % 4 == 0) as a V:2:4 matrix over the ORIGINAL K (the "dense-K"
 * execution plan, reading #18). A group of M columns keeps 2 values, so every aligned
 * 4-column subgroup of it holds at most 2 kept positions: the V:N:M pattern is a 2:4 pattern. Per
 * row and 4-column subgroup j (columns 4j..4j+3), take the kept positions of the V:N:M structure
 * that fall inside it (from column_idx and the m-indices — the structure, not the values):
 *   two kept  -> values (a, b) at positions (i0, i1), i0 < i1
 *   one kept  -> position i: (v, 0) at (0, 1) if i == 0, else (0, v) at (0, i)
 *   none      -> (0, 0) at (0, 1)
 * where an inserted 0 is +0.0 (bits 0x0000) and kept values keep their original bits. The output
 * column_idx is the identity [0,1,2,3] for every block. Outputs: values2 R x (K/4) x 2,
 * metadata2 R x ceil((K/4)/2), column_idx2 (R/V) x (K/4) x 4.
 */
int oracle_expand_2to4(const uint16_t* values, const uint8_t* metadata, const uint8_t* column_idx,
                       int64_t R, int64_t K, int V, int N, int M,
                       uint16_t* values2, uint8_t* metadata2, uint8_t* column_idx2) {
  int st = oracle_validate(R, K, V, N, M);
  if (st != ORC_OK) return st;
  if (M % 4 != 0) return ORC_UNSUPPORTED_PATTERN;
  const int64_t G = K / M, meta_row = (G + 1) / 2;
  const int64_t G2 = K / 4, meta_row2 = (G2 + 1) / 2;
  if (!column_idx_ok(column_idx, R, V, G, M)) return ORC_CORRUPT_METADATA;
  memset(metadata2, 0, (size_t)(R * meta_row2));
  for (int64_t b = 0; b < (R / V) * G2; ++b) {
    for (int t = 0; t < 4; ++t) column_idx2[b * 4 + t] = (uint8_t)t;
  }
  for (int64_t i = 0; i < R; ++i) {
    const int64_t rb = i / V;
    for (int64_t g = 0; g < G; ++g) {
      int p[2];
      if (nib_positions(metadata, meta_row, i, g, &p[0], &p[1])) return ORC_CORRUPT_METADATA;
      /* absolute columns of the two kept values, ascending (column_idx and m-indices ascend) */
      int64_t col[2];
      uint16_t val[2];
      for (int s2 = 0; s2 < 2; ++s2) {
        col[s2] = g * M + column_idx[(rb * G + g) * 4 + p[s2]];
        val[s2] = values[(i * G + g) * 2 + s2];
      }
      for (int64_t j = g * (M / 4); j < (g + 1) * (M / 4); ++j) {   /* subgroups of this group */
        int n = 0, pos[2];
        uint16_t v[2];
        for (int s2 = 0; s2 < 2; ++s2) {
          if (col[s2] >= 4 * j && col[s2] < 4 * j + 4) {
            pos[n] = (int)(col[s2] - 4 * j);
            v[n] = val[s2];
            ++n;
          }
        }
        uint16_t out0, out1;
        int q0, q1;
        if (n == 2) {
          out0 = v[0]; out1 = v[1]; q0 = pos[0]; q1 = pos[1];
        } else if (n == 1) {
          if (pos[0] == 0) { out0 = v[0]; out1 = 0x0000; q0 = 0; q1 = 1; }
          else             { out0 = 0x0000; out1 = v[0]; q0 = 0; q1 = pos[0]; }
        } else {
          out0 = 0x0000; out1 = 0x0000; q0 = 0; q1 = 1;
        }
        values2[(i * G2 + j) * 2 + 0] = out0;
        values2[(i * G2 + j) * 2 + 1] = out1;
        metadata2[i * meta_row2 + j / 2] |= (uint8_t)((q0 | (q1 << 2)) << (4 * (j % 2)));
      }
    }
  }
  return ORC_OK;
}

/* Number of OpenMP threads the parallel loops above use (1 when built without OpenMP). */
int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Thread-count control for the timing legs (bench.py cpu_baseline: single-thread and all-core
 * runs); no arithmetic. n <= 0 restores the OpenMP default. */
void oracle_set_num_threads(int n) {
#ifdef _OPENMP
  extern void omp_set_num_threads(int);
  extern int omp_get_num_procs(void);
  omp_set_num_threads(n > 0 ? n : omp_get_num_procs());
#else
  (void)n;
#endif
}
