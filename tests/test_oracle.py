"""Pins for the CPU oracle (-m "not gpu"): the oracle is checked against what the paper and the
mathematics fix, never against itself. Each test names the passage or property it pins."""
from __future__ import annotations

import itertools
import math

import numpy as np
import pytest

import oracle
import synth
from tests.helpers import (BF16, F16, bits_to_f64, f64_to_bits, load_golden,
                           mask_from_compressed, rel_fro)


# --------------------------------------------------------------------------- format decoding
def test_decode_fp16_exhaustive():
    """oracle_decode (fp16) == numpy's IEEE binary16 conversion for all 65536 patterns."""
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = bits.view(np.float16).astype(np.float64)
    got = np.array([oracle.decode(int(b), F16) for b in bits])
    same = (got == ref) | (np.isnan(got) & np.isnan(ref))
    assert same.all()
    assert math.copysign(1.0, oracle.decode(0x8000, F16)) == -1.0


def test_decode_bf16_exhaustive():
    """oracle_decode (bf16) == torch.bfloat16 -> float64 for all 65536 patterns."""
    import torch
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).to(torch.float64).numpy()
    got = np.array([oracle.decode(int(b), BF16) for b in bits])
    same = (got == ref) | (np.isnan(got) & np.isnan(ref))
    assert same.all()


# --------------------------------------------------------------------------- validation
@pytest.mark.parametrize("R,K,V,N,M,expect", [
    (1024, 4096, 64, 2, 8, oracle.OK),
    (10, 16, 4, 2, 8, oracle.NON_DIVISIBLE_ROWS),
    (8, 8, 4, 2, 3, oracle.UNSUPPORTED_PATTERN),
    (8, 12, 4, 2, 8, oracle.NON_DIVISIBLE_COLS),
    (8, 16, 4, 1, 8, oracle.UNSUPPORTED_PATTERN),        # N fixed at 2
    (8, 512, 4, 2, 512, oracle.UNSUPPORTED_PATTERN),     # u8 column_idx (reading #10)
])
def test_validate_spec_examples(R, K, V, N, M, expect):
    assert oracle.validate(R, K, V, N, M) == expect


def test_non_finite_rejected():
    A = synth.gaussian((4, 8), 1.0, F16, 1)
    A[2, 5] = 0x7C00  # +inf
    assert oracle.compress(A, F16, V=2, M=8, check=False) == oracle.NON_FINITE
    A[2, 5] = 0x7E00  # nan
    assert oracle.compress(A, F16, V=2, M=8, check=False) == oracle.NON_FINITE


# --------------------------------------------------------------------------- worked examples
def _golden_bits(g, key_f, key_b):
    dt = F16 if g["dtype"] == "f16" else BF16
    if key_b in g:
        return np.array(g[key_b], dtype=np.uint16), dt
    return f64_to_bits(np.array(g[key_f], dtype=np.float64), dt), dt


@pytest.mark.parametrize("name", ["P1_spec_worked_example.json", "P2_greedy_not_joint.json",
                                  "P3_fp64_exact_column_sums.json", "P4_raw_bits_and_zero_ties.json"])
def test_compress_golden(name):
    g = load_golden(name)
    A, dt = _golden_bits(g, "A", "A_bits")
    values, meta, cidx = oracle.compress(A, dt, V=g["V"], M=g["M"], N=g["N"])
    assert cidx.tolist() == g["expected_column_idx"]
    assert meta.tolist() == g["expected_metadata"]
    exp_vals, _ = _golden_bits(g, "expected_values", "expected_values_bits")
    assert np.array_equal(values, exp_vals)


def test_decompress_golden_P5():
    g = load_golden("P5_spec_decompress.json")
    vals = f64_to_bits(np.array(g["values"]), F16)
    dense = oracle.decompress(vals, np.array(g["metadata"], np.uint8), np.array(g["column_idx"], np.uint8),
                              R=1, K=8, dtype=F16, V=1, M=8)
    assert np.array_equal(dense, f64_to_bits(np.array(g["expected_dense"]), F16))
    assert dense[0, 0] == 0x0000  # +0.0 fill


def test_decompress_all_zero_values():
    """all-zero values with any valid metadata -> zero matrix."""
    R, K, V, M = 4, 16, 2, 8
    vals = np.zeros((R, 2, 2), np.uint16)
    meta = np.full((R, 1), 0x4C, np.uint8)       # groups: (0,1) and (0,3)
    cidx = np.array([[[0, 2, 5, 7], [1, 2, 3, 4]]] * 2, np.uint8)
    assert not oracle.decompress(vals, meta, cidx, R, K, F16, V, M).any()


def test_decompress_corrupt_metadata():
    R, K, V, M = 2, 8, 2, 8
    vals = np.zeros((R, 1, 2), np.uint16)
    good = np.array([[[0, 2, 5, 7]]], np.uint8)
    assert oracle.decompress(vals, np.array([[0x5], [0x4]], np.uint8), good, R, K, F16, V, M,
                             check=False) == oracle.CORRUPT_METADATA      # p0 == p1
    assert oracle.decompress(vals, np.array([[0x1], [0x4]], np.uint8), good, R, K, F16, V, M,
                             check=False) == oracle.CORRUPT_METADATA      # p0 > p1
    bad_c = np.array([[[0, 5, 5, 7]]], np.uint8)
    assert oracle.decompress(vals, np.array([[0x4], [0x4]], np.uint8), bad_c, R, K, F16, V, M,
                             check=False) == oracle.CORRUPT_METADATA
    bad_c = np.array([[[0, 2, 5, 8]]], np.uint8)
    assert oracle.decompress(vals, np.array([[0x4], [0x4]], np.uint8), bad_c, R, K, F16, V, M,
                             check=False) == oracle.CORRUPT_METADATA


# --------------------------------------------------------------------------- brute force
def _brute_force_compress(A, dt, V, M):
    """Exhaustive reading of PAPER.md:187-188: among all C(M,4) column subsets take the one with
    the largest exact L1 mass (lexicographically first on ties); then per row among the 6 pairs of
    the 4 selected columns the largest exact |a|+|b| (lexicographically first). Independent of the
    oracle's greedy selection code."""
    R, K = A.shape
    G = K // M
    x = np.abs(bits_to_f64(A, dt))
    cidx = np.zeros((R // V, G, 4), np.uint8)
    vals = np.zeros((R, G, 2), np.uint16)
    meta = np.zeros((R, (G + 1) // 2), np.uint8)
    for rb in range(R // V):
        for g in range(G):
            blk = x[rb * V:(rb + 1) * V, g * M:(g + 1) * M]
            colsum = [math.fsum(blk[:, j]) for j in range(M)]
            best = max(itertools.combinations(range(M), 4),
                       key=lambda s: (math.fsum(colsum[j] for j in s), [-j for j in s]))
            cidx[rb, g] = best
            for i in range(rb * V, (rb + 1) * V):
                row = [x[i, g * M + c] for c in best]
                p = max(itertools.combinations(range(4), 2),
                        key=lambda q: (row[q[0]] + row[q[1]], -q[0], -q[1]))
                vals[i, g] = [A[i, g * M + best[p[0]]], A[i, g * M + best[p[1]]]]
                meta[i, g // 2] |= (p[0] | (p[1] << 2)) << (4 * (g % 2))
    return vals, meta, cidx


@pytest.mark.parametrize("V,M,R,K,seed,kind", [
    (1, 4, 3, 8, 1, "gauss"), (2, 5, 4, 10, 2, "gauss"), (3, 6, 6, 12, 3, "int"),
    (4, 7, 8, 14, 4, "int"), (2, 8, 4, 16, 5, "gauss"), (8, 9, 8, 18, 6, "int"),
    (2, 10, 4, 20, 7, "special"), (1, 8, 4, 24, 8, "special"), (4, 12, 8, 24, 9, "int"),
])
def test_compress_matches_brute_force(V, M, R, K, seed, kind):
    if kind == "gauss":
        A = synth.gaussian((R, K), 1.0, F16, seed)
    elif kind == "int":
        A = synth.small_integers((R, K), F16, seed, -2, 2)
    else:
        A = synth.special_values((R, K), F16, seed)
    got = oracle.compress(A, F16, V=V, M=M)
    exp = _brute_force_compress(A, F16, V, M)
    for a, b in zip(got, exp):
        assert np.array_equal(a, b)


def test_m4_is_textbook_2_4_pruning():
    """M=4 degenerates to plain 2:4 magnitude pruning (reading #12):
    column_idx == [0,1,2,3], each group keeps its two largest |w| (stable ties)."""
    for dt in (F16, BF16):
        A = synth.small_integers((16, 64), dt, 11, -3, 3)
        vals, meta, cidx = oracle.compress(A, dt, V=8, M=4)
        assert (cidx == np.array([0, 1, 2, 3], np.uint8)).all()
        mag = np.abs(bits_to_f64(A, dt)).reshape(16, 16, 4)
        order = np.argsort(-mag, axis=2, kind="stable")[:, :, :2]
        keep = np.sort(order, axis=2)
        exp_vals = np.take_along_axis(A.reshape(16, 16, 4), keep, axis=2)
        assert np.array_equal(vals, exp_vals)
        nib = keep[:, :, 0] | (keep[:, :, 1] << 2)
        exp_meta = (nib[:, 0::2] | (nib[:, 1::2] << 4)).astype(np.uint8)
        assert np.array_equal(meta, exp_meta)


# --------------------------------------------------------------------------- invariants
@pytest.mark.parametrize("dt", [F16, BF16])
@pytest.mark.parametrize("V,M,R,K", [(64, 8, 128, 128), (128, 16, 256, 512), (32, 20, 64, 200),
                                     (1, 4, 8, 32), (16, 7, 48, 63), (8, 100, 16, 400)])
def test_compress_invariants(dt, V, M, R, K):
    """Shape identities PAPER.md:194-195; V-block column sharing and 2-per-row;
    kept values are the original bits; selected columns dominate; kept weights dominate."""
    A = synth.gaussian((R, K), 0.02, dt, 100 + V + M)
    vals, meta, cidx = oracle.compress(A, dt, V=V, M=M)
    G = K // M
    assert vals.size == R * (K // M) * 2 and cidx.size == (R // V) * (K // M) * 4
    assert (np.diff(cidx.astype(int), axis=2) > 0).all() and (cidx < M).all()
    mask = mask_from_compressed(meta, cidx, R, K, V, M)
    assert mask.sum() == R * G * 2                                   # popcount = R*K/M*2
    dense = oracle.decompress(vals, meta, cidx, R, K, dt, V, M)
    assert np.array_equal(dense[mask], A[mask]) and not dense[~mask].any()
    x = np.abs(bits_to_f64(A, dt))
    for rb in range(R // V):
        for g in range(G):
            blk = x[rb * V:(rb + 1) * V, g * M:(g + 1) * M]
            s = blk.sum(axis=0)
            sel = set(cidx[rb, g].tolist())
            assert min(s[j] for j in sel) >= max([s[j] for j in range(M) if j not in sel] or [0])
            cols_used = np.nonzero(mask[rb * V:(rb + 1) * V, g * M:(g + 1) * M].any(axis=0))[0]
            assert set(cols_used.tolist()) <= sel
            for i in range(V):
                kept = blk[i, mask[rb * V + i, g * M:(g + 1) * M]]
                dropped = [blk[i, c] for c in sel if not mask[rb * V + i, g * M + c]]
                assert kept.min() >= max(dropped)


def test_compress_deterministic_and_lda():
    """Canonical form and row stride handling: a view with lda > K gives the same
    bytes as the contiguous matrix."""
    big = synth.gaussian((64, 200), 1.0, F16, 5)
    A = big[:, :160]
    a1 = oracle.compress(A, F16, V=16, M=10)
    a2 = oracle.compress(np.ascontiguousarray(A), F16, V=16, M=10)
    for x, y in zip(a1, a2):
        assert np.array_equal(x, y)


# --------------------------------------------------------------------------- SpMM
@pytest.mark.parametrize("dt", [F16, BF16])
@pytest.mark.parametrize("V,M,R,K,T,bias", [(64, 8, 128, 128, 128, False), (4, 4, 32, 64, 24, True),
                                            (128, 16, 256, 256, 40, True), (32, 20, 64, 160, 16, False),
                                            (2, 100, 8, 400, 8, True)])
def test_spmm_two_formulations_agree(dt, V, M, R, K, T, bias):
    """SpMM on the compressed form == dense fp64 product on decompress(A)
     to 1e-12; and == numpy float64 matmul (library routine)."""
    A = synth.gaussian((R, K), 0.02, dt, 7)
    B = synth.gaussian((K, T), 1.0, dt, 8)
    bvec = synth.gaussian((R,), 0.5, dt, 9) if bias else None
    vals, meta, cidx = oracle.compress(A, dt, V=V, M=M)
    C1 = oracle.spmm(vals, meta, cidx, R, K, dt, V, M, B, bias=bvec)
    D = oracle.decompress(vals, meta, cidx, R, K, dt, V, M)
    C2 = oracle.gemm_dense(D, B, dt, bias=bvec)
    assert rel_fro(C1, C2) <= 1e-12
    C3 = bits_to_f64(D, dt) @ bits_to_f64(B, dt)
    if bias:
        C3 = C3 + bits_to_f64(bvec, dt)[:, None]
    assert rel_fro(C1, C3) <= 1e-12


def test_spmm_identity_B_is_decompress():
    """B = I_K (T = K) => C = decompress(A), exactly."""
    R, K, V, M = 64, 96, 16, 12
    A = synth.gaussian((R, K), 1.0, F16, 21)
    vals, meta, cidx = oracle.compress(A, F16, V=V, M=M)
    I = f64_to_bits(np.eye(K), F16)
    C = oracle.spmm(vals, meta, cidx, R, K, F16, V, M, I)
    D = oracle.decompress(vals, meta, cidx, R, K, F16, V, M)
    assert np.array_equal(C, bits_to_f64(D, F16))


def test_spmm_zero_A_gives_bias():
    R, K, T, V, M = 32, 64, 16, 8, 8
    A = np.zeros((R, K), np.uint16)
    vals, meta, cidx = oracle.compress(A, F16, V=V, M=M)
    B = synth.gaussian((K, T), 1.0, F16, 3)
    bvec = synth.gaussian((R,), 1.0, F16, 4)
    C = oracle.spmm(vals, meta, cidx, R, K, F16, V, M, B, bias=bvec)
    assert np.array_equal(C, np.repeat(bits_to_f64(bvec, F16)[:, None], T, axis=1))


def test_spmm_reads_only_selected_rows_of_B():
    """'each thread-block will load only the rows of B selected by column-loc':
    poison every B row no block selects with NaN — the output stays finite."""
    R, K, T, V, M = 64, 128, 8, 64, 16
    A = synth.gaussian((R, K), 1.0, F16, 31)
    vals, meta, cidx = oracle.compress(A, F16, V=V, M=M)
    B = synth.gaussian((K, T), 1.0, F16, 32)
    used = set()
    for rb in range(R // V):
        for g in range(K // M):
            used |= {g * M + int(c) for c in cidx[rb, g]}
    for k in range(K):
        if k not in used:
            B[k, :] = 0x7E00
    assert len(used) < K
    C = oracle.spmm(vals, meta, cidx, R, K, F16, V, M, B)
    assert np.isfinite(C).all()


def test_spmm_linearity_and_column_subset():
    """Linearity in B (exact power-of-two scaling) and column independence (a T-subset via ldb
    equals the same columns of the full product — the T-split of DESIGN.md §multi-GPU)."""
    R, K, T, V, M = 64, 128, 32, 32, 8
    A = synth.gaussian((R, K), 0.02, F16, 41)
    B = synth.gaussian((K, T), 1.0, F16, 42)
    vals, meta, cidx = oracle.compress(A, F16, V=V, M=M)
    C = oracle.spmm(vals, meta, cidx, R, K, F16, V, M, B)
    B2 = f64_to_bits(bits_to_f64(B, F16) * 2.0, F16)
    assert np.array_equal(oracle.spmm(vals, meta, cidx, R, K, F16, V, M, B2), 2.0 * C)
    Csub = oracle.spmm(vals, meta, cidx, R, K, F16, V, M, B[:, 8:24])
    assert np.array_equal(Csub, C[:, 8:24])


def test_cost_identities():
    """PAPER.md:209 (2:8: MACs 16 -> 4 per output, half the B rows) and PAPER.md:272 (ideal
    speedups 5x/10x/20x/50x for 2:10/2:20/2:40/2:100): nnz = R*K*2/M."""
    for M, ideal in [(10, 5), (20, 10), (40, 20), (100, 50)]:
        R, K = 8, 4 * M
        nv, _, _ = oracle.sizes(R, K, 8, M)
        assert (R * K) / nv == ideal
    nv, _, nc = oracle.sizes(16, 32, 4, 8)
    assert nv / 16 == 32 / 4 and nc == (16 // 4) * (32 // 8) * 4   # B rows fetched per block: 4 of 8


# --------------------------------------------------------------------------- 2:4 re-encoding
@pytest.mark.parametrize("V,M,R,K,kind", [(64, 8, 128, 256, "gauss"), (4, 16, 16, 128, "int"),
                                          (2, 4, 8, 64, "special"), (8, 32, 16, 256, "gauss"),
                                          (16, 12, 32, 96, "int"), (1, 8, 8, 64, "special")])
def test_expand_2to4_is_same_matrix(V, M, R, K, kind):
    """expand(x) re-encodes the V:N:M matrix as V:2:4 over K (reading #18): the dense
    matrices are bit-identical, the result is a valid 2:4 structure, and M = 4 is the identity."""
    dt = F16
    A = {"gauss": synth.gaussian((R, K), 1.0, dt, 5), "int": synth.small_integers((R, K), dt, 6),
         "special": synth.special_values((R, K), dt, 7)}[kind]
    vals, meta, cidx = oracle.compress(A, dt, V=V, M=M)
    v2, m2, c2 = oracle.expand_2to4(vals, meta, cidx, R, K, V, M)
    assert (c2 == np.array([0, 1, 2, 3], np.uint8)).all()
    d1 = oracle.decompress(vals, meta, cidx, R, K, dt, V, M)
    d2 = oracle.decompress(v2, m2, c2, R, K, dt, V, 4)
    assert np.array_equal(d1, d2)
    # the kept positions of the 2:4 form are a superset of the V:N:M kept positions
    mask1 = mask_from_compressed(meta, cidx, R, K, V, M)
    mask2 = mask_from_compressed(m2, c2, R, K, V, 4)
    assert (mask2 | ~mask1).all() and mask2.sum() == R * K // 2
    # SpMM through either encoding is the same product (exactly: one formulation, same terms)
    B = synth.gaussian((K, 8), 1.0, dt, 8)
    assert np.array_equal(oracle.spmm(vals, meta, cidx, R, K, dt, V, M, B),
                          oracle.spmm(v2, m2, c2, R, K, dt, V, 4, B)) or \
        rel_fro(oracle.spmm(vals, meta, cidx, R, K, dt, V, M, B), oracle.spmm(v2, m2, c2, R, K, dt, V, 4, B)) < 1e-15


def test_expand_2to4_m4_identity_and_rules():
    """M = 4: expand is the identity on (values, metadata). Hand case (M = 8, one row): kept columns
    1 and 6 fall in different subgroups -> (0, a) at (0, 1) and (b, 0)... worked by hand below."""
    A = synth.gaussian((8, 32), 1.0, F16, 9)
    vals, meta, cidx = oracle.compress(A, F16, V=4, M=4)
    v2, m2, _ = oracle.expand_2to4(vals, meta, cidx, 8, 32, 4, 4)
    assert np.array_equal(v2, vals) and np.array_equal(m2, meta)
    # one V:N:M group of 8 columns, column_idx [1,2,5,6], m-indices (0,3) -> kept columns 1 and 6
    a, b = f64_to_bits(np.array([1.5, -2.0]), F16)
    vals = np.array([[[a, b]]], np.uint16)
    meta = np.array([[0x0C]], np.uint8)
    cidx = np.array([[[1, 2, 5, 6]]], np.uint8)
    v2, m2, _ = oracle.expand_2to4(vals, meta, cidx, 1, 8, 1, 8)
    # subgroup 0 (cols 0-3): a at position 1 -> (0, a) at (0, 1); subgroup 1 (cols 4-7): b at 2 -> (0, b) at (0, 2)
    assert v2.tolist() == [[[0, int(a)], [0, int(b)]]]
    assert m2.tolist() == [[(0 | 1 << 2) | ((0 | 2 << 2) << 4)]]


# --------------------------------------------------------------------------- masked compression
# SURVEY §8(f) rank 4 / DESIGN.md readings #20-#21: the kept set from an external V:N:M mask.
@pytest.mark.parametrize("name", ["P7_masked_compress.json", "P8_masked_fill.json"])
def test_compress_masked_golden(name):
    g = load_golden(name)
    A, dt = _golden_bits(g, "A", "A_bits")
    mask = np.array(g["mask"], np.uint8)
    values, meta, cidx = oracle.compress_masked(A, mask, dt, V=g["V"], M=g["M"], N=g["N"])
    assert cidx.tolist() == g["expected_column_idx"]
    assert meta.tolist() == g["expected_metadata"]
    exp_vals, _ = _golden_bits(g, "expected_values", "expected_values_bits")
    assert np.array_equal(values, exp_vals)
    assert oracle.energy(A, values, dt)[2] == pytest.approx(g["expected_energy"], rel=1e-15)


@pytest.mark.parametrize("R,K,V,M,dt,seed", [(8, 64, 4, 8, F16, 1), (16, 96, 8, 16, BF16, 2),
                                             (12, 40, 3, 10, F16, 3), (4, 32, 1, 4, F16, 4)])
def test_compress_masked_roundtrip_is_A_times_mask(R, K, V, M, dt, seed):
    """decompress(compress_masked(A, m)) == A∘m bit for bit, with pruned entries +0.0 (the operand
    is exactly the masked matrix); A∘m written with numpy, not the oracle."""
    A = synth.gaussian((R, K), 1.0, dt, seed)
    m = synth.vnm_mask(R, K, V, M, seed + 100)
    v, md, c = oracle.compress_masked(A, m, dt, V=V, M=M)
    D = oracle.decompress(v, md, c, R, K, dt, V, M)
    assert np.array_equal(D, np.where(m != 0, A, np.uint16(0)))
    # every kept entry is addressed by the metadata; every stored position is kept or +0.0
    kept = mask_from_compressed(md, c, R, K, V, M)
    assert not (m.astype(bool) & ~kept).any()
    # the shape identities of PAPER.md:194-195 and the ascending invariants
    assert v.size == R * (K // M) * 2 and c.size == (R // V) * (K // M) * 4
    assert (np.diff(c.astype(int), axis=2) > 0).all()


def test_compress_masked_with_the_magnitude_mask_equals_compress():
    """Independent formulation: feeding the magnitude compressor's own kept set as
    the external mask reproduces the same matrix (decompressed bit for bit)."""
    R, K, V, M = 16, 128, 8, 8
    A = synth.gaussian((R, K), 1.0, F16, 9)
    v, md, c = oracle.compress(A, F16, V=V, M=M)
    m = mask_from_compressed(md, c, R, K, V, M).astype(np.uint8)
    v2, md2, c2 = oracle.compress_masked(A, m, F16, V=V, M=M)
    assert np.array_equal(oracle.decompress(v2, md2, c2, R, K, F16, V, M),
                          oracle.decompress(v, md, c, R, K, F16, V, M))


def test_compress_masked_rejects_non_vnm_masks():
    """A mask with 5 columns in one V x M block, or 3 kept entries in one row-group, is not V:N:M
    (PAPER.md:187-189): status INVALID_MASK."""
    A = synth.gaussian((4, 16), 1.0, F16, 5)
    m = np.zeros((4, 16), np.uint8)
    m[0, [0, 1]] = 1
    m[1, [2, 3]] = 1
    m[2, [4]] = 1  # fifth column of block (rows 0-3, cols 0-7)
    assert oracle.compress_masked(A, m, F16, V=4, M=8, check=False) == oracle.INVALID_MASK
    m[:] = 0
    m[3, [8, 9, 10]] = 1  # three kept in one row-group
    assert oracle.compress_masked(A, m, F16, V=4, M=8, check=False) == oracle.INVALID_MASK
    m[:] = 0
    m[3, [8, 9]] = 1
    assert isinstance(oracle.compress_masked(A, m, F16, V=4, M=8, check=False), tuple)


def test_energy_definition_and_special_cases():
    """energy = sum|kept| / sum|dense|, against numpy on A∘mask; 1 when nothing
    is pruned (an already V:N:M matrix), 1 for an all-zero matrix (reading #21), and within (0, 1]."""
    R, K, V, M = 8, 64, 4, 8
    A = synth.gaussian((R, K), 1.0, F16, 11)
    v, md, c = oracle.compress(A, F16, V=V, M=M)
    kept, dense, e = oracle.energy(A, v, F16)
    m = mask_from_compressed(md, c, R, K, V, M)
    a = np.abs(bits_to_f64(A, F16))
    assert dense == pytest.approx(a.sum(), rel=1e-14)
    assert kept == pytest.approx(a[m].sum(), rel=1e-14)
    assert 0.0 < e <= 1.0 and e == pytest.approx(a[m].sum() / a.sum(), rel=1e-14)
    D = oracle.decompress(v, md, c, R, K, F16, V, M)        # already V:N:M: nothing left to prune
    v2, _, _ = oracle.compress(D, F16, V=V, M=M)
    assert oracle.energy(D, v2, F16)[2] == pytest.approx(1.0, rel=1e-15)
    Z = np.zeros((R, K), np.uint16)
    vz, _, _ = oracle.compress(Z, F16, V=V, M=M)
    assert oracle.energy(Z, vz, F16) == (0.0, 0.0, 1.0)
    # magnitude pruning keeps at least the 2/M fraction of the mass that a uniform keep would
    assert e >= 2.0 / M
