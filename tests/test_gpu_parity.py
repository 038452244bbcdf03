"""GPU parity (-m gpu): the CUDA path through the C ABI vs the CPU oracle on identical seeded
inputs. Compressor / decompressor: bit-exact. SpMM: ‖C_gpu − C_ref‖_F / ‖C_ref‖_F ≤ 2e-3
(BASELINE.json north_star) plus an element-wise bound, and exact probes (identity / one-hot B)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_2310_02065_b200 as venom
import synth
from tests.helpers import BF16, F16, bits_to_f64, f64_to_bits, load_golden, rel_fro

pytestmark = pytest.mark.gpu

TOL_FRO = 2e-3  # north_star


def tdt(dt):
    return torch.float16 if dt == F16 else torch.bfloat16


def to_dev(bits: np.ndarray, dt: int) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(tdt(dt)).cuda()


def to_bits(t: torch.Tensor) -> np.ndarray:
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def gpu_compress(A_bits, dt, V, M):
    A = to_dev(A_bits, dt)
    x = venom.compress(A, V=V, M=M, check=True)
    torch.cuda.synchronize()
    return x, (to_bits(x.values), x.metadata.cpu().numpy(), x.column_idx.cpu().numpy())


def check_spmm(C_gpu: torch.Tensor, C_ref: np.ndarray, dt: int):
    got = bits_to_f64(to_bits(C_gpu), dt)
    assert np.isfinite(got).all()
    assert rel_fro(got, C_ref) <= TOL_FRO, rel_fro(got, C_ref)
    # element-wise: output rounding (half ulp) + fp32 accumulation, scale-aware for cancellation
    ulp = 2.0 ** -10 if dt == F16 else 2.0 ** -7
    scale = np.sqrt(np.mean(C_ref ** 2)) + 1e-30
    err = np.abs(got - C_ref)
    assert (err <= ulp * np.abs(C_ref) + 1e-3 * scale).all(), float((err / (np.abs(C_ref) + scale)).max())


# ------------------------------------------------------------------ compressor: bit-exact
CASES = [
    # (R, K, V, M, kind, dt)
    (128, 128, 64, 8, "gauss", F16),          # configs[0] shape
    (1024, 4096, 64, 8, "gauss", F16),        # configs[1] BERT-large FFN2
    (256, 1024, 128, 16, "gauss", BF16),
    (96, 280, 3, 7, "int", F16),
    (64, 200, 32, 10, "special", F16),
    (64, 200, 32, 10, "special", BF16),
    (40, 500, 1, 100, "gauss", F16),
    (512, 512, 256, 4, "int", BF16),
    (128, 640, 64, 40, "sparse", F16),
    (130, 256, 13, 32, "gauss", F16),
    (64, 1280, 64, 20, "int", F16),
    (16, 768, 8, 256, "gauss", BF16),
    (48, 90, 16, 5, "special", F16),
]


def make_input(R, K, kind, dt, seed, M=8):
    if kind == "gauss":
        return synth.gaussian((R, K), 0.02, dt, seed)
    if kind == "int":
        return synth.small_integers((R, K), dt, seed)
    if kind == "special":
        return synth.special_values((R, K), dt, seed)
    return synth.sparse_columns((R, K), dt, seed, live_cols_per_block=2, M=M)


@pytest.mark.parametrize("R,K,V,M,kind,dt", CASES)
def test_compress_bit_exact(R, K, V, M, kind, dt):
    A = make_input(R, K, kind, dt, 1000 + R + K + V + M, M)
    exp = oracle.compress(A, dt, V=V, M=M)
    _, got = gpu_compress(A, dt, V, M)
    for name, g, e in zip(("values", "metadata", "column_idx"), got, exp):
        assert np.array_equal(g.reshape(e.shape), e), name


# shapes whose V × W tile exceeds the shared-memory tile kernel's budget: the streaming compressor
# (vnm_compress_kernel, row-split fp64 partial sums) — fp16 and bf16, odd G, 16-byte vector and
# element-wise loads (an lda view that is not a multiple of 8)
STREAM_CASES = [
    # (R, K, V, M, kind, dt, lda_pad)
    (512, 1024, 256, 128, "gauss", F16, 0),
    (1024, 2048, 1024, 32, "int", BF16, 0),
    (512, 384, 256, 128, "special", F16, 0),      # G = 3 (odd)
    (512, 1024, 256, 128, "gauss", BF16, 3),      # lda % 8 != 0: element-wise loads
    (2048, 512, 2048, 64, "sparse", F16, 5),
]


@pytest.mark.parametrize("R,K,V,M,kind,dt,pad", STREAM_CASES)
def test_compress_streaming_kernel_bit_exact(R, K, V, M, kind, dt, pad):
    A = make_input(R, K + pad, kind, dt, 2000 + R + K + V + M + pad, M)
    x = venom.compress(to_dev(A, dt)[:, :K], V=V, M=M, check=True)
    exp = oracle.compress(np.ascontiguousarray(A[:, :K]), dt, V=V, M=M)
    got = (to_bits(x.values), x.metadata.cpu().numpy(), x.column_idx.cpu().numpy())
    for name, g, e in zip(("values", "metadata", "column_idx"), got, exp):
        assert np.array_equal(g.reshape(e.shape), e), name


def near_tie_input(R, K, V, M, dt, seed):
    """Every column of a V-row block has the same bulk (V - 1 entries of 1.0) plus one tiny entry
    whose size decides the column order: the column sums differ by far less than an fp32 sum can
    resolve, so the compressor's approximate scores cannot decide the top-4 and its exact path
    must (fp16: subnormal steps of 2^-24; bf16: steps of 2^-16 on top of 1.0 entries)."""
    rng = np.random.default_rng(seed)
    one = 0x3C00 if dt == F16 else 0x3F80
    A = np.full((R, K), one, np.uint16)
    for rb in range(R // V):
        for g in range(K // M):
            perm = rng.permutation(M) + 1
            r = rb * V + int(rng.integers(0, V))
            tiny = perm.astype(np.uint16) if dt == F16 else (0x3780 + perm).astype(np.uint16)  # bf16 ~2^-16·k
            A[r, g * M:(g + 1) * M] = tiny
    return A


@pytest.mark.parametrize("R,K,V,M,dt", [(256, 1024, 128, 16, F16), (128, 512, 64, 8, BF16),
                                        (64, 640, 32, 40, F16), (128, 256, 128, 32, F16)])
def test_compress_near_ties_bit_exact(R, K, V, M, dt):
    A = near_tie_input(R, K, V, M, dt, 11 + R + M)
    exp = oracle.compress(A, dt, V=V, M=M)
    _, got = gpu_compress(A, dt, V, M)
    for name, g, e in zip(("values", "metadata", "column_idx"), got, exp):
        assert np.array_equal(g.reshape(e.shape), e), name
    if M % 8 == 0 and 128 % M == 0 and V % 16 == 0:  # the fused compress + V:2:4 path decides alike
        x2, _ = venom.compress_2to4(to_dev(A, dt), V=V, M=M, check=True)
        assert np.array_equal(x2.column_idx.cpu().numpy(), exp[2])


@pytest.mark.parametrize("R,K,V,M,dt", [(3072, 4096, 128, 16, F16), (2048, 2048, 64, 8, BF16),
                                        (512, 8192, 256, 32, F16)])
def test_compress_many_tiles_per_cta(R, K, V, M, dt):
    """More (row block, column chunk) tiles than the persistent compressor has CTAs: every CTA runs
    its double-buffered TMA pipeline over several tiles (GPT-3-like aspect, scaled down); the fused
    compress + V:2:4 kernel takes the same path."""
    A = synth.gaussian((R, K), 0.02, dt, 5 + R + M)
    exp = oracle.compress(A, dt, V=V, M=M)
    _, got = gpu_compress(A, dt, V, M)
    for name, g, e in zip(("values", "metadata", "column_idx"), got, exp):
        assert np.array_equal(g.reshape(e.shape), e), name
    if M % 8 == 0 and 128 % M == 0 and V % 16 == 0:
        x2, y2 = venom.compress_2to4(to_dev(A, dt), V=V, M=M, check=True)
        assert np.array_equal(to_bits(x2.values).reshape(exp[0].shape), exp[0])
        assert np.array_equal(x2.column_idx.cpu().numpy(), exp[2])
        exp2 = oracle.expand_2to4(*exp, R, K, V, M)
        assert np.array_equal(to_bits(y2.values).reshape(exp2[0].shape), exp2[0])


def test_compress_more_than_65535_row_blocks():
    """V = 1 with R > 65535: the row blocks exceed one launch's grid.y (chunked launches)."""
    R, K, V, M = 70000, 32, 1, 8
    A = synth.gaussian((R, K), 0.02, F16, 77)
    exp = oracle.compress(A, F16, V=V, M=M)
    _, got = gpu_compress(A, F16, V, M)
    for name, g, e in zip(("values", "metadata", "column_idx"), got, exp):
        assert np.array_equal(g.reshape(e.shape), e), name


@pytest.mark.parametrize("name", ["P1_spec_worked_example.json", "P2_greedy_not_joint.json",
                                  "P3_fp64_exact_column_sums.json", "P4_raw_bits_and_zero_ties.json"])
def test_compress_golden_on_gpu(name):
    g = load_golden(name)
    dt = F16
    A = np.array(g["A_bits"], np.uint16) if "A_bits" in g else f64_to_bits(np.array(g["A"], float), dt)
    _, (vals, meta, cidx) = gpu_compress(A, dt, g["V"], g["M"])
    assert cidx.tolist() == g["expected_column_idx"]
    assert meta.tolist() == g["expected_metadata"]
    ev = np.array(g["expected_values_bits"], np.uint16) if "expected_values_bits" in g else \
        f64_to_bits(np.array(g["expected_values"], float), dt)
    assert np.array_equal(vals.reshape(ev.shape), ev)


def test_compress_lda_view():
    big = synth.gaussian((128, 700), 1.0, F16, 3)
    A = to_dev(big, F16)[:, :640]
    x = venom.compress(A, V=64, M=10, check=True)
    exp = oracle.compress(big[:, :640], F16, V=64, M=10)
    assert np.array_equal(to_bits(x.values).reshape(exp[0].shape), exp[0])
    assert np.array_equal(x.metadata.cpu().numpy(), exp[1])
    assert np.array_equal(x.column_idx.cpu().numpy(), exp[2])


def test_compress_non_finite_status():
    A = synth.gaussian((64, 64), 1.0, F16, 5)
    A[3, 17] = 0x7C00
    with pytest.raises(venom.VenomError) as e:
        gpu_compress(A, F16, 32, 8)
    assert e.value.status == 6


# ------------------------------------------------------------------ decompressor: bit-exact
@pytest.mark.parametrize("R,K,V,M,kind,dt", CASES[:8])
def test_decompress_bit_exact(R, K, V, M, kind, dt):
    A = make_input(R, K, kind, dt, 7 + R + K, M)
    vals, meta, cidx = oracle.compress(A, dt, V=V, M=M)
    exp = oracle.decompress(vals, meta, cidx, R, K, dt, V, M)
    x = venom.VNMTensor(to_dev(vals, dt), torch.from_numpy(meta).cuda(), torch.from_numpy(cidx).cuda(),
                        R, K, V, M)
    got = to_bits(venom.decompress(x, check=True))
    assert np.array_equal(got, exp)


def test_decompress_corrupt_metadata_status():
    R, K, V, M = 64, 64, 32, 8
    A = synth.gaussian((R, K), 1.0, F16, 9)
    vals, meta, cidx = oracle.compress(A, F16, V=V, M=M)
    meta = meta.copy()
    meta[5, 2] = 0x11  # p0 == p1
    x = venom.VNMTensor(to_dev(vals, F16), torch.from_numpy(meta).cuda(), torch.from_numpy(cidx).cuda(),
                        R, K, V, M)
    with pytest.raises(venom.VenomError) as e:
        venom.decompress(x, check=True)
    assert e.value.status == 7


# ------------------------------------------------------------------ V:N:M -> V:2:4 re-encoding: bit-exact
EXPAND_CASES = [c for c in CASES if c[3] % 4 == 0] + [
    (64, 8 * 7, 32, 8, "gauss", F16),      # odd G: last metadata byte half used
    (32, 4 * 9, 16, 4, "int", BF16),       # M = 4, odd G2
    (64, 96 * 3, 64, 96, "sparse", F16),   # most subgroups empty
]


@pytest.mark.parametrize("R,K,V,M,kind,dt", EXPAND_CASES)
def test_expand_2to4_bit_exact(R, K, V, M, kind, dt):
    A = make_input(R, K, kind, dt, 11 + R + K, M)
    parts = oracle.compress(A, dt, V=V, M=M)
    v2, m2, c2 = oracle.expand_2to4(*parts, R, K, V, M)
    y = venom.expand_2to4(vnm_from(parts, R, K, V, M, dt), check=True)
    assert (y.V, y.M, y.K) == (V, 4, K)
    assert np.array_equal(to_bits(y.values), v2)
    assert np.array_equal(y.metadata.cpu().numpy(), m2)
    assert np.array_equal(y.column_idx.cpu().numpy(), c2)
    # and the re-encoded operand decompresses to the original sparse matrix on the GPU
    assert np.array_equal(to_bits(venom.decompress(y, check=True)),
                          oracle.decompress(*parts, R, K, dt, V, M))


def test_expand_2to4_then_spmm_matches_oracle():
    R, K, T, V, M, dt = 512, 1024, 384, 64, 8, F16
    A, B, _, parts = oracle_problem(R, K, T, V, M, dt, 77)
    y = venom.expand_2to4(vnm_from(parts, R, K, V, M, dt), check=True)
    C = venom.spmm(y, to_dev(B, dt))
    torch.cuda.synchronize()
    check_spmm(C, oracle.spmm(*parts, R, K, dt, V, M, B), dt)


def test_expand_2to4_corrupt_metadata_status():
    R, K, V, M = 64, 64, 32, 8
    parts = list(oracle.compress(synth.gaussian((R, K), 1.0, F16, 9), F16, V=V, M=M))
    parts[1] = parts[1].copy()
    parts[1][3, 1] = 0x05  # p0 == p1
    with pytest.raises(venom.VenomError) as e:
        venom.expand_2to4(vnm_from(parts, R, K, V, M, F16), check=True)
    assert e.value.status == 7


# ------------------------------------------------------------------ SpMM
def oracle_problem(R, K, T, V, M, dt, seed, bias=False, kind="gauss"):
    A = make_input(R, K, kind, dt, seed, M) if kind != "gauss" else synth.gaussian((R, K), 0.02, dt, seed)
    B = synth.gaussian((K, T), 1.0, dt, seed + 1)
    bv = synth.gaussian((R,), 0.5, dt, seed + 2) if bias else None
    vals, meta, cidx = oracle.compress(A, dt, V=V, M=M)
    return A, B, bv, (vals, meta, cidx)


def vnm_from(parts, R, K, V, M, dt):
    vals, meta, cidx = parts
    return venom.VNMTensor(to_dev(vals, dt), torch.from_numpy(meta).cuda(), torch.from_numpy(cidx).cuda(),
                           R, K, V, M)


def test_spmm_identity_probe_exact():
    """P6: B = I_K => C == decompress(A) exactly (one product per output)."""
    for (R, K, V, M, dt) in [(256, 256, 128, 8, F16), (128, 512, 64, 16, F16), (256, 256, 128, 4, BF16),
                             (128, 320, 32, 10, F16)]:
        A = synth.gaussian((R, K), 1.0, dt, 77)
        vals, meta, cidx = oracle.compress(A, dt, V=V, M=M)
        D = oracle.decompress(vals, meta, cidx, R, K, dt, V, M)
        I = to_dev(f64_to_bits(np.eye(K), dt), dt)
        x = vnm_from((vals, meta, cidx), R, K, V, M, dt)
        for prepared in (False, True):
            if prepared:
                venom.order_metadata(x)
            C = venom.spmm(x, I)
            got = bits_to_f64(to_bits(C), dt)
            assert np.array_equal(got, bits_to_f64(D, dt)), (R, K, V, M, dt, prepared)


def test_spmm_one_hot_probes():
    """One-hot B columns isolate single (row, group, position) entries: column t of B selects B row
    k_t, so C[:, t] must equal column k_t of decompress(A) for every probe."""
    R, K, V, M, dt = 128, 256, 128, 8, F16
    A = synth.gaussian((R, K), 1.0, dt, 78)
    vals, meta, cidx = oracle.compress(A, dt, V=V, M=M)
    D = bits_to_f64(oracle.decompress(vals, meta, cidx, R, K, dt, V, M), dt)
    T = 64
    ks = np.random.Generator(np.random.PCG64(5)).choice(K, size=T, replace=False)
    Bm = np.zeros((K, T))
    Bm[ks, np.arange(T)] = 1.0
    x = vnm_from((vals, meta, cidx), R, K, V, M, dt)
    for prepared in (False, True):
        if prepared:
            venom.order_metadata(x)
        C = venom.spmm(x, to_dev(f64_to_bits(Bm, dt), dt))
        got = bits_to_f64(to_bits(C), dt)
        assert np.array_equal(got, D[:, ks]), prepared


SPMM_CASES = [
    # R, K, T, V, M, dt, bias, tile_t
    (128, 128, 128, 64, 8, F16, False, 0),     # configs[0]
    (256, 512, 256, 128, 8, F16, True, 0),
    (256, 512, 256, 128, 8, BF16, True, 0),
    (384, 1024, 200, 128, 16, F16, False, 0),  # T tail, 3 row tiles
    (192, 640, 136, 64, 40, F16, True, 0),     # odd number of 64-blocks (ragged last tile)
    (256, 576, 96, 32, 36, F16, True, 0),      # V = 32
    (256, 896, 128, 256, 28, BF16, False, 0),  # V = 256 (two 128-row slices share column_idx)
    (256, 1600, 264, 128, 100, F16, True, 0),  # 2:100, K' tail (G = 16)
    (512, 1024, 512, 128, 4, F16, True, 256),  # plain 2:4, tile 256
    (768, 1024, 512, 128, 4, F16, True, 256),  # 2:4, multicast pair clusters with an idle pair
    (384, 512, 264, 64, 4, BF16, False, 256),  # 2:4, half-filled cluster tile, T tail
    (512, 1024, 384, 128, 16, F16, True, 192),
    (512, 2048, 256, 128, 32, BF16, False, 64),
    (256, 1024, 256, 64, 8, F16, True, 128),   # V=64 tile 128
    (128, 4096, 64, 128, 16, F16, False, 0),   # long K
    # V = 64 as two M = 64 MMAs on the TMEM lane halves (spmm_kernel.cuh M64): a single 64-row
    # block (the tile's second half is padding), 2.5 row tiles, and last k-stages of 4 / 16 / 12
    # real groups (G = 36, 112, 44: the MMAs and gathers past them are skipped)
    (64, 288, 72, 64, 8, BF16, True, 0),
    (320, 960, 200, 64, 10, F16, True, 0),
    (448, 1120, 128, 64, 10, BF16, False, 64),
    (192, 880, 136, 64, 20, F16, True, 128),
    # V = 32 on the same lane halves (two M = 64 MMAs per half, odd blocks in the second BN
    # columns): three of a tile's four blocks (R = 96), bf16, a partial last k-stage
    (96, 704, 136, 32, 16, BF16, True, 0),
    (416, 1120, 64, 32, 10, F16, False, 0),
]


def strategies(K, V, M):
    """Strategies applicable to a problem (include/venom.h): AUTO plus each forced one."""
    out = [venom.STRATEGY_AUTO]
    if (M == 4 or V in (32, 64) or V % 128 == 0) and (K // M) % 4 == 0:
        out.append(venom.STRATEGY_GATHER)
    if M in (4, 8, 16, 32) and (K // M) % 4 == 0:
        out.append(venom.STRATEGY_DENSE_K)
    return out


@pytest.mark.parametrize("R,K,T,V,M,dt,bias,tile_t", SPMM_CASES)
def test_spmm_vs_oracle(R, K, T, V, M, dt, bias, tile_t):
    A, B, bv, parts = oracle_problem(R, K, T, V, M, dt, 500 + R + K + T + M, bias)
    C_ref = oracle.spmm(*parts, R, K, dt, V, M, B, bias=bv)
    x = vnm_from(parts, R, K, V, M, dt)
    for strat in strategies(K, V, M):
        tt = tile_t if strat != venom.STRATEGY_DENSE_K or tile_t in (0, 128, 256) else 0
        C = venom.spmm(x, to_dev(B, dt), bias=to_dev(bv, dt) if bias else None, tile_t=tt,
                       strategy=strat)
        check_spmm(C, C_ref, dt)
    # tensor-core-ordered metadata (TMA + tcgen05.cp path), every CTA grouping that applies
    venom.order_metadata(x)
    pairs = [0, 1] + ([2] if M == 4 or V % 256 == 0 else [])
    for pair in pairs:
        C = venom.spmm(x, to_dev(B, dt), bias=to_dev(bv, dt) if bias else None, tile_t=tile_t,
                       strategy=venom.STRATEGY_GATHER, cta_pair=pair)
        check_spmm(C, C_ref, dt)


K_TAIL_CASES = [
    # R, K, T, V, M, dt — G = K/M not a multiple of 4 (a K' tail): padded values + metadata_tc
    (256, 330, 136, 64, 10, F16),     # G = 33
    (128, 2040, 200, 128, 40, BF16),  # G = 51
    (384, 148, 64, 128, 4, F16),      # M = 4 (contiguous, CTA pair), G = 37
    (256, 1000, 128, 32, 20, F16),    # V = 32, G = 50
    (512, 4050, 264, 256, 90, BF16),  # V = 256 (CTA pair), G = 45
    (192, 70, 72, 64, 10, F16),       # G = 7: a single partial k-stage
]


@pytest.mark.parametrize("R,K,T,V,M,dt", K_TAIL_CASES)
def test_spmm_k_tail_vs_oracle(R, K, T, V, M, dt):
    """Any G (PAPER.md:223, 271-272 sweep K freely): order_metadata attaches the padded values
    (venom_pad_values) with the tensor-core metadata, and the SpMM matches the oracle; without the
    execution form the pattern is refused."""
    A, B, bv, parts = oracle_problem(R, K, T, V, M, dt, 1300 + R + K + M, True)
    C_ref = oracle.spmm(*parts, R, K, dt, V, M, B, bias=bv)
    x = vnm_from(parts, R, K, V, M, dt)
    with pytest.raises(venom.VenomError) as ei:
        venom.spmm(x, to_dev(B, dt), bias=to_dev(bv, dt))
    assert ei.value.status == 4
    venom.order_metadata(x)
    assert x.values_padded is not None
    vp = to_bits(x.values_padded).reshape(R, -1, 2)
    G = K // M
    assert np.array_equal(vp[:, :G], parts[0].reshape(R, G, 2)) and not vp[:, G:].any()
    pairs = [0, 1] + ([2] if M == 4 or V % 256 == 0 else [])
    for pair in pairs:
        C = venom.spmm(x, to_dev(B, dt), bias=to_dev(bv, dt), cta_pair=pair)
        check_spmm(C, C_ref, dt)
    if M != 4:
        Ct = venom.spmm(x, to_dev(B, dt), bias=to_dev(bv, dt), transposed_out=True)
        check_spmm(Ct.t().contiguous(), C_ref, dt)


def test_spmm_k_tail_after_recompress():
    """compress(A, out=x) refreshes both execution-form arrays of x (metadata_tc, values_padded)."""
    R, K, T, V, M = 128, 330, 64, 64, 10
    A1 = torch.randn(R, K, device="cuda").half()
    A2 = torch.randn(R, K, device="cuda").half()
    x = venom.order_metadata(venom.compress(A1, V=V, M=M))
    B = torch.randn(K, T, device="cuda").half()
    venom.compress(A2, V=V, M=M, out=x)
    C = venom.spmm(x, B)
    ref = venom.decompress(x).float() @ B.float()
    assert float((C.float() - ref).norm() / ref.norm()) <= TOL_FRO


DENSEK_CASES = [
    # R, K, T, V, M, dt, bias — dense-K only shapes: any V, K not a multiple of 128, M = 4 .. 32
    (128, 224, 64, 16, 8, F16, True),
    (96, 384, 40, 1, 4, F16, False),
    (256, 512, 136, 8, 16, BF16, True),
    (384, 1280, 256, 128, 32, F16, True),
    (200, 640, 72, 40, 32, F16, False),
    (256, 1088, 512, 64, 16, BF16, True),
    (128, 4096, 64, 128, 4, F16, True),
]


@pytest.mark.parametrize("R,K,T,V,M,dt,bias", DENSEK_CASES)
def test_spmm_densek_vs_oracle(R, K, T, V, M, dt, bias):
    A, B, bv, parts = oracle_problem(R, K, T, V, M, dt, 700 + R + K + T + M, bias)
    C_ref = oracle.spmm(*parts, R, K, dt, V, M, B, bias=bv)
    x = vnm_from(parts, R, K, V, M, dt)
    # the default CTA pair and the single-CTA instantiations (cta_pair = 1), both tile widths
    for pair in (0, 1):
        for tt in (0, 128):
            C = venom.spmm(x, to_dev(B, dt), bias=to_dev(bv, dt) if bias else None, tile_t=tt,
                           strategy=venom.STRATEGY_DENSE_K, cta_pair=pair)
            check_spmm(C, C_ref, dt)


def test_spmm_identity_probe_exact_densek():
    """P6 through the dense-K strategy: B = I => C == decompress(A) exactly."""
    for (R, K, V, M, dt) in [(256, 256, 128, 8, F16), (128, 512, 16, 16, F16), (256, 256, 64, 4, BF16)]:
        A = synth.gaussian((R, K), 1.0, dt, 79)
        vals, meta, cidx = oracle.compress(A, dt, V=V, M=M)
        D = oracle.decompress(vals, meta, cidx, R, K, dt, V, M)
        I = to_dev(f64_to_bits(np.eye(K), dt), dt)
        C = venom.spmm(vnm_from((vals, meta, cidx), R, K, V, M, dt), I, strategy=venom.STRATEGY_DENSE_K)
        assert np.array_equal(bits_to_f64(to_bits(C), dt), bits_to_f64(D, dt)), (R, K, V, M, dt)


def tc_order(meta: np.ndarray, R: int, G: int) -> np.ndarray:
    """The tensor-core metadata order include/venom.h states, written out: uint32[mt][ks][L][kb]."""
    nks = (G + 31) // 32
    mt_n = (R + 127) // 128

    def half(row, g0):  # nibbles of groups g0 .. g0+3; rows >= R and groups >= G: the 0x4 code
        h = 0
        for t in range(4):
            g = g0 + t
            nib = (int(meta[row, g // 2]) >> (4 * (g & 1))) & 0xF if (row < R and g < G) else 0x4
            h |= nib << (4 * t)
        return h
    exp = np.zeros((mt_n, nks, 128, 4), np.uint32)
    for mt in range(mt_n):
        for ks in range(nks):
            for L in range(128):
                ra = mt * 128 + (L & 7) + 16 * (L >> 4)
                for kb in range(4):
                    g0 = ks * 32 + kb * 8 + 4 * ((L >> 3) & 1)
                    exp[mt, ks, L, kb] = half(ra, g0) | (half(ra + 8, g0) << 16)
    return exp


@pytest.mark.parametrize("R,K,V,M", [(256, 512, 128, 8), (200, 256, 8, 4), (64, 1280, 64, 40),
                                     (384, 640, 128, 20), (64, 330, 64, 10), (130, 2040, 13, 40)])
def test_order_metadata_layout(R, K, V, M):
    """venom_order_metadata against the permutation include/venom.h states."""
    A = synth.gaussian((R, K), 1.0, F16, 31)
    vals, meta, cidx = oracle.compress(A, F16, V=V, M=M)
    x = vnm_from((vals, meta, cidx), R, K, V, M, F16)
    venom.order_metadata(x)
    exp = tc_order(meta, R, K // M)
    assert np.array_equal(x.metadata_tc.cpu().numpy().view(np.uint32).reshape(exp.shape), exp)


@pytest.mark.parametrize("R,K,V,M,kind,dt", [
    (1024, 4096, 64, 8, "gauss", F16),      # BERT-large FFN2 shape
    (192, 1040, 64, 8, "int", F16),         # ragged last row tile; partial last k-stage
    (256, 768, 256, 16, "gauss", BF16),     # V = 256 (128-column CTA chunks)
    (96, 512, 32, 32, "special", F16),      # V = 32, ragged rows
    (160, 384, 16, 8, "sparse", BF16),      # V = 16
])
def test_compress_2to4_fused(R, K, V, M, kind, dt):
    """venom_compress_2to4 == venom_compress (bit-exact canonical arrays) + the oracle's V:2:4
    re-encoding (values) + the tensor-core order of the re-encoded metadata; SpMM on it == oracle."""
    A = make_input(R, K, kind, dt, 13 + R + K, M)
    parts = oracle.compress(A, dt, V=V, M=M)
    v2, m2, c2 = oracle.expand_2to4(*parts, R, K, V, M)
    x, y = venom.compress_2to4(to_dev(A, dt), V=V, M=M, check=True)
    torch.cuda.synchronize()
    assert np.array_equal(to_bits(x.values).reshape(parts[0].shape), parts[0])
    assert np.array_equal(x.metadata.cpu().numpy(), parts[1])
    assert np.array_equal(x.column_idx.cpu().numpy(), parts[2])
    assert np.array_equal(to_bits(y.values).reshape(v2.shape), v2)
    exp = tc_order(m2, R, K // 4)
    assert np.array_equal(y.metadata_tc.cpu().numpy().view(np.uint32)[:exp.size].reshape(exp.shape), exp)
    if kind != "special":  # max-finite inputs overflow the fp16 product legitimately
        T = 136
        B = synth.gaussian((K, T), 1.0, dt, 14 + R)
        C = venom.spmm(y, to_dev(B, dt))
        check_spmm(C, oracle.spmm(*parts, R, K, dt, V, M, B), dt)


def test_spmm_ldb_ldc_views_and_shard_equality():
    """B/C column slices through ldb/ldc (the multi-GPU T-split): each shard equals the matching
    columns of the full product bit-for-bit (no split-K: same accumulation order)."""
    R, K, T, V, M, dt = 256, 1024, 512, 128, 16, F16
    A, B, bv, parts = oracle_problem(R, K, T, V, M, dt, 900, True)
    x = vnm_from(parts, R, K, V, M, dt)
    Bd = to_dev(B, dt)
    bias = to_dev(bv, dt)
    full = venom.spmm(x, Bd, bias=bias)
    Cbig = torch.zeros((R, T), dtype=tdt(dt), device="cuda")
    for r in range(4):
        sl = slice(r * T // 4, (r + 1) * T // 4)
        venom.spmm(x, Bd[:, sl], bias=bias, out=Cbig[:, sl])
    assert torch.equal(full.view(torch.int16), Cbig.view(torch.int16))
    check_spmm(full, oracle.spmm(*parts, R, K, dt, V, M, B, bias=bv), dt)


def test_spmm_zero_A_gives_bias():
    R, K, T, V, M, dt = 128, 256, 64, 64, 8, F16
    A = np.zeros((R, K), np.uint16)
    parts = oracle.compress(A, dt, V=V, M=M)
    bv = synth.gaussian((R,), 1.0, dt, 3)
    B = synth.gaussian((K, T), 1.0, dt, 4)
    C = venom.spmm(vnm_from(parts, R, K, V, M, dt), to_dev(B, dt), bias=to_dev(bv, dt))
    assert np.array_equal(to_bits(C), np.repeat(bv[:, None], T, axis=1))


def test_spmm_gpu_compress_then_spmm_matches_library_gemm():
    """End-to-end on the GPU path (compress -> spmm) vs the oracle, and vs cuBLAS on the
    GPU-decompressed matrix (library pin)."""
    R, K, T, V, M, dt = 512, 2048, 512, 128, 16, F16
    A = synth.gaussian((R, K), 0.02, dt, 61)
    B = synth.gaussian((K, T), 1.0, dt, 62)
    x = venom.compress(to_dev(A, dt), V=V, M=M, check=True)
    Bd = to_dev(B, dt)
    C = venom.spmm(x, Bd)
    parts = oracle.compress(A, dt, V=V, M=M)
    check_spmm(C, oracle.spmm(*parts, R, K, dt, V, M, B), dt)
    D = venom.decompress(x)
    ref = (D.float() @ Bd.float()).double().cpu().numpy()
    assert rel_fro(bits_to_f64(to_bits(C), dt), ref) <= TOL_FRO


def test_spmm_reads_only_selected_rows():
    """Rows of B that no block selects are poisoned with NaN: the output stays finite
    (PAPER.md:231 'load only the rows of B selected by column-loc')."""
    R, K, T, V, M, dt = 256, 1024, 128, 128, 16, F16
    A, B, _, parts = oracle_problem(R, K, T, V, M, dt, 70)
    cidx = parts[2]
    used = set()
    for rb in range(R // V):
        for g in range(K // M):
            used |= {g * M + int(c) for c in cidx[rb, g]}
    Bp = B.copy()
    for k in range(K):
        if k not in used:
            Bp[k] = 0x7E00
    C = venom.spmm(vnm_from(parts, R, K, V, M, dt), to_dev(Bp, dt))
    check_spmm(C, oracle.spmm(*parts, R, K, dt, V, M, B), dt)


@pytest.mark.parametrize("wl", ["bert_large_ffn2_1024x4096x4096_64:2:8",
                                "bert_large_ffn1_4096x1024x4096_64:2:8"])
def test_spmm_full_size_bert_sampled(wl):
    """BASELINE configs[1] at full size in the bench launch configuration: compressor bit-exact on
    every element; SpMM checked on 64 sampled output columns (all rows) against the oracle."""
    w = synth.WORKLOADS[wl]
    R, K, T, V, M = w["R"], w["K"], w["T"], w["V"], w["M"]
    sa, sb = synth.seeds(w["cfg"])
    A = synth.gaussian((R, K), 0.02, F16, sa)
    B = synth.gaussian((K, T), 1.0, F16, sb)
    x, got = gpu_compress(A, F16, V, M)
    parts = oracle.compress(A, F16, V=V, M=M)
    for g, e in zip(got, parts):
        assert np.array_equal(g.reshape(e.shape), e)
    cols = np.random.Generator(np.random.PCG64(1)).choice(T, size=64, replace=False)
    C_ref = oracle.spmm(*parts, R, K, F16, V, M, np.ascontiguousarray(B[:, cols]))
    Bd = to_dev(B, F16)
    for strat in strategies(K, V, M):
        C = venom.spmm(x, Bd, strategy=strat)
        check_spmm(C[:, torch.from_numpy(cols).cuda()], C_ref, F16)
    # bench.py's launch configuration: planner-chosen operand form + tensor-core-ordered metadata
    if venom.prefers_2to4(R, K, T, V, M):
        x2, y = venom.compress_2to4(to_dev(A, F16), V=V, M=M, check=True)
    else:
        y = venom.order_metadata(x)
    C = venom.spmm(y, Bd)
    check_spmm(C[:, torch.from_numpy(cols).cuda()], C_ref, F16)


def test_step_under_cuda_graph_matches_eager():
    """bench.py times the step as a CUDA graph replay: the captured launches (compress_2to4,
    spmm with tensor-core metadata, decompress on a second stream) give bit-identical results."""
    R, K, T, V, M = 512, 1024, 512, 64, 8
    A = to_dev(synth.gaussian((R, K), 0.02, F16, 41), F16)
    B = to_dev(synth.gaussian((K, T), 1.0, F16, 42), F16)
    x, y = venom.compress_2to4(A, V=V, M=M, check=True)
    C = torch.empty((R, T), dtype=torch.float16, device="cuda")
    D = torch.empty((R, K), dtype=torch.float16, device="cuda")
    side = torch.cuda.Stream()

    def step():
        venom.compress_2to4(A, V=V, M=M, out=(x, y))
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            venom.decompress(x, out=D)
        venom.spmm(y, B, out=C)
        torch.cuda.current_stream().wait_stream(side)
    step()
    torch.cuda.synchronize()
    C_eager, D_eager = C.clone(), D.clone()
    C.zero_()
    D.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    C.zero_()
    D.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(C.view(torch.int16), C_eager.view(torch.int16))
    assert torch.equal(D.view(torch.int16), D_eager.view(torch.int16))
    parts = oracle.compress(to_bits(A), F16, V=V, M=M)
    check_spmm(C, oracle.spmm(*parts, R, K, F16, V, M, to_bits(B)), F16)


@pytest.mark.parametrize("R,K,T,V,M,dt,bias", [
    (640, 512, 520, 64, 4, F16, True),      # ragged 512-row tile, ragged 240-column tile
    (1024, 1024, 480, 128, 4, BF16, False),
    (512, 2048, 240, 32, 4, F16, True),
    (1536, 256, 1000, 16, 4, F16, False),   # short K (2 k-stages), several tiles per CTA pair
])
def test_spmm_two_row_blocks_per_cta(R, K, T, V, M, dt, bias):
    """tile_t = 240: 512 × 240 CTA-pair tiles with two accumulators per CTA."""
    A, B, bv, parts = oracle_problem(R, K, T, V, M, dt, 800 + R + K + T, bias)
    C_ref = oracle.spmm(*parts, R, K, dt, V, M, B, bias=bv)
    x = venom.order_metadata(vnm_from(parts, R, K, V, M, dt))
    C = venom.spmm(x, to_dev(B, dt), bias=to_dev(bv, dt) if bias else None, tile_t=240)
    check_spmm(C, C_ref, dt)


def test_spmm_two_row_blocks_identity_and_2to4_form():
    """B = I through the 512 × 240 tiles is exact; and the fused V:2:4 form of a 64:2:8 matrix."""
    R, K, V, M = 768, 512, 64, 4
    A = synth.gaussian((R, K), 1.0, F16, 83)
    parts = oracle.compress(A, F16, V=V, M=M)
    D = oracle.decompress(*parts, R, K, F16, V, M)
    x = venom.order_metadata(vnm_from(parts, R, K, V, M, F16))
    C = venom.spmm(x, to_dev(f64_to_bits(np.eye(K), F16), F16), tile_t=240)
    assert np.array_equal(bits_to_f64(to_bits(C), F16), bits_to_f64(D, F16))
    R, K, T, V, M = 1024, 1024, 960, 64, 8
    A = synth.gaussian((R, K), 0.02, F16, 84)
    B = synth.gaussian((K, T), 1.0, F16, 85)
    _, y = venom.compress_2to4(to_dev(A, F16), V=V, M=M, check=True)
    C = venom.spmm(y, to_dev(B, F16), tile_t=240)
    parts = oracle.compress(A, F16, V=V, M=M)
    check_spmm(C, oracle.spmm(*parts, R, K, F16, V, M, B), F16)


def test_sparse_encoder_matches_dense_on_pruned_weights():
    """§8(f) rank 1: two BERT-large encoder layers with every linear layer 64:2:10 through
    venom_spmm equal the same encoder with torch fp32 GEMMs on the decompressed weights."""
    from paper_2310_02065_b200 import encoder as enc
    cfg = enc.EncoderConfig(layers=2, batch=2, seq=128)
    W = enc.init_weights(cfg, torch.device("cuda"), seed=3)
    model = enc.SparseEncoder(cfg, W)
    dense = model.dense_weights()
    x = (torch.randn(cfg.tokens, cfg.hidden, generator=torch.Generator().manual_seed(5))).half().cuda()
    ys = model.forward(x).float()
    d32 = [{k: (tuple(t.float() for t in v) if isinstance(v, tuple) else v.float()) for k, v in L.items()}
           for L in dense]
    yd = enc.dense_forward(cfg, d32, x.float())
    rel = float((ys - yd).norm() / yd.norm())
    # composite tolerance: the sparse encoder rounds to fp16 at ~8 points per layer (4 SpMM outputs,
    # SDPA, two LayerNorms, the attention transpose), the reference runs in fp32; each rounding adds
    # an RMS relative error of about 2^-11/sqrt(3) = 2.8e-4, and LayerNorm renormalises instead of
    # compounding, so 2 layers give about sqrt(16)·2.8e-4 = 1.1e-3 plus SDPA's own fp16 softmax;
    # 5e-3 leaves 2-4x headroom over that (measured: see the assertion message)
    assert rel <= 5e-3, rel


@pytest.mark.parametrize("dt", [F16])
def test_encoder_linear_layers_vs_oracle(dt):
    """§8(f) rank 1: each of an encoder layer's four V:N:M linear layers, called exactly as the
    encoder calls it (QKV / O / FFN2 token-major C, FFN1 with the GELU epilogue; 64:2:10 with K
    padded to 1040 / 4160), against the oracle's fp64 product on the oracle's own compression of
    the same padded weight, at the north-star tolerance."""
    import math
    from paper_2310_02065_b200 import encoder as enc
    cfg = enc.EncoderConfig(layers=1, batch=1, seq=264)  # T = 264: two 128-column tiles + a tail
    W = enc.init_weights(cfg, torch.device("cuda"), seed=11)
    model = enc.SparseEncoder(cfg, W)
    L, lw = model.layers[0], W[0]
    T = cfg.tokens
    erf = np.vectorize(math.erf)
    for key, wkey, bkey, tm, gelu in (("qkv", "wqkv", "bqkv", True, False), ("o", "wo", "bo", True, False),
                                      ("f1", "w1", "b1", False, True), ("f2", "w2", "b2", True, False)):
        lin = L[key]
        w = lw[wkey].cpu()
        Wp = torch.zeros((lin.out_f, lin.K), dtype=torch.float16)
        Wp[:, :lin.in_f] = w
        parts = oracle.compress(Wp.view(torch.int16).numpy().view(np.uint16), F16, V=cfg.V, M=cfg.M)
        xb = synth.gaussian((lin.K, T), 1.0, F16, 60 + len(key))
        xb[lin.in_f:] = 0  # the encoder's zero K-padding rows
        bits_b = lw[bkey].cpu().view(torch.int16).numpy().view(np.uint16)
        ref = oracle.spmm(*parts, lin.out_f, lin.K, F16, cfg.V, cfg.M, xb, bias=bits_b)
        if gelu and cfg.gelu == "tanh":
            ref = 0.5 * ref * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (ref + 0.044715 * ref ** 3)))
        elif gelu:
            ref = 0.5 * ref * (1.0 + erf(ref / math.sqrt(2.0)))
        out = torch.empty((T, lin.out_f) if tm else (lin.out_f, T), dtype=torch.float16, device="cuda")
        got = lin(to_dev(xb, F16), out=out, token_major=tm, gelu=cfg.gelu if gelu else False)
        check_spmm(got.t().contiguous() if tm else got, ref, F16)


# ------------------------------------------------------------------ masked compression + energy
# SURVEY §8(f) rank 4 (readings #20-#21): bit-exact against oracle.compress_masked, the
# SpMM on the masked operand against the oracle, energy within 1e-12 (fp64, summation order).
MASKED_CASES = [
    # (R, K, V, M, kind, dt, p_keep)
    (128, 512, 64, 8, "gauss", F16, 0.8),
    (256, 1024, 128, 16, "gauss", BF16, 0.5),
    (96, 280, 3, 7, "int", F16, 1.0),
    (64, 200, 32, 10, "special", BF16, 0.7),
    (40, 500, 1, 100, "gauss", F16, 0.9),
    (16, 768, 8, 256, "gauss", F16, 0.6),
]


@pytest.mark.parametrize("R,K,V,M,kind,dt,p_keep", MASKED_CASES)
def test_compress_masked_bit_exact_and_energy(R, K, V, M, kind, dt, p_keep):
    A = make_input(R, K, kind, dt, 900 + R + K + M, M)
    mask = synth.vnm_mask(R, K, V, M, 950 + R + M, p_keep=p_keep)
    ref = oracle.compress_masked(A, mask, dt, V=V, M=M)
    x = venom.compress_masked(to_dev(A, dt), torch.from_numpy(mask).cuda(), V=V, M=M, check=True)
    torch.cuda.synchronize()
    assert np.array_equal(to_bits(x.values), ref[0])
    assert np.array_equal(x.metadata.cpu().numpy(), ref[1])
    assert np.array_equal(x.column_idx.cpu().numpy(), ref[2])
    e = venom.energy(to_dev(A, dt), x).cpu().numpy()
    e_ref = oracle.energy(A, ref[0], dt)
    assert e[0] == pytest.approx(e_ref[0], rel=1e-12, abs=1e-300)
    assert e[1] == pytest.approx(e_ref[1], rel=1e-12, abs=1e-300)
    assert e[2] == pytest.approx(e_ref[2], rel=1e-12)


def test_compress_masked_golden_and_invalid_masks_on_gpu():
    for name in ("P7_masked_compress.json", "P8_masked_fill.json"):
        g = load_golden(name)
        A = f64_to_bits(np.array(g["A"], np.float64), F16)
        x = venom.compress_masked(to_dev(A, F16), torch.tensor(g["mask"], dtype=torch.uint8).cuda(),
                                  V=g["V"], M=g["M"], check=True)
        assert x.column_idx.cpu().numpy().tolist() == g["expected_column_idx"]
        assert x.metadata.cpu().numpy().tolist() == g["expected_metadata"]
        assert bits_to_f64(to_bits(x.values), F16).tolist() == g["expected_values"]
        assert float(venom.energy(to_dev(A, F16), x)[2]) == pytest.approx(g["expected_energy"], rel=1e-15)
    A = synth.gaussian((4, 16), 1.0, F16, 5)
    m = np.zeros((4, 16), np.uint8)
    m[0, [0, 1]] = 1
    m[1, [2, 3]] = 1
    m[2, [4]] = 1          # a fifth column in one V x M block
    with pytest.raises(venom.VenomError) as ei:
        venom.compress_masked(to_dev(A, F16), torch.from_numpy(m).cuda(), V=4, M=8, check=True)
    assert ei.value.status == 10
    m[:] = 0
    m[3, [8, 9, 10]] = 1   # three kept entries in one row-group
    with pytest.raises(venom.VenomError) as ei:
        venom.compress_masked(to_dev(A, F16), torch.from_numpy(m).cuda(), V=4, M=8, check=True)
    assert ei.value.status == 10


def test_spmm_on_masked_operand_matches_oracle():
    """The masked operand runs through the unchanged SpMM (gathered and pre-ordered paths)."""
    R, K, T, V, M = 256, 1024, 256, 128, 8
    A = synth.gaussian((R, K), 0.02, F16, 31)
    B = synth.gaussian((K, T), 1.0, F16, 32)
    mask = synth.vnm_mask(R, K, V, M, 33)
    v, md, c = oracle.compress_masked(A, mask, F16, V=V, M=M)
    C_ref = oracle.spmm(v, md, c, R, K, F16, V, M, B)
    x = venom.compress_masked(to_dev(A, F16), torch.from_numpy(mask).cuda(), V=V, M=M, check=True)
    check_spmm(venom.spmm(x, to_dev(B, F16)), C_ref, F16)
    venom.order_metadata(x)
    check_spmm(venom.spmm(x, to_dev(B, F16), strategy=venom.STRATEGY_GATHER), C_ref, F16)


# ------------------------------------------------------------------ full size GPT-3, degenerate shapes
def test_spmm_full_size_gpt3_sampled():
    """BASELINE configs[3] (GPT-3 FFN 12288×49152×8192 at 128:2:16) at full size in the bench's
    launch configuration (gathered kernel, tensor-core-ordered metadata). A and B are drawn on the
    GPU (bench recipe); the compressor is checked bit-exactly on sampled row blocks (compression is
    independent per V-row block) and the SpMM on those rows × 32 sampled columns against the oracle."""
    w = synth.WORKLOADS["gpt3_ffn_12288x49152x8192_128:2:16"]
    R, K, T, V, M = w["R"], w["K"], w["T"], w["V"], w["M"]
    sa, sb = synth.seeds(w["cfg"])
    A = synth.gaussian_device((R, K), 0.02, F16, sa, "cuda")
    B = synth.gaussian_device((K, T), 1.0, F16, sb, "cuda")
    x = venom.compress(A, V=V, M=M, check=True)
    y = venom.order_metadata(x)
    C = venom.spmm(y, B)
    torch.cuda.synchronize()
    rng = np.random.Generator(np.random.PCG64(3))
    cols = np.sort(rng.choice(T, size=32, replace=False))
    Bs = to_bits(B[:, torch.from_numpy(cols).cuda()])
    for rb in (0, 37, R // V - 1):
        rows = slice(rb * V, rb * V + V)
        Ab = to_bits(A[rows])
        v, md, c = oracle.compress(Ab, F16, V=V, M=M)
        assert np.array_equal(to_bits(x.values[rows]), v)
        assert np.array_equal(x.metadata[rows].cpu().numpy(), md)
        assert np.array_equal(x.column_idx[rb:rb + 1].cpu().numpy(), c)
        C_ref = oracle.spmm(v, md, c, V, K, F16, V, M, Bs)
        check_spmm(C[rows][:, torch.from_numpy(cols).cuda()], C_ref, F16)


def test_spmm_degenerate_shapes():
    """Empty and minimal problems (include/venom.h): T = 8 (the minimum), one V-block, K = 0
    (C = bias), R = 0 and T = 0 (nothing to do, no error)."""
    # T = 8, a single 64-row block
    R, K, T, V, M = 64, 256, 8, 64, 8
    A = synth.gaussian((R, K), 0.02, F16, 61)
    B = synth.gaussian((K, T), 1.0, F16, 62)
    parts = oracle.compress(A, F16, V=V, M=M)
    C_ref = oracle.spmm(*parts, R, K, F16, V, M, B)
    x = venom.compress(to_dev(A, F16), V=V, M=M, check=True)
    check_spmm(venom.spmm(x, to_dev(B, F16)), C_ref, F16)
    venom.order_metadata(x)
    check_spmm(venom.spmm(x, to_dev(B, F16)), C_ref, F16)
    # K = 0: C = bias broadcast (nothing to multiply)
    bias = to_dev(synth.gaussian((128,), 0.5, F16, 63), F16)
    x0 = venom.compress(torch.empty((128, 0), dtype=torch.float16, device="cuda"), V=64, M=8)
    C0 = venom.spmm(x0, torch.empty((0, 16), dtype=torch.float16, device="cuda"), bias=bias)
    torch.cuda.synchronize()
    assert torch.equal(C0, bias[:, None].expand(128, 16))
    # R = 0 and T = 0
    xr = venom.compress(torch.empty((0, 64), dtype=torch.float16, device="cuda"), V=64, M=8)
    assert venom.spmm(xr, torch.randn(64, 16, device="cuda").half()).shape == (0, 16)
    assert venom.spmm(x, torch.empty((K, 0), dtype=torch.float16, device="cuda")).shape == (R, 0)


@pytest.mark.parametrize("R,K,T,V,M,dt,bias", [
    (192, 640, 136, 64, 10, F16, True),    # encoder's 64:2:10 (gathered, two V-blocks per tile)
    (320, 960, 200, 64, 10, BF16, False),  # V = 64, 2.5 row tiles, T tail (16-row C^T boxes)
    (224, 640, 72, 32, 10, F16, True),     # V = 32: seven blocks (the last tile's fourth is padding)
    (384, 1024, 200, 128, 16, BF16, False),
    (512, 1024, 264, 128, 4, F16, True),   # 2:4 (contiguous, CTA pair)
    (130, 256, 64, 13, 8, F16, True),      # dense-K-only V -> rejected for token-major C
])
def test_spmm_transposed_output(R, K, T, V, M, dt, bias):
    """Token-major C^T (opts.c_transposed): bitwise the transpose of the row-major result (same
    accumulation and rounding) and within tolerance of the oracle; unsupported paths are refused."""
    A, B, bv, parts = oracle_problem(R, K, T, V, M, dt, 800 + R + T + M, bias)
    C_ref = oracle.spmm(*parts, R, K, dt, V, M, B, bias=bv)
    x = vnm_from(parts, R, K, V, M, dt)
    bd = to_dev(bv, dt) if bias else None
    can = (M == 4 or V in (32, 64) or V % 128 == 0) and (K // M) % 4 == 0
    if not can:
        with pytest.raises(venom.VenomError) as ei:
            venom.spmm(x, to_dev(B, dt), bias=bd, transposed_out=True)
        assert ei.value.status == 1
        return
    for pre in (False, True):
        if pre:
            venom.order_metadata(x)
        C = venom.spmm(x, to_dev(B, dt), bias=bd)
        Ct = venom.spmm(x, to_dev(B, dt), bias=bd, transposed_out=True)
        assert Ct.shape == (T, R)
        assert torch.equal(Ct.t(), C)
        check_spmm(Ct.t().contiguous(), C_ref, dt)
    # a wider leading dimension (a column slice of a [T, 3R] buffer, as the encoder's QKV uses)
    buf = torch.full((T, R + 64), float("nan"), dtype=tdt(dt), device="cuda")
    venom.spmm(x, to_dev(B, dt), bias=bd, transposed_out=True, out=buf[:, :R])
    assert torch.equal(buf[:, :R].t(), C) and torch.isnan(buf[:, R:]).all()
    with pytest.raises(venom.VenomError):
        venom.spmm(x, to_dev(B, dt), bias=bd, transposed_out=True, strategy=venom.STRATEGY_DENSE_K)


def test_encoder_layout_helpers():
    """include/venom_encoder.h: add+LayerNorm (token-major out within 1 ulp of torch's fp32-internal
    layer_norm, feature-major copy bitwise its transpose) and the attention-output transpose (exact)."""
    torch.manual_seed(5)
    for dt in (torch.float16, torch.bfloat16):
        T, h = 96, 1024
        x = torch.randn(T, h, device="cuda").to(dt)
        y = torch.randn(T, h, device="cuda").to(dt)
        w = (1 + 0.1 * torch.randn(h, device="cuda")).to(dt)
        b = (0.1 * torch.randn(h, device="cuda")).to(dt)
        out = torch.empty_like(x)
        fm = torch.full((h, T + 8), float("nan"), dtype=dt, device="cuda")
        venom.enc_add_layernorm(x, y, w, b, 1e-12, out, fm)
        ref = torch.nn.functional.layer_norm((x.float() + y.float()), (h,), w.float(), b.float(), 1e-12)
        ulp = 2.0 ** -10 if dt == torch.float16 else 2.0 ** -7
        assert ((out.float() - ref).abs() <= ulp * ref.abs() + 1e-3).all()
        assert torch.equal(fm[:, :T], out.t()) and torch.isnan(fm[:, T:]).all()
        # attention output [B, H, S, D], also as a transposed view ([B, S, H, D] storage)
        Bt, H, S, D = 2, 4, 128, 64
        for a in (torch.randn(Bt, H, S, D, device="cuda").to(dt),
                  torch.randn(Bt, S, H, D, device="cuda").to(dt).transpose(1, 2)):
            o = torch.empty((H * D, Bt * S), dtype=dt, device="cuda")
            venom.enc_heads_to_fm(a, o)
            assert torch.equal(o, a.permute(1, 3, 0, 2).reshape(H * D, Bt * S))


@pytest.mark.parametrize("R,K,T,V,M,dt,bias,tile_t,pair", [
    (512, 1024, 512, 128, 4, F16, True, 256, 0),   # 2:4, CTA pair 256 x 256
    (384, 640, 264, 64, 4, BF16, False, 128, 0),   # pair 256 x 128, ragged R and T
    (256, 512, 256, 128, 4, F16, True, 256, 1),    # one CTA per 128 rows, 256 columns
])
def test_spmm_kmajor_b(R, K, T, V, M, dt, bias, tile_t, pair):
    """K-major B (opts.b_kmajor, token-major activations [T, K]): bitwise the row-major-B result
    (the MMA reads the same values in the same K order), for row-major and token-major C."""
    A, B, bv, parts = oracle_problem(R, K, T, V, M, dt, 900 + R + T, bias)
    C_ref = oracle.spmm(*parts, R, K, dt, V, M, B, bias=bv)
    x = vnm_from(parts, R, K, V, M, dt)
    bd = to_dev(bv, dt) if bias else None
    Bd = to_dev(B, dt)
    Bt = Bd.t().contiguous()  # [T, K]
    for pre in (False, True):
        if pre:
            venom.order_metadata(x)
        kw = dict(bias=bd, tile_t=tile_t, cta_pair=pair, strategy=venom.STRATEGY_GATHER)
        C = venom.spmm(x, Bd, **kw)
        Ck = venom.spmm(x, Bt, b_kmajor=True, **kw)
        assert torch.equal(Ck, C)
        check_spmm(Ck, C_ref, dt)
        Ckt = venom.spmm(x, Bt, b_kmajor=True, transposed_out=True, **kw)
        assert torch.equal(Ckt.t(), C)


def test_spmm_kmajor_b_on_2to4_form_is_torch_linear():
    """The #18 V:2:4 form with K-major B and token-major C is F.linear on PyTorch-layout activations."""
    R, K, T, V, M = 1024, 1024, 512, 64, 8
    torch.manual_seed(3)
    W = (torch.randn(R, K, device="cuda") * 0.02).half()
    X = torch.randn(T, K, device="cuda").half()
    x, y = venom.compress_2to4(W, V=V, M=M, check=True)
    Y = venom.spmm(y, X, b_kmajor=True, transposed_out=True)
    ref = torch.nn.functional.linear(X.float(), venom.decompress(x).float())
    assert (Y.float() - ref).norm() / ref.norm() <= 2e-3
    assert torch.equal(Y.t(), venom.spmm(y, X.t().contiguous()))
    # the gathered (M = 8) operand itself with the same K-major activations: B^T transposed into
    # the scratch first, then bitwise the feature-major result
    venom.order_metadata(x)
    assert torch.equal(venom.spmm(x, X, b_kmajor=True), venom.spmm(x, X.t().contiguous()))


@pytest.mark.parametrize("R,K,T,V,M,dt,ct", [
    (256, 1040, 264, 64, 10, F16, False),   # the encoder's 64:2:10, ragged T
    (384, 1024, 200, 128, 16, BF16, True),  # token-major C too: F.linear on [T, K] activations
    (192, 2080, 72, 32, 40, F16, False),    # V = 32, a wider ldb (a column slice of [T, K + 8])
])
def test_spmm_kmajor_b_gathered(R, K, T, V, M, dt, ct):
    """K-major B for the gathered operand (b_kmajor with M > 4): the token-major activations are
    transposed into the scratch (vnm_transpose16_kernel) and the feature-major path runs on them —
    bitwise its result, and against the oracle."""
    A, B, bv, parts = oracle_problem(R, K, T, V, M, dt, 950 + R + T, True)
    C_ref = oracle.spmm(*parts, R, K, dt, V, M, B, bias=bv)
    x = venom.order_metadata(vnm_from(parts, R, K, V, M, dt))
    Bd, bd = to_dev(B, dt), to_dev(bv, dt)
    wide = torch.zeros((T, K + 8), dtype=tdt(dt), device="cuda")
    wide[:, :K] = Bd.t()
    Bt = wide[:, :K] if V == 32 else Bd.t().contiguous()
    C = venom.spmm(x, Bd, bias=bd, transposed_out=ct)
    Ck = venom.spmm(x, Bt, bias=bd, b_kmajor=True, transposed_out=ct)
    assert torch.equal(Ck, C)
    check_spmm(Ck.t().contiguous() if ct else Ck, C_ref, dt)


@pytest.mark.parametrize("R,K,T,V,M,dt", [(256, 1040, 264, 64, 10, F16), (512, 1024, 256, 128, 4, BF16),
                                          (384, 1024, 200, 128, 16, F16)])
def test_spmm_gelu_epilogue(R, K, T, V, M, dt):
    """opts.activation = GELU: C = gelu(A·B + bias), gelu(v) = v·Φ(v) in fp32 before the output
    rounding; against the oracle's fp64 product passed through the fp64 erf GELU."""
    import math
    A, B, bv, parts = oracle_problem(R, K, T, V, M, dt, 300 + R + M, True)
    C_lin = oracle.spmm(*parts, R, K, dt, V, M, B, bias=bv)
    erf = np.vectorize(math.erf)
    C_ref = 0.5 * C_lin * (1.0 + erf(C_lin / math.sqrt(2.0)))
    C_tanh = 0.5 * C_lin * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (C_lin + 0.044715 * C_lin ** 3)))
    x = vnm_from(parts, R, K, V, M, dt)
    for pre in (False, True):
        if pre:
            venom.order_metadata(x)
        check_spmm(venom.spmm(x, to_dev(B, dt), bias=to_dev(bv, dt), gelu=True), C_ref, dt)
        # the tanh form (opts.activation = 2, hardware tanh.approx) against its fp64 definition
        check_spmm(venom.spmm(x, to_dev(B, dt), bias=to_dev(bv, dt), gelu="tanh"), C_tanh, dt)
    with pytest.raises(venom.VenomError):
        venom.spmm(x, to_dev(B, dt), gelu=True, transposed_out=True)


def test_tensor_parallel_allgather_on_gpu():
    """paper_2310_02065_b200/tp.py over NCCL (a one-rank group on this GPU): token-major local SpMM +
    all_gather_into_tensor gives C^T of the full product, bitwise venom.spmm's C transposed."""
    import socket
    import torch.distributed as dist
    from paper_2310_02065_b200 import tp
    R, K, T, V, M = 256, 512, 256, 128, 8
    A, B, bv, parts = oracle_problem(R, K, T, V, M, F16, 77, True)
    x = vnm_from(parts, R, K, V, M, F16)
    venom.order_metadata(x)
    created = False
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", world_size=1, rank=0)
        created = True
    try:
        Bd, bd = to_dev(B, F16), to_dev(bv, F16)
        t0, t1 = tp.t_slice(T, dist.get_world_size(), dist.get_rank())
        Ct = tp.spmm_tp_allgather(x, Bd[:, t0:t1], bias=bd)
        torch.cuda.synchronize()
        assert Ct.shape == (T, R)
        assert torch.equal(Ct.t(), venom.spmm(x, Bd, bias=bd))
    finally:
        if created:
            dist.destroy_process_group()


def test_tensor_parallel_row_split_on_gpu():
    """tp's row split (V-block-aligned weight shards): each "rank" runs the
    SpMM on its shard_rows operand; (a) the shards' row blocks stacked equal the unsharded C bit
    for bit; (b) the fused variant's epilogue fan-out, emulated with one local buffer per rank and
    each shard storing into every other buffer at its row offset (the addressing of
    tp.peer_row_slices), fills every buffer with the full C; (c) the one-rank NCCL group runs
    spmm_tp_rows_allgather end to end."""
    import socket
    import torch.distributed as dist
    from paper_2310_02065_b200 import tp
    for (R, K, T, V, M, world) in [(512, 512, 136, 128, 16, 2), (384, 640, 200, 64, 10, 3), (256, 330, 64, 64, 10, 2)]:
        A, B, bv, parts = oracle_problem(R, K, T, V, M, F16, 83 + R, True)
        x = venom.order_metadata(vnm_from(parts, R, K, V, M, F16))
        Bd, bd = to_dev(B, F16), to_dev(bv, F16)
        C_full = venom.spmm(x, Bd, bias=bd)
        check_spmm(C_full, oracle.spmm(*parts, R, K, F16, V, M, B, bias=bv), F16)
        bufs = [torch.full((R, T), float("nan"), dtype=torch.float16, device="cuda") for _ in range(world)]
        blocks = []
        for rank in range(world):
            r0, r1 = tp.row_slice(R, V, world, rank)
            xr = venom.order_metadata(tp.shard_rows(x, r0, r1))
            blocks.append(venom.spmm(xr, Bd, bias=bd[r0:r1]))
            peers = [bufs[q][r0:r1] for q in range(world) if q != rank]
            venom.spmm(xr, Bd, bias=bd[r0:r1], out=bufs[rank][r0:r1], c_peers=peers)
        torch.cuda.synchronize()
        assert torch.equal(torch.cat(blocks, 0), C_full), (R, V, M)
        for q in range(world):
            assert torch.equal(bufs[q], C_full), (R, V, M, q)
    created = False
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", world_size=1, rank=0)
        created = True
    try:
        r0, r1 = tp.row_slice(R, V, dist.get_world_size(), dist.get_rank())
        xr = venom.order_metadata(tp.shard_rows(x, r0, r1))
        C = tp.spmm_tp_rows_allgather(xr, Bd, bias_rows=bd[r0:r1])
        torch.cuda.synchronize()
        assert torch.equal(C, C_full)
    finally:
        if created:
            dist.destroy_process_group()


def test_spmm_argument_errors_are_synchronous():
    """out-of-range cta_pair, a non-zero stages override and misaligned metadata /
    column_idx views return VENOM_ERR_INVALID_ARGUMENT before anything is launched."""
    R, K, T, V, M = 256, 512, 64, 128, 16
    A, B, bv, parts = oracle_problem(R, K, T, V, M, F16, 5, False)
    x = vnm_from(parts, R, K, V, M, F16)
    Bd = to_dev(B, F16)
    for kw in (dict(cta_pair=3), dict(cta_pair=-1), dict(stages=2)):
        with pytest.raises(venom.VenomError) as ei:
            venom.spmm(x, Bd, **kw)
        assert ei.value.status == 1, kw
    # a metadata view that is only 1-byte aligned (canonical metadata is read with 16-byte loads)
    meta_buf = torch.zeros(x.metadata.numel() + 16, dtype=torch.uint8, device=Bd.device)
    meta_view = meta_buf[1:1 + x.metadata.numel()].view(x.metadata.shape)
    meta_view.copy_(x.metadata)
    y = venom.VNMTensor(x.values, meta_view, x.column_idx, R, K, V, M)
    with pytest.raises(venom.VenomError) as ei:
        venom.spmm(y, Bd, use_metadata_tc=False)
    assert ei.value.status == 1
    # dense-K reads column_idx with 16-byte loads: a 4-byte-aligned view is refused there
    cbuf = torch.zeros(x.column_idx.numel() + 16, dtype=torch.uint8, device=Bd.device)
    cview = cbuf[4:4 + x.column_idx.numel()].view(x.column_idx.shape)
    cview.copy_(x.column_idx)
    z = venom.VNMTensor(x.values, x.metadata, cview, R, K, V, M)
    with pytest.raises(venom.VenomError) as ei:
        venom.spmm(z, Bd, strategy=venom.STRATEGY_DENSE_K)
    assert ei.value.status == 1
    torch.cuda.synchronize()


def test_compress_out_refreshes_tensor_core_metadata():
    """compress(A, out=x) on an operand that carries tensor-core-ordered metadata
    re-derives it, so spmm(x, B) pairs the new values with the new m-indices."""
    R, K, T, V, M = 256, 1024, 128, 128, 16
    A1 = synth.gaussian((R, K), 0.02, F16, 41)
    A2 = synth.gaussian((R, K), 0.02, F16, 42)
    B = synth.gaussian((K, T), 1.0, F16, 43)
    x = venom.order_metadata(venom.compress(to_dev(A1, F16), V=V, M=M))
    venom.compress(to_dev(A2, F16), V=V, M=M, out=x)
    C = venom.spmm(x, to_dev(B, F16))  # uses x.metadata_tc
    parts = oracle.compress(A2, F16, V=V, M=M)
    check_spmm(C, oracle.spmm(*parts, R, K, F16, V, M, B), F16)


@pytest.mark.parametrize("R,K,T,dt", [(256, 512, 128, F16), (1024, 4096, 512, F16), (512, 1024, 256, BF16)])
def test_spmm_m4_matches_cusparselt(R, K, T, dt):
    """SURVEY §8(c) M = 4 pin: plain 2:4 magnitude pruning (V:2:4) multiplied by cuSPARSELt
    (torch._cslt_sparse_mm on the same pruned weight, a library routine) agrees with venom_spmm
    within the north-star tolerance, and both with the oracle."""
    if not torch.backends.cusparselt.is_available():
        pytest.skip("cuSPARSELt not available in this torch build")
    A, B, _, parts = oracle_problem(R, K, T, 128, 4, dt, 61 + R + K, False)
    x = venom.order_metadata(vnm_from(parts, R, K, 128, 4, dt))
    Ap = venom.decompress(x)
    Bd = to_dev(B, dt)
    C_lt = torch._cslt_sparse_mm(torch._cslt_compress(Ap), Bd)
    C_v = venom.spmm(x, Bd)
    C_ref = oracle.spmm(*parts, R, K, dt, 128, 4, B)
    check_spmm(C_v, C_ref, dt)
    got_lt = C_lt.double().cpu().numpy()
    assert rel_fro(bits_to_f64(to_bits(C_v), dt), got_lt) <= TOL_FRO


def test_spmm_fused_allgather_fanout():
    """The fused all-gather's epilogue fan-out (opts.c_peers), on one GPU: peer buffers that are
    other allocations on this device must receive exactly this call's C — row-major C (TMA-store
    epilogue + copies from the staging slot) and token-major C, ragged edges included."""
    for (R, K, T, V, M, ct) in [(256, 512, 136, 128, 16, False), (192, 512, 256, 64, 8, True),
                                (256, 1024, 264, 128, 4, False), (384, 512, 200, 128, 16, True)]:
        A, B, bv, parts = oracle_problem(R, K, T, V, M, F16, 91 + R + T, True)
        x = venom.order_metadata(vnm_from(parts, R, K, V, M, F16))
        Bd, bd = to_dev(B, F16), to_dev(bv, F16)
        shape = (T, R) if ct else (R, T)
        peers = [torch.full(shape, float("nan"), dtype=torch.float16, device=Bd.device) for _ in range(3)]
        C = venom.spmm(x, Bd, bias=bd, transposed_out=ct, c_peers=peers)
        torch.cuda.synchronize()
        for q in peers:
            assert torch.equal(q, C)
        C_ref = oracle.spmm(*parts, R, K, F16, V, M, B, bias=bv)
        check_spmm(C.t() if ct else C, C_ref, F16)
    with pytest.raises(venom.VenomError):
        venom.spmm(x, Bd, c_peers=[peers[0]] * 9)
    with pytest.raises(venom.VenomError):
        venom.spmm(vnm_from(parts, R, K, V, M, F16), Bd, strategy=venom.STRATEGY_DENSE_K, c_peers=[peers[0]])


def test_tensor_parallel_fused_allgather_on_gpu():
    """tp.spmm_tp_fused_allgather over symmetric memory on a one-rank NCCL group: the full C^T in
    the symmetric buffer equals venom.spmm's C transposed (the peer fan-out itself is covered by
    test_spmm_fused_allgather_fanout; more ranks need more GPUs than this run has)."""
    import socket
    import torch.distributed as dist
    from paper_2310_02065_b200 import tp
    R, K, T, V, M = 256, 512, 256, 128, 16
    A, B, bv, parts = oracle_problem(R, K, T, V, M, F16, 79, True)
    x = venom.order_metadata(vnm_from(parts, R, K, V, M, F16))
    created = False
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", world_size=1, rank=0,
                                device_id=torch.device("cuda", 0))
        created = True
    try:
        Bd, bd = to_dev(B, F16), to_dev(bv, F16)
        try:
            buf, hdl = tp.fused_allgather_buffer(R, T, torch.float16, Bd.device)
        except Exception as e:  # symmetric memory unavailable in this build / environment
            pytest.skip(f"symmetric memory unavailable: {e!r}")
        t0, t1 = tp.t_slice(T, dist.get_world_size(), dist.get_rank())
        tp.spmm_tp_fused_allgather(x, Bd[:, t0:t1], buf, hdl, bias=bd)
        torch.cuda.synchronize()
        assert torch.equal(buf.t(), venom.spmm(x, Bd, bias=bd))
    finally:
        if created:
            dist.destroy_process_group()
