"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no scoring, selection, packing or products):
it only draws random numbers and names workload shapes. Both sides receive identical 16-bit
patterns from here, so a parity test compares two independent computations on the same input.

Recipe: transformer-scaled weights A ~ N(0, 0.02^2), activations
B ~ N(0, 1), both rounded once to fp16 (or bf16); seeds A = 1000 + 10*cfg, B = 1001 + 10*cfg.
Special-value generators add the edge cases the tests need (ties, zeros, -0.0, subnormals,
the largest finite values).
"""
from __future__ import annotations

import numpy as np

F16, BF16 = 0, 1

# (name, R, K, T, V, M) — BASELINE.json configs; K padded per DESIGN.md reading #11.
WORKLOADS = {
    "tiny_128x128x128_64:2:8": dict(R=128, K=128, T=128, V=64, M=8, cfg=0),
    "bert_large_ffn2_1024x4096x4096_64:2:8": dict(R=1024, K=4096, T=4096, V=64, M=8, cfg=1),
    "bert_large_ffn1_4096x1024x4096_64:2:8": dict(R=4096, K=1024, T=4096, V=64, M=8, cfg=1),
    "sweep_4096x4096x4096_128:2:4": dict(R=4096, K=4096, T=4096, V=128, M=4, cfg=2),
    "sweep_4096x4096x4096_128:2:8": dict(R=4096, K=4096, T=4096, V=128, M=8, cfg=2),
    "sweep_4096x4096x4096_128:2:16": dict(R=4096, K=4096, T=4096, V=128, M=16, cfg=2),
    "sweep_4096x4096x4096_128:2:32": dict(R=4096, K=4096, T=4096, V=128, M=32, cfg=2),
    "sweep_4096x4160x4096_128:2:40": dict(R=4096, K=4160, T=4096, V=128, M=40, cfg=2),
    "sweep_4096x4096x4096_64:2:4": dict(R=4096, K=4096, T=4096, V=64, M=4, cfg=2),
    "sweep_4096x4096x4096_64:2:8": dict(R=4096, K=4096, T=4096, V=64, M=8, cfg=2),
    "sweep_4096x4096x4096_64:2:16": dict(R=4096, K=4096, T=4096, V=64, M=16, cfg=2),
    "sweep_4096x4096x4096_64:2:32": dict(R=4096, K=4096, T=4096, V=64, M=32, cfg=2),
    # V-scaling study (the paper's Fig 8 axis): V in {32, 256}
    "sweep_4096x4096x4096_32:2:8": dict(R=4096, K=4096, T=4096, V=32, M=8, cfg=2),
    "sweep_4096x4096x4096_32:2:16": dict(R=4096, K=4096, T=4096, V=32, M=16, cfg=2),
    "sweep_4096x4096x4096_32:2:32": dict(R=4096, K=4096, T=4096, V=32, M=32, cfg=2),
    "sweep_4096x4096x4096_256:2:8": dict(R=4096, K=4096, T=4096, V=256, M=8, cfg=2),
    "sweep_4096x4096x4096_256:2:16": dict(R=4096, K=4096, T=4096, V=256, M=16, cfg=2),
    "sweep_4096x4096x4096_256:2:32": dict(R=4096, K=4096, T=4096, V=256, M=32, cfg=2),
    "sweep_4096x4160x4096_64:2:40": dict(R=4096, K=4160, T=4096, V=64, M=40, cfg=2),
    # the paper's Fig 6 family: BERT-large-shaped 1024×K×4096 at V = 128,
    # N:M = 2:10 / 2:20 / 2:40 / 2:100 (K padded to a multiple of 8M, reading #11)
    "fig6_1024x4160x4096_128:2:10": dict(R=1024, K=4160, T=4096, V=128, M=10, cfg=1),
    "fig6_1024x4160x4096_128:2:20": dict(R=1024, K=4160, T=4096, V=128, M=20, cfg=1),
    "fig6_1024x4160x4096_128:2:40": dict(R=1024, K=4160, T=4096, V=128, M=40, cfg=1),
    "fig6_1024x4800x4096_128:2:100": dict(R=1024, K=4800, T=4096, V=128, M=100, cfg=1),
    "gpt3_ffn_12288x49152x8192_128:2:16": dict(R=12288, K=49152, T=8192, V=128, M=16, cfg=3),
    # the sparse BERT-large encoder's linear layers (configs[4]: 64:2:10, batch 32 x seq 512;
    # K padded to a multiple of 8M, reading #11)
    "enc_qkv_3072x1040x16384_64:2:10": dict(R=3072, K=1040, T=16384, V=64, M=10, cfg=4),
    "enc_o_1024x1040x16384_64:2:10": dict(R=1024, K=1040, T=16384, V=64, M=10, cfg=4),
    "enc_ffn1_4096x1040x16384_64:2:10": dict(R=4096, K=1040, T=16384, V=64, M=10, cfg=4),
    "enc_ffn2_1024x4160x16384_64:2:10": dict(R=1024, K=4160, T=16384, V=64, M=10, cfg=4),
}


def seeds(cfg: int):
    return 1000 + 10 * cfg, 1001 + 10 * cfg


def to_bits(x_f32: np.ndarray, dtype: int) -> np.ndarray:
    """Round float32 values once to fp16 / bf16 (round-to-nearest-even) and return uint16 bits."""
    x_f32 = np.ascontiguousarray(x_f32, dtype=np.float32)
    if dtype == F16:
        return x_f32.astype(np.float16).view(np.uint16)
    import torch
    return torch.from_numpy(x_f32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def gaussian(shape, std: float, dtype: int, seed: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return to_bits(rng.standard_normal(shape, dtype=np.float32) * np.float32(std), dtype)


def small_integers(shape, dtype: int, seed: int, lo: int = -3, hi: int = 3) -> np.ndarray:
    """Tie-heavy input: integers in [lo, hi] (exact in fp16 and bf16)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return to_bits(rng.integers(lo, hi + 1, size=shape).astype(np.float32), dtype)


def special_values(shape, dtype: int, seed: int) -> np.ndarray:
    """Mixture of zeros, -0.0, subnormals, the largest finite magnitude, and normals."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n = int(np.prod(shape))
    if dtype == F16:
        pool = np.array([0x0000, 0x8000, 0x0001, 0x8001, 0x03FF, 0x7BFF, 0xFBFF, 0x3C00, 0xBC00,
                         0x0400, 0x3555], np.uint16)
    else:
        pool = np.array([0x0000, 0x8000, 0x0001, 0x8001, 0x007F, 0x7F7F, 0xFF7F, 0x3F80, 0xBF80,
                         0x0080, 0x3EAA], np.uint16)
    pick = rng.integers(0, len(pool), size=n)
    out = pool[pick]
    normal = gaussian((n,), 1.0, dtype, seed + 7)
    use_normal = rng.random(n) < 0.4
    out = np.where(use_normal, normal, out).astype(np.uint16)
    return out.reshape(shape)


def sparse_columns(shape, dtype: int, seed: int, live_cols_per_block: int, M: int) -> np.ndarray:
    """Gaussian matrix where each M-column group keeps only `live_cols_per_block` (< 4) random
    columns non-zero: exercises blocks with fewer than 4 significant columns."""
    R, K = shape
    rng = np.random.Generator(np.random.PCG64(seed))
    a = gaussian(shape, 1.0, dtype, seed + 3)
    mask = np.zeros(shape, bool)
    for g in range(K // M):
        cols = rng.choice(M, size=live_cols_per_block, replace=False)
        mask[:, g * M + cols] = True
    return np.where(mask, a, np.uint16(0)).astype(np.uint16)


def gaussian_device(shape, std: float, dtype: int, seed: int, device):
    """Same distribution generated on the GPU (torch Philox) for bench-sized inputs."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    tdt = torch.float16 if dtype == F16 else torch.bfloat16
    x = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    return (x * std).to(tdt)


def vnm_mask(R: int, K: int, V: int, M: int, seed: int, max_cols: int = 4, max_keep: int = 2,
             p_keep: float = 0.8) -> np.ndarray:
    """A random keep-mask with V:N:M structure (uint8, 1 = keep): per V x M block a random set of
    at most `max_cols` columns, per row and group at most `max_keep` of them, each candidate kept
    with probability `p_keep` (so some blocks / rows use fewer — the fill cases). Stands in for an
    external pruner's output (e.g. second-order); no method arithmetic."""
    rng = np.random.default_rng(seed)
    mask = np.zeros((R, K), np.uint8)
    for rb in range(R // V):
        for g in range(K // M):
            ncols = int(rng.integers(0, max_cols + 1))
            cols = rng.choice(M, size=ncols, replace=False)
            for i in range(rb * V, rb * V + V):
                if ncols == 0:
                    continue
                k = int(rng.integers(0, min(max_keep, ncols) + 1))
                for c in rng.choice(cols, size=k, replace=False):
                    if rng.random() < p_keep:
                        mask[i, g * M + int(c)] = 1
    return mask
