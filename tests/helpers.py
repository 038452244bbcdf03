"""Small numpy helpers shared by tests (no method arithmetic: bit-pattern <-> float views only)."""
from __future__ import annotations

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
F16, BF16 = 0, 1


def bits_to_f64(bits: np.ndarray, dtype: int) -> np.ndarray:
    bits = np.asarray(bits, dtype=np.uint16)
    if dtype == F16:
        return bits.view(np.float16).astype(np.float64)
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def f64_to_bits(x, dtype: int) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    if dtype == F16:
        return x.astype(np.float16).view(np.uint16)
    import torch
    return torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def load_golden(name: str) -> dict:
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def mask_from_compressed(metadata, column_idx, R, K, V, M):
    """Boolean keep-mask implied by (metadata, column_idx): written with numpy indexing, not by
    calling the oracle, so tests can cross-check the oracle's decompress."""
    G = K // M
    mask = np.zeros((R, K), bool)
    for i in range(R):
        for g in range(G):
            nib = (int(metadata[i, g // 2]) >> (4 * (g % 2))) & 0xF
            for p in (nib & 3, nib >> 2):
                mask[i, g * M + int(column_idx[i // V, g, p])] = True
    return mask


def rel_fro(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    if nb == 0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)
