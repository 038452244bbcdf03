"""a sparse BERT-large encoder forward on venom_spmm (PAPER.md:476-500,
BASELINE.json configs[4]: every linear layer V:N:M 64:2:10, batch 32 × seq 512).

The four linear layers of each encoder layer (QKV 3072×1024, attention output 1024×1024, FFN1
4096×1024, FFN2 1024×4096) run as V:N:M SpMMs through the C ABI; attention (torch SDPA),
GELU, residual adds and LayerNorm stay dense in torch, as in the paper's STen integration
(PAPER.md:443-474). The SpMM's B operand is feature-major ([features, tokens], DESIGN.md reading
#14); its output is written feature-major where the next op is another SpMM (FFN1 -> GELU -> FFN2)
and token-major (``transposed_out``) where attention or LayerNorm reads it (QKV, attention
output, FFN2), so the residual stream stays token-major as in the dense model and only the three
B operands that follow a token-major op (x, the attention output, the post-LN x1) are transposed.
K is padded to a multiple of 8·M with zero weight columns and zero activation rows (reading #11):
the padded activation buffers are allocated once with zero tails and only the real rows are written.

This module is a user of the library, not part of the hot path: every SpMM is venom_spmm; the
dense parts are plain torch ops.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional

import torch
import torch.nn.functional as F

from . import (VNMTensor, compress, compress_2to4, enc_add_layernorm, enc_heads_to_fm, order_metadata,
               prefers_2to4, spmm)


def padded(k: int, M: int) -> int:
    """K rounded up to a multiple of 8·M (reading #11)."""
    q = 8 * M
    return (k + q - 1) // q * q


class SparseLinear:
    """y_fm = W·x_fm + b with W in V:N:M (compressed once from a dense weight by magnitude,
    PAPER.md:187-189), executed by venom_spmm in the planner's operand form."""

    def __init__(self, weight: torch.Tensor, bias: Optional[torch.Tensor], V: int, M: int, T: int):
        out_f, in_f = weight.shape
        self.out_f, self.in_f = out_f, in_f
        self.K = padded(in_f, M)
        Wp = torch.zeros((out_f, self.K), dtype=weight.dtype, device=weight.device)
        Wp[:, :in_f] = weight
        if prefers_2to4(out_f, self.K, T, V, M):
            self.x, self.op = compress_2to4(Wp, V=V, M=M, check=True)
        else:
            self.x = compress(Wp, V=V, M=M, check=True)
            self.op = order_metadata(self.x)
        self.bias = bias

    def __call__(self, x_fm: torch.Tensor, out: Optional[torch.Tensor] = None,
                 token_major: bool = False, gelu=False) -> torch.Tensor:
        assert x_fm.shape[0] == self.K, (x_fm.shape, self.K)
        return spmm(self.op, x_fm, bias=self.bias, out=out, transposed_out=token_major, gelu=gelu)


@dataclass
class EncoderConfig:
    hidden: int = 1024
    heads: int = 16
    ffn: int = 4096
    layers: int = 24
    batch: int = 32
    seq: int = 512
    V: int = 64
    M: int = 10
    eps: float = 1e-12
    # GELU form: "tanh" as the original BERT (and GPT-2/3) define it, the hardware tanh in the SpMM
    # epilogue; "erf" is torch's default form (its erff epilogue costs FFN1 ~25%)
    gelu: str = "tanh"

    @property
    def tokens(self) -> int:
        return self.batch * self.seq


def init_weights(cfg: EncoderConfig, device, seed: int = 0, dtype=torch.float16):
    """Random-init BERT-large-shaped weights (no checkpoints: DESIGN.md input recipe)."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    h, f = cfg.hidden, cfg.ffn

    def w(o, i):
        return (torch.randn(o, i, generator=g) * 0.02).to(device=device, dtype=dtype)

    def b(o):
        return (torch.randn(o, generator=g) * 0.02).to(device=device, dtype=dtype)
    layers = []
    for _ in range(cfg.layers):
        layers.append(dict(wqkv=w(3 * h, h), bqkv=b(3 * h), wo=w(h, h), bo=b(h), w1=w(f, h), b1=b(f),
                           w2=w(h, f), b2=b(h), ln1_w=torch.ones(h, device=device, dtype=dtype),
                           ln1_b=torch.zeros(h, device=device, dtype=dtype),
                           ln2_w=torch.ones(h, device=device, dtype=dtype),
                           ln2_b=torch.zeros(h, device=device, dtype=dtype)))
    return layers


class SparseEncoder:
    """The encoder with V:N:M linear layers; `dense_weights()` returns the pruned weights
    (decompressed) for the dense cuBLAS baseline of the same model."""

    def __init__(self, cfg: EncoderConfig, weights: List[dict]):
        self.cfg = cfg
        T = cfg.tokens
        dev = weights[0]["wqkv"].device
        dt = weights[0]["wqkv"].dtype
        self.layers = []
        for lw in weights:
            L = dict(qkv=SparseLinear(lw["wqkv"], lw["bqkv"], cfg.V, cfg.M, T),
                     o=SparseLinear(lw["wo"], lw["bo"], cfg.V, cfg.M, T),
                     f1=SparseLinear(lw["w1"], lw["b1"], cfg.V, cfg.M, T),
                     f2=SparseLinear(lw["w2"], lw["b2"], cfg.V, cfg.M, T))
            for k in ("ln1_w", "ln1_b", "ln2_w", "ln2_b"):
                L[k] = lw[k]
            self.layers.append(L)
        L0 = self.layers[0]
        # feature-major B operands with zero K-padding rows (written only in [:real rows])
        self.x_fm = torch.zeros((L0["qkv"].K, T), dtype=dt, device=dev)
        self.attn_fm = torch.zeros((L0["o"].K, T), dtype=dt, device=dev)
        self.x1_fm = torch.zeros((L0["f1"].K, T), dtype=dt, device=dev)
        self.hid = torch.zeros((L0["f2"].K, T), dtype=dt, device=dev)
        # token-major SpMM outputs (transposed_out) and the feature-major FFN1 output
        self.qkv_tm = torch.empty((T, 3 * cfg.hidden), dtype=dt, device=dev)
        self.o_tm = torch.empty((T, cfg.hidden), dtype=dt, device=dev)
        self.f2_tm = torch.empty((T, cfg.hidden), dtype=dt, device=dev)

    def dense_weights(self) -> List[dict]:
        from . import decompress
        out = []
        for L in self.layers:
            d = {}
            for k in ("qkv", "o", "f1", "f2"):
                lin = L[k]
                d[k] = (decompress(lin.x)[:, :lin.in_f].contiguous(), lin.bias)
            for k in ("ln1_w", "ln1_b", "ln2_w", "ln2_b"):
                d[k] = L[k]
            out.append(d)
        return out

    def forward(self, x_tm: torch.Tensor) -> torch.Tensor:
        """x_tm: [tokens, hidden] (token-major, as a user holds it); returns the same layout."""
        h = self.cfg.hidden
        self.x_fm[:h].copy_(x_tm.t())  # the first layer's B operand; later ones come from LayerNorm
        x = x_tm
        for L in self.layers:
            x = self._layer(L, x)
        return x

    def _attention(self, qkv_tm: torch.Tensor, out_fm: torch.Tensor):
        cfg = self.cfg
        Bt, S, H = cfg.batch, cfg.seq, cfg.heads
        h = cfg.hidden
        D = h // H
        # token-major [T, 3h] straight from the QKV SpMM: [B, H, S, D] views for SDPA (flash)
        q, k, v = (qkv_tm[:, i * h:(i + 1) * h].view(Bt, S, H, D).transpose(1, 2) for i in range(3))
        a = F.scaled_dot_product_attention(q, k, v)  # [B, H, S, D]
        enc_heads_to_fm(a, out_fm)  # the O projection's B operand, feature-major [h, T]

    def _layer(self, L: dict, x: torch.Tensor) -> torch.Tensor:
        cfg = self.cfg
        h = cfg.hidden
        # x: token-major residual stream; self.x_fm: the same values feature-major (QKV's B)
        L["qkv"](self.x_fm, out=self.qkv_tm, token_major=True)
        self._attention(self.qkv_tm, self.attn_fm)
        L["o"](self.attn_fm, out=self.o_tm, token_major=True)
        x1 = torch.empty_like(x)
        enc_add_layernorm(x, self.o_tm, L["ln1_w"], L["ln1_b"], cfg.eps, x1, self.x1_fm)
        L["f1"](self.x1_fm, out=self.hid[:cfg.ffn], gelu=cfg.gelu)  # GELU in the epilogue; FFN2's B
        L["f2"](self.hid, out=self.f2_tm, token_major=True)
        out = torch.empty_like(x)
        enc_add_layernorm(x1, self.f2_tm, L["ln2_w"], L["ln2_b"], cfg.eps, out, self.x_fm)
        return out


def dense_forward(cfg: EncoderConfig, dense: List[dict], x_tm: torch.Tensor) -> torch.Tensor:
    """The same encoder with dense cuBLAS GEMMs on the pruned (decompressed) weights, token-major
    (the usual torch layout) — the paper's dense baseline."""
    Bt, S, H = cfg.batch, cfg.seq, cfg.heads
    h = cfg.hidden
    D = h // H
    x = x_tm
    for L in dense:
        w, b = L["qkv"]
        qkv = torch.addmm(b, x, w.t())  # [T, 3h]
        q, k, v = (qkv[:, i * h:(i + 1) * h].view(Bt, S, H, D).transpose(1, 2) for i in range(3))
        a = F.scaled_dot_product_attention(q, k, v).transpose(1, 2).reshape(Bt * S, h)
        w, b = L["o"]
        x = F.layer_norm(x + torch.addmm(b, a, w.t()), (h,), L["ln1_w"], L["ln1_b"], cfg.eps)
        w, b = L["f1"]
        f = F.gelu(torch.addmm(b, x, w.t()), approximate="tanh" if cfg.gelu == "tanh" else "none")
        w, b = L["f2"]
        x = F.layer_norm(x + torch.addmm(b, f, w.t()), (h,), L["ln2_w"], L["ln2_b"], cfg.eps)
    return x


def useful_flops(cfg: EncoderConfig) -> float:
    """Useful FLOPs of the sparse linear layers per forward: 2·nnz·T summed (nnz = out·in·2/M)."""
    h, f, T = cfg.hidden, cfg.ffn, cfg.tokens
    per_layer = 2 * T * 2 / cfg.M * (3 * h * h + h * h + f * h + h * f)
    return per_layer * cfg.layers
