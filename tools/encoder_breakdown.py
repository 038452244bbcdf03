"""Per-op device time of one sparse encoder layer (tools only): CUDA events around each step of
SparseEncoder._layer, median of 10 repetitions. Usage: python tools/encoder_breakdown.py"""
import os, statistics, sys
import torch
import torch.nn.functional as F
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_02065_b200 as venom
from paper_2310_02065_b200 import encoder as enc

cfg = enc.EncoderConfig(layers=1)
dev = torch.device("cuda")
W = enc.init_weights(cfg, dev)
m = enc.SparseEncoder(cfg, W)
L = m.layers[0]
h, T = cfg.hidden, cfg.tokens
x = torch.randn(T, h, device=dev).half()
Bt, S, H = cfg.batch, cfg.seq, cfg.heads
D = h // H
st = {}


def step(name, fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    r = fn()
    b.record()
    st.setdefault(name, []).append((a, b))
    return r


x1 = torch.empty_like(x)
o2 = torch.empty_like(x)
for rep in range(12):
    step("qkv spmm (token-major out)", lambda: L["qkv"](m.x_fm, out=m.qkv_tm, token_major=True))
    q, k, v = (m.qkv_tm[:, i * h:(i + 1) * h].view(Bt, S, H, D).transpose(1, 2) for i in range(3))
    a = step("sdpa", lambda: F.scaled_dot_product_attention(q, k, v))
    step("heads -> attn_fm", lambda: venom.enc_heads_to_fm(a, m.attn_fm))
    step("o spmm (token-major out)", lambda: L["o"](m.attn_fm, out=m.o_tm, token_major=True))
    step("add + layer_norm (+ fm copy)", lambda: venom.enc_add_layernorm(x, m.o_tm, L["ln1_w"], L["ln1_b"], cfg.eps, x1, m.x1_fm))
    step("f1 spmm (+ GELU epilogue)", lambda: L["f1"](m.x1_fm, out=m.hid[:cfg.ffn], gelu=cfg.gelu))
    step("f2 spmm (token-major out)", lambda: L["f2"](m.hid, out=m.f2_tm, token_major=True))
    step("add + layer_norm 2 (+ fm copy)", lambda: venom.enc_add_layernorm(x1, m.f2_tm, L["ln2_w"], L["ln2_b"], cfg.eps, o2, m.x_fm))
torch.cuda.synchronize()
tot = 0.0
for k2, v2 in st.items():
    ms = statistics.median(a.elapsed_time(b) for a, b in v2[2:])
    tot += ms
    print(f"{k2:32s} {ms * 1e3:9.1f} us")
print(f"{'total':32s} {tot * 1e3:9.1f} us")
