"""sparse BERT-large encoder forward (all linear layers V:N:M 64:2:10, batch
32 × seq 512, BASELINE.json configs[4]) vs the same encoder with dense cuBLAS GEMMs on the pruned
weights. Prints one JSON line. Usage: python tools/bench_encoder.py [--layers 24] [--steps 5]."""
import argparse, json, os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_02065_b200 import encoder as enc


def time_it(fn, steps, warmup=2):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--seq", type=int, default=512)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--gelu", choices=["tanh", "erf"], default="tanh")
    args = ap.parse_args()
    cfg = enc.EncoderConfig(layers=args.layers, batch=args.batch, seq=args.seq, gelu=args.gelu)
    dev = torch.device("cuda")
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    W = enc.init_weights(cfg, dev)
    model = enc.SparseEncoder(cfg, W)
    dense = model.dense_weights()
    del W
    x = (torch.randn(cfg.tokens, cfg.hidden, generator=torch.Generator().manual_seed(1)) * 1.0).half().to(dev)
    ys = model.forward(x)
    yd = enc.dense_forward(cfg, dense, x)
    rel = float((ys.float() - yd.float()).norm() / yd.float().norm())
    t_s = time_it(lambda: model.forward(x), args.steps)
    t_d = time_it(lambda: enc.dense_forward(cfg, dense, x), args.steps)
    fl = enc.useful_flops(cfg)
    print(json.dumps({"workload": "bert_large_encoder_forward_64:2:10", "layers": cfg.layers,
                      "batch": cfg.batch, "seq": cfg.seq, "sparse_ms": round(t_s, 3), "dense_ms": round(t_d, 3),
                      "speedup_e2e": round(t_d / t_s, 3), "rel_fro_vs_dense_on_pruned_weights": rel,
                      "sparse_linear_useful_tflops_per_s": round(fl / (t_s / 1e3) / 1e12, 2),
                      "gelu": cfg.gelu + " form (sparse epilogue and dense F.gelu alike)",
                      "dtype": "f16", "data": "random-init weights, N(0,1) activations (no checkpoints)"}))


if __name__ == "__main__":
    main()
