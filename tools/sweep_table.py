"""The SpMM sweep table of DESIGN.md §6 on the current build (tools only): for each workload the
planner's operand form, the median SpMM time and cuBLAS fp16 dense GEMM time on the decompressed
weight (interleaved, L2 flushed before every launch), useful TF/s, fraction of the measured dense
peak, algorithmic HBM fraction, speedup. Usage: python tools/sweep_table.py [ROUNDS]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

WORKLOADS = [
    "bert_large_ffn2_1024x4096x4096_64:2:8", "bert_large_ffn1_4096x1024x4096_64:2:8",
    "sweep_4096x4096x4096_128:2:4", "sweep_4096x4096x4096_128:2:8", "sweep_4096x4096x4096_128:2:16",
    "sweep_4096x4096x4096_128:2:32", "sweep_4096x4160x4096_128:2:40",
    "sweep_4096x4096x4096_64:2:16", "sweep_4096x4096x4096_64:2:32", "sweep_4096x4160x4096_64:2:40",
    "sweep_4096x4096x4096_256:2:16", "sweep_4096x4096x4096_32:2:16",
    "fig6_1024x4160x4096_128:2:10", "fig6_1024x4160x4096_128:2:20", "fig6_1024x4160x4096_128:2:40",
    "fig6_1024x4800x4096_128:2:100",
    "enc_qkv_3072x1040x16384_64:2:10", "enc_ffn2_1024x4160x16384_64:2:10",
    "gpt3_ffn_12288x49152x8192_128:2:16",
]


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 15
    dev = torch.device("cuda", 0)
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    peak, _, hbm, _ = bench.load_peaks()
    print(f"| workload (R×K×T, V:N:M) | operand form | SpMM ms | useful TF/s | frac of {peak:.0f} | "
          f"HBM frac (alg. bytes) | cuBLAS ms | speedup |")
    print("|---|---|---|---|---|---|---|---|")
    for name in WORKLOADS:
        L = bench.Layer(name, dev, 0)
        dense = L.venom.decompress(L.x)
        n = 2 if name.startswith("gpt3") else 1
        sp, cb = [], []
        for r in range(rounds + 2):
            for fn, acc in ((lambda: L.spmm(), sp), (lambda: torch.matmul(dense, L.B), cb)):
                flush.zero_()
                a, b = bench.ev_pair()
                a.record()
                fn()
                b.record()
                acc.append((a, b))
        torch.cuda.synchronize(dev)
        t_s = statistics.median(a.elapsed_time(b) for a, b in sp[2:])
        t_c = statistics.median(a.elapsed_time(b) for a, b in cb[2:])
        tf = L.flops / t_s / 1e9
        hb = bench.algorithmic_bytes(L.w, L.T) / (t_s / 1e3) / 1e9 / hbm
        form = "V:2:4 (#18)" if L.expand else ("2:4" if L.w["M"] == 4 else "gathered")
        print(f"| {name} | {form} | {t_s:.4f} | {tf:.0f} | {tf / peak:.2f} | {hb:.2f} | {t_c:.4f} | "
              f"{t_c / t_s:.2f}× |", flush=True)
        del L, dense
        torch.cuda.empty_cache()
        _ = n


if __name__ == "__main__":
    main()
