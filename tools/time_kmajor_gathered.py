"""K-major (token-major) B on the gathered operand vs feature-major B (tools only): the cost of the
transpose pass venom_spmm_ex runs into the scratch. Usage: python tools/time_kmajor_gathered.py"""
import os, sys, statistics, torch
sys.path.insert(0, "/root/repo")
import bench
dev = torch.device("cuda", 0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for name in ["enc_ffn1_4096x1040x16384_64:2:10", "gpt3_ffn_12288x49152x8192_128:2:16"]:
    L = bench.Layer(name, dev, 0)
    Bt = L.B.t().contiguous()
    res = {}
    for r in range(12):
        for k, fn in (("feature-major B", lambda: L.spmm()), ("token-major B (b_kmajor)", lambda: L.spmm(B=Bt, b_kmajor=True))):
            flush.zero_()
            a, b = bench.ev_pair(); a.record(); fn(); b.record()
            res.setdefault(k, []).append((a, b))
    torch.cuda.synchronize()
    for k, v in res.items():
        print(name, k, f"{statistics.median(x.elapsed_time(y) for x, y in v[2:]):.4f} ms")
