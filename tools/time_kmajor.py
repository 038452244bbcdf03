"""Times the K-major-B / token-major-C SpMM options against the default layouts and dense F.linear (tools only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, statistics
import paper_2310_02065_b200 as venom
def t(fn, n=20):
    fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(n):
        fl.zero_(); torch.cuda._sleep(100000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); ts.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ts[3:]) * 1e3
for (R, K, T) in [(1024, 4096, 4096), (4096, 1024, 4096)]:
    W = (torch.randn(R, K, device="cuda") * 0.02).half()
    x, y = venom.compress_2to4(W, V=64, M=8, check=True)
    B = torch.randn(K, T, device="cuda").half(); X = B.t().contiguous()
    C = torch.empty(R, T, device="cuda").half(); Ct = torch.empty(T, R, device="cuda").half()
    print(R, K, T, "row-major B, row-major C %.1f us" % t(lambda: venom.spmm(y, B, out=C)),
          "| K-major B %.1f us" % t(lambda: venom.spmm(y, X, out=C, b_kmajor=True)),
          "| K-major B, token-major C %.1f us" % t(lambda: venom.spmm(y, X, out=Ct, b_kmajor=True, transposed_out=True)),
          "| torch F.linear dense %.1f us" % t(lambda: torch.nn.functional.linear(X, W)))
