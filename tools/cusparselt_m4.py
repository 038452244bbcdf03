"""cuSPARSELt at M = 4 beside venom_spmm (the paper's Fig 10 comparison; SURVEY
§8(c) "M = 4 -> library routine"): the same 2:4-pruned weight (venom_compress at V:2:4, i.e. plain
2:4 magnitude pruning, decompressed) multiplied by cuSPARSELt through torch._cslt_compress /
torch._cslt_sparse_mm, by venom_spmm, and by dense cuBLAS. Prints the relative errors against an
fp64 product and the median times (L2 flushed). Tools only: a library pin and a baseline, not on
the product path."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2310_02065_b200 as venom  # noqa: E402


def timeit(fn, flush, reps=20):
    st = torch.cuda.current_stream()
    ts = []
    for k in range(reps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        if k >= 3:
            ts.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ts)


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(3)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    for (R, K, T) in [(1024, 4096, 4096), (4096, 1024, 4096), (4096, 4096, 4096), (12288, 12288, 8192)]:
        A = (torch.randn(R, K, generator=g, device=dev) * 0.02).half()
        B = torch.randn(K, T, generator=g, device=dev).half()
        x = venom.order_metadata(venom.compress(A, V=128, M=4, check=True))  # plain 2:4 magnitude pruning
        Ap = venom.decompress(x)                                              # the pruned dense weight
        ref = Ap.double() @ B.double()
        Ac = torch._cslt_compress(Ap)
        C_lt = torch._cslt_sparse_mm(Ac, B)
        C_v = venom.spmm(x, B)
        C_d = Ap @ B
        rel = lambda C: float((C.double() - ref).norm() / ref.norm())  # noqa: E731
        t_lt = timeit(lambda: torch._cslt_sparse_mm(Ac, B), flush)
        t_v = timeit(lambda: venom.spmm(x, B, out=C_v), flush)
        t_d = timeit(lambda: torch.matmul(Ap, B, out=C_d), flush)
        flops = 2.0 * R * K * T / 2  # useful (2:4)
        print(f"{R}x{K}x{T} 2:4: rel err cuSPARSELt {rel(C_lt):.2e}  venom {rel(C_v):.2e}  cuBLAS dense {rel(C_d):.2e} | "
              f"ms cuSPARSELt {t_lt:.4f} ({flops / t_lt / 1e9:.0f} TF/s)  venom {t_v:.4f} ({flops / t_v / 1e9:.0f} TF/s)  "
              f"cuBLAS dense {t_d:.4f} | venom vs cuSPARSELt {t_lt / t_v:.2f}x", flush=True)


if __name__ == "__main__":
    main()
