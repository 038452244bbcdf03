"""Interleaved A/B timing of SpMM option sets (tools only): every round times each option set once
(L2 flushed before each launch), so clock / power drift affects all sets alike. Prints the median
and the SM clock NVML reports at the end.
Usage: python tools/time_spmm_ab.py WORKLOAD ROUNDS 'opts1' 'opts2' ..."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402


def main():
    name, rounds, specs = sys.argv[1], int(sys.argv[2]), sys.argv[3:] or [""]
    dev = torch.device("cuda", 0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    L = bench.Layer(name, dev, 0, form=os.environ.get("FORM", "auto"))  # FORM=vnm: the gathered form
    st = torch.cuda.current_stream(dev)
    kws = [{k: int(v) for k, v in (x.split("=") for x in s.split(",") if x)} for s in specs]
    for kw in kws:
        L.spmm(**kw)
    ev = {i: [] for i in range(len(kws))}
    for r in range(rounds):
        for i, kw in enumerate(kws):
            flush.zero_()
            a, b = bench.ev_pair()
            a.record(st)
            L.spmm(**kw)
            b.record(st)
            ev[i].append((a, b))
    torch.cuda.synchronize(dev)
    for i, s in enumerate(specs):
        t = [a.elapsed_time(b) for a, b in ev[i]]
        print(f"{name} {s or 'default'}: median {statistics.median(t):.4f} ms  min {min(t):.4f}  "
              f"{L.flops / statistics.median(t) / 1e9:.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
