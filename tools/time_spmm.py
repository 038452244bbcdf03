"""Median SpMM launch time (L2 flushed before each launch) for one workload under several option
sets: python tools/time_spmm.py WORKLOAD 'group_n=1' 'group_n=3' ... (VENOM_LIB selects a build)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    name = sys.argv[1]
    dev = torch.device("cuda", 0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    L = bench.Layer(name, dev, 0)
    st = torch.cuda.current_stream(dev)
    for spec in sys.argv[2:] or [""]:
        kw = {k: int(v) for k, v in (x.split("=") for x in spec.split(",") if x)}
        if kw.get("transposed_out"):  # token-major C^T [T, R]
            kw["out"] = torch.empty((L.T, L.w["R"]), dtype=L.C.dtype, device=dev)
        for _ in range(3):
            L.spmm(**kw)
        ts = []
        for _ in range(int(os.environ.get("REPS", "10"))):
            flush.zero_()
            a, b = bench.ev_pair()
            a.record(st)
            L.spmm(**kw)
            b.record(st)
            ts.append((a, b))
        torch.cuda.synchronize(dev)
        ms = statistics.median(a.elapsed_time(b) for a, b in ts)
        print(f"{os.path.basename(os.environ.get('VENOM_LIB', 'libvenom.so'))} {name} {spec or 'default'}: "
              f"{ms:.4f} ms  {L.flops / ms / 1e9:.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
