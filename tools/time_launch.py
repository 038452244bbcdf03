"""Fixed per-launch cost of the SpMM (tools only): one launch after the L2 flush vs two and four
back-to-back launches, and one launch preceded by another SpMM (same shared-memory configuration)
instead of the flush kernel. Usage: python tools/time_launch.py WORKLOAD [ROUNDS]"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402


def main():
    name = sys.argv[1]
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    dev = torch.device("cuda", 0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    L = bench.Layer(name, dev, 0)
    st = torch.cuda.current_stream(dev)
    for _ in range(3):
        L.spmm()
    res = {}
    for r in range(rounds):
        for n in (1, 2, 4):
            flush.zero_()
            torch.cuda._sleep(200000)  # the host enqueues everything before the GPU gets there
            a, b = bench.ev_pair()
            a.record(st)
            for _ in range(n):
                L.spmm()
            b.record(st)
            res.setdefault(f"{n} launch(es) after the flush", []).append((a, b))
        # one launch right after another SpMM (no flush kernel in between)
        flush.zero_()
        L.spmm()
        torch.cuda._sleep(200000)
        a, b = bench.ev_pair()
        a.record(st)
        L.spmm()
        b.record(st)
        res.setdefault("1 launch after an SpMM (L2 warm)", []).append((a, b))
    torch.cuda.synchronize(dev)
    for k, v in res.items():
        print(f"{name} {k:36s}: {statistics.median(x.elapsed_time(y) for x, y in v) * 1e3:8.1f} us")


if __name__ == "__main__":
    main()
