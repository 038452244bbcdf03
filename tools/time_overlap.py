"""Concurrency check (tools only): the GPT-3 FFN layer's SpMM and its decompression alone and
launched together on two streams (either order), default vs background decompression launch.
Usage: python tools/time_overlap.py [workload]"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else bench.DEFAULT_WORKLOAD
    dev = torch.device("cuda", 0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    L = bench.Layer(name, dev, 0)
    L.compress()
    side = torch.cuda.Stream(dev)
    main_s = torch.cuda.current_stream(dev)

    def run(order, bg):
        if order == "spmm":
            L.spmm()
        elif order == "dec":
            L.decompress(background=bg)
        else:
            first, second = (("spmm", "dec") if order == "spmm+dec" else ("dec", "spmm"))
            side.wait_stream(main_s)
            for k in (first, second):
                if k == "spmm":
                    L.spmm()
                else:
                    with torch.cuda.stream(side):
                        L.decompress(background=bg)
            main_s.wait_stream(side)

    for order in ("spmm", "dec", "spmm+dec", "dec+spmm"):
        for bg in ((False, True) if order != "spmm" else (False,)):
            ts = []
            for rep in range(8):
                flush.zero_()
                a, b = bench.ev_pair()
                a.record(main_s)
                run(order, bg)
                b.record(main_s)
                ts.append((a, b))
            torch.cuda.synchronize(dev)
            ms = statistics.median(a.elapsed_time(b) for a, b in ts[2:])
            print(f"{order:10s} background={bg}: {ms:.4f} ms", flush=True)


if __name__ == "__main__":
    main()
