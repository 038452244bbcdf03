"""Times the format kernels (compress, compress_2to4, order_metadata, decompress) on a BASELINE
shape, with a cold L2 (flushed before every launch) and a warm L2. Tools only."""
import os, sys, statistics
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_02065_b200.build import build as _build
if os.environ.get("ABLATE"):
    os.environ.setdefault("VENOM_LIB", _build(ablation=True))  # the build that honours VENOM_DEBUG_FLAGS
import paper_2310_02065_b200 as venom

R, K, V, M = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (1024, 4096, 64, 8)))
A = (torch.randn(R, K, device="cuda") * 0.02).half()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
x = venom.compress(A, V=V, M=M)
x2, y = venom.compress_2to4(A, V=V, M=M)
venom.order_metadata(x)
D = torch.empty_like(A)
ops = {
    "compress": lambda: venom.compress(A, V=V, M=M, out=x),
    "compress_2to4": lambda: venom.compress_2to4(A, V=V, M=M, out=(x2, y)),
    "order_metadata": lambda: venom.order_metadata(x),
    "decompress": lambda: venom.decompress(x, out=D),
    "torch copy (same bytes as A)": lambda: D.copy_(A),
}
for name, fn in ops.items():
    for cold in (True, False):
        ts = []
        for i in range(15):
            if cold:
                flush.zero_()
            torch.cuda._sleep(100000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        us = statistics.median(a.elapsed_time(b) for a, b in ts[3:]) * 1e3
        print(f"{name:30s} {'cold' if cold else 'warm'} L2: {us:8.2f} us  ({2 * R * K / us / 1e3:7.1f} GB/s of A)")
if os.environ.get("ABLATE"):
    for fl in (1, 2, 4, 8, 15, 16, 32, 48):
        os.environ["VENOM_DEBUG_FLAGS"] = str(fl)
        ts = []
        for i in range(15):
            torch.cuda._sleep(100000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            venom.compress_2to4(A, V=V, M=M, out=(x2, y))
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        print(f"compress_2to4 ablation flags {fl}: {statistics.median(a.elapsed_time(b) for a, b in ts[3:]) * 1e3:8.2f} us")
    os.environ["VENOM_DEBUG_FLAGS"] = "0"
