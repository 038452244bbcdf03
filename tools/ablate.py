"""Ablation timing of venom_spmm (tools only): VENOM_DEBUG_FLAGS disables parts of the kernel
(1 B loads, 2 MMAs, 4 C stores, 8 metadata TMEM stores, 16 A loads) to find the binding resource.
Usage: python tools/ablate.py R K T V M strategy pair flags..."""
import os, sys, statistics
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_02065_b200.build import build as _build
os.environ.setdefault("VENOM_LIB", _build(ablation=True))  # the build that honours VENOM_DEBUG_FLAGS
import paper_2310_02065_b200 as venom

R, K, T, V, M, strat, pair = (int(x) for x in sys.argv[1:8])
flags = [int(x) for x in sys.argv[8:]] or [0]
prepared = os.environ.get("PREPARED", "1") == "1"
tile = int(os.environ.get("TILE", "0"))
torch.manual_seed(0)
A = (torch.randn(R, K, device="cuda") * 0.02).half()
B = torch.randn(K, T, device="cuda").half()
x = venom.compress(A, V=V, M=M, check=True)
if prepared:
    venom.order_metadata(x)
C = torch.empty(R, T, device="cuda", dtype=torch.half)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for fl in flags:
    os.environ["VENOM_DEBUG_FLAGS"] = str(fl)
    ts = []
    for i in range(12):
        flush.zero_()
        torch.cuda._sleep(200000)  # ~100 us: the host enqueues the launch before the GPU gets there
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        venom.spmm(x, B, out=C, strategy=strat, cta_pair=pair, tile_t=tile)
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in ts[2:])
    print(f"R{R} K{K} T{T} V{V} M{M} strat{strat} pair{pair} tile{tile} flags {fl:3d}: {ms*1e3:8.1f} us "
          f"{4*R*K*T/M/ms/1e9:7.1f} TF/s")
os.environ["VENOM_DEBUG_FLAGS"] = "0"
# host-side cost of one call (enqueue only)
import time
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    venom.spmm(x, B, out=C, strategy=strat, cta_pair=pair)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host enqueue per venom.spmm call: {(t1 - t0) / 50 * 1e6:.1f} us")
