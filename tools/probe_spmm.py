"""Diagnostics for layout bugs: runs tiny SpMMs with structured inputs and prints where the GPU
result departs from the oracle (rows / columns / k-blocks). Not a test; output goes to stdout."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle, synth
import paper_2310_02065_b200 as venom
from tests.helpers import bits_to_f64, f64_to_bits

def dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.float16).cuda()

def run(R, K, T, V, M, Akind, Bkind, tile_t=0, strategy=0, pair=0):
    if Akind == "ones":
        A = f64_to_bits(np.ones((R, K)), 0)
    elif Akind == "rowid":
        A = f64_to_bits(np.repeat((np.arange(R) % 64 + 1.0)[:, None], K, 1), 0)
    else:
        A = synth.gaussian((R, K), 1.0, 0, 3)
    if Bkind == "eye":
        assert T == K
        B = f64_to_bits(np.eye(K), 0)
    elif Bkind == "rowid":
        B = f64_to_bits(np.repeat((np.arange(K) % 16 + 1.0)[:, None], T, 1) / 16, 0)
    else:
        B = synth.gaussian((K, T), 1.0, 0, 4)
    vals, meta, cidx = oracle.compress(A, 0, V=V, M=M)
    ref = oracle.spmm(vals, meta, cidx, R, K, 0, V, M, B)
    x = venom.VNMTensor(dev(vals), torch.from_numpy(meta).cuda(), torch.from_numpy(cidx).cuda(), R, K, V, M)
    C = venom.spmm(x, dev(B), tile_t=tile_t, strategy=strategy, cta_pair=pair)
    torch.cuda.synchronize()
    got = C.double().cpu().numpy()
    bad = ~np.isclose(got, ref, rtol=2e-2, atol=1e-2)
    print(f"== R{R} K{K} T{T} V{V} M{M} A={Akind} B={Bkind} tile={tile_t} strat={strategy} pair={pair}: bad {bad.sum()}/{bad.size}")
    if bad.any():
        rows = np.nonzero(bad.any(1))[0]
        cols = np.nonzero(bad.any(0))[0]
        print("  bad rows:", rows[:40], "... n", len(rows))
        print("  bad cols:", cols[:40], "... n", len(cols))
        r = rows[0]
        print("  row", r, "got", got[r, :8], "ref", ref[r, :8])
        if Bkind == "eye":
            print("  bad k (cols) histogram by 128-stage:", np.bincount(cols // 128, minlength=K // 128))
            print("  bad rows count by 8-row group:", np.bincount(rows // 8, minlength=R // 8))
        for rr in list(rows[:4]):
            print("  row", rr, "got[:4]", np.round(got[rr, :4], 3), "ref[:4]", np.round(ref[rr, :4], 3))

if __name__ == "__main__":
    torch.cuda.init()
    import sys as _s
    if len(_s.argv) > 1 and _s.argv[1] == "pair":
        for c in [(256, 256, 256, 128, 8, "gauss", "eye", 256, 2, 2), (256, 1024, 512, 128, 8, "gauss", "gauss", 256, 2, 2),
                  (128, 1024, 512, 128, 8, "gauss", "gauss", 256, 2, 2), (384, 1024, 512, 64, 4, "gauss", "gauss", 256, 2, 2),
                  (512, 2048, 512, 64, 16, "gauss", "gauss", 128, 2, 2), (512, 1024, 1024, 128, 8, "gauss", "eye", 256, 2, 2)]:
            try:
                run(*c)
            except Exception as e:
                print("EXC", c, repr(e))
        _s.exit(0)
    if len(_s.argv) > 1 and _s.argv[1] == "densek":
        for c in [(128, 1024, 512, 128, 4, "gauss", "gauss", 256, 2), (128, 1024, 512, 128, 4, "gauss", "gauss", 128, 2),
                  (128, 1024, 512, 128, 8, "gauss", "gauss", 256, 2), (128, 1024, 1024, 128, 4, "gauss", "eye", 256, 2), (128, 1024, 1024, 128, 16, "gauss", "eye", 256, 2),
                  (128, 1024, 1024, 128, 32, "gauss", "eye", 256, 2), (128, 1024, 1024, 128, 8, "gauss", "eye", 256, 2),
                  (128, 256, 256, 128, 4, "gauss", "eye", 256, 2), (128, 256, 256, 128, 8, "gauss", "eye", 256, 2),
                  (512, 1024, 512, 128, 4, "gauss", "gauss", 256, 2)]:
            try:
                run(*c)
            except Exception as e:
                print("EXC", c, repr(e))
        _s.exit(0)
    cases = [
        (128, 128, 128, 128, 4, "ones", "eye"),
        (128, 128, 128, 128, 4, "gauss", "eye"),
        (128, 128, 64, 128, 4, "rowid", "rowid"),
        (128, 256, 64, 128, 8, "gauss", "gauss"),
        (128, 256, 256, 128, 8, "gauss", "eye"),
        (128, 128, 128, 64, 8, "gauss", "gauss"),
    ]
    for c in cases:
        try:
            run(*c)
        except Exception as e:
            print("EXC", c, repr(e))
