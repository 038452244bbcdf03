import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, oracle, synth
import paper_2310_02065_b200 as venom
from tests.helpers import bits_to_f64, f64_to_bits
def dev(bits): return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.float16).cuda()
R, K, V, M = 128, 1024, 128, 4
A = synth.gaussian((R, K), 1.0, 0, 3)
vals, meta, cidx = oracle.compress(A, 0, V=V, M=M)
D = bits_to_f64(oracle.decompress(vals, meta, cidx, R, K, 0, V, M), 0)
x = venom.VNMTensor(dev(vals), torch.from_numpy(meta).cuda(), torch.from_numpy(cidx).cuda(), R, K, V, M)
I = dev(f64_to_bits(np.eye(K), 0))
for rep in range(2):
    C = venom.spmm(x, I, tile_t=256, strategy=2).double().cpu().numpy()
    bad = C != D
    print("rep", rep, "bad", bad.sum())
    r = np.nonzero(bad.any(1))[0][0]
    ks = np.nonzero(bad[r])[0]
    print(" row", r, "bad k:", ks[:40])
    for k in ks[:12]:
        cand = [(kk, rr) for rr in range(R) for kk in range(K) if D[rr, kk] == C[r, k] and C[r, k] != 0][:4]
        print("  k", k, "got", C[r, k], "ref", D[r, k], "got matches ref at (k,row):", cand)
