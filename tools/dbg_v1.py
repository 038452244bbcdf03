import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth, oracle
import paper_2310_02065_b200 as venom
for (R, K, V, M) in [(70000, 32, 1, 8), (1000, 32, 1, 8), (4096, 64, 1, 8), (256, 1024, 128, 16)]:
    A = synth.gaussian((R, K), 0.02, synth.F16, 77)
    exp = oracle.compress(A, synth.F16, V=V, M=M)
    x = venom.compress(torch.from_numpy(A.view(np.int16)).view(torch.float16).cuda(), V=V, M=M, check=True)
    got = x.values.view(torch.int16).cpu().numpy().view(np.uint16).reshape(exp[0].shape)
    bad = np.nonzero((got != exp[0]).any(axis=(1, 2)))[0]
    print(R, K, V, M, "bad rows", len(bad), bad[:5], bad[-5:] if len(bad) else "")
