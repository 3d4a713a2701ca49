import sys, os, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2504_02658_b200 as mb
from paper_2504_02658_b200.synth import packed_random_words
rng = np.random.default_rng(0)
k, n = int(sys.argv[1]), int(sys.argv[2]); ms = [int(x) for x in sys.argv[3:]]
P = packed_random_words(k, n, rng)
W = mb.Weight(P)
# reference: identity-free check -> compare against the decode path (m<=16 chunks) by splitting rows
for m in ms:
    A = torch.randn(m, k, device="cuda").half()
    outs = []
    for rep in range(3):
        o = mb.gemm_w3a16(A, W, None).float(); torch.cuda.synchronize(); outs.append(o)
    ref = torch.cat([mb.gemm_w3a16(A[i:i+16], W, None).float() for i in range(0, m, 16)])
    errs = [float((o - ref).norm() / ref.norm()) for o in outs]
    print(f"k={k} n={n} m={m}: rel err vs decode path per repeat {['%.2e' % e for e in errs]}", flush=True)
