import sys, os, time, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_02658_b200 as mb
from oracle.oracle import Oracle
from tests.helpers import random_quantized, random_comp, rel_err
o = Oracle("oracle")
for (k, n, m, mode) in [(128, 128, 64, 1), (512, 1024, 64, 1), (512, 1024, 200, 0), (640, 256, 130, 1), (4096, 14336, 256, 1)]:
    P, _ = random_quantized(o, k, n, seed=1, mode=mode)
    A = np.random.default_rng(3).normal(0, 1, (m, k)).astype(np.float32)
    t0 = time.time()
    got = mb.gemm_w3a16(torch.from_numpy(A).cuda(), mb.Weight(P), None).cpu().numpy()
    want = o.gemm_w3a16(A, P, None)
    print(k, n, m, "err", rel_err(got, want), "time", round(time.time() - t0, 2), flush=True)
for (k, n, m, r, storage) in [(512, 1024, 64, 32, 1), (512, 1024, 200, 70, 1), (640, 256, 130, 4, 0), (4096, 14336, 256, 32, 1), (512, 512, 128, 16, 0)]:
    P, _ = random_quantized(o, k, n, seed=2)
    comp = random_comp(o, k, n, r, seed=5, storage=storage) if 'storage' in random_comp.__code__.co_varnames else random_comp(o, k, n, r, seed=5)
    A = np.random.default_rng(4).normal(0, 1, (m, k)).astype(np.float32)
    got = mb.gemm_w3a16(torch.from_numpy(A).cuda(), mb.Weight(P), mb.Comp(comp)).cpu().numpy()
    print(k, n, m, "rank", r, "storage", storage, "err", rel_err(got, o.gemm_w3a16(A, P, comp)), flush=True)
