import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_02658_b200 as mb
from oracle.oracle import Oracle
from tests.helpers import random_quantized, random_comp, rel_err
o = Oracle("oracle")
k = n = 128
rng = np.random.default_rng(3)
codes = rng.integers(0, 8, (k, n), dtype=np.uint8)
P = o.pack_matrix(codes, np.full(k * n // 64, 0.25, np.float32), np.full(k * n // 64, 4.0, np.float32))
W = mb.Weight(P)
for m in (128, 16, 8, 1):
    A = torch.eye(k, dtype=torch.float32, device="cuda")[:m]
    C = mb.gemm_w3a16(A, W).cpu().numpy()
    want = np.array([o.half_to_float(int(h)) for h in o.dequant_half(P).ravel()], np.float32).reshape(k, n)[:m]
    bad = np.argwhere(C != want)
    print("m", m, "bad", len(bad), bad[:10].tolist(), C[tuple(bad[0])] if len(bad) else None, want[tuple(bad[0])] if len(bad) else None)
for (k, n, m) in [(512, 1024, 1), (512, 1024, 16), (4096, 14336, 1)]:
    P, _ = random_quantized(o, k, n, seed=1)
    comp = random_comp(o, k, n, 32, seed=2)
    A = np.random.default_rng(3).normal(0, 1, (m, k)).astype(np.float32)
    got = mb.gemm_w3a16(torch.from_numpy(A).cuda(), mb.Weight(P), None).cpu().numpy()
    print(k, n, m, "nocomp err", rel_err(got, o.gemm_w3a16(A, P, None)))
    got = mb.gemm_w3a16(torch.from_numpy(A).cuda(), mb.Weight(P), mb.Comp(comp)).cpu().numpy()
    print(k, n, m, "comp err", rel_err(got, o.gemm_w3a16(A, P, comp)))
