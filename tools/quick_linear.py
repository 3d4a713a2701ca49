"""Quick single-linear timing (C1: 4096x14336 g64 r32) — development aid."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_02658_b200 as mb
from oracle.oracle import Oracle
from tests.helpers import random_quantized, random_comp

o = Oracle("oracle")
k, n = 4096, 14336
P, _ = random_quantized(o, k, n, seed=7)
comp = random_comp(o, k, n, 32, seed=8)
W, Cp = mb.Weight(P), mb.Comp(comp)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
res = {}
for m in [1, 4, 8, 16, 32, 64]:
    A = torch.randn(m, k, device="cuda").half()
    out = torch.empty(m, n, device="cuda", dtype=torch.float16)
    for withc in [False, True]:
        for _ in range(5):
            mb.gemm_w3a16(A, W, Cp if withc else None, out=out, out_dtype=torch.float16)
        ts = []
        for _ in range(20):
            flush.zero_()
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record(); mb.gemm_w3a16(A, W, Cp if withc else None, out=out, out_dtype=torch.float16); e.record()
            torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
        t = float(np.median(ts))
        byts = o.matrix_memory_bytes(k, n, 32 if withc else 0) + 2 * m * (k + n)
        res[f"m{m}_comp{int(withc)}"] = dict(us=round(t, 2), GBps=round(byts / t / 1e3, 1))
        print(m, withc, res[f"m{m}_comp{int(withc)}"], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/quick_linear.json", "w"), indent=1)
