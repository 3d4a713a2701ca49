"""Diagnostic: GPU layer vs CPU oracle vs an fp64 restatement (h rounded to binary16
from fp64 values) at a real config; per-token error spread.  python tools/diag_real.py arctic 64"""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_gpu_real_configs import RealLayer
from tests.helpers import rel_err
import paper_2504_02658_b200 as mb
from oracle.oracle import Oracle

name, m = sys.argv[1], int(sys.argv[2])
o = Oracle("oracle")
L = RealLayer(mb, name, distinct=8 if name == "arctic" else None)
spec = L.spec
rng = np.random.default_rng(3000 + m)
x = rng.normal(0, 1, (m, spec.d)).astype(np.float32)
logits = rng.normal(0, 1, (m, spec.experts)).astype(np.float32)
ids, w = o.router_topk(logits, spec.top_k, spec.score_mode)
want = o.moe_forward(L.o_ex, L.o_sh, x, ids, w, n_threads=os.cpu_count())
got = L.layer.forward(torch.from_numpy(x).cuda(), torch.from_numpy(logits).cuda()).cpu().numpy()
xh = x.astype(np.float16).astype(np.float64)
cache = {}
def deq(P):
    k = id(P)
    if k not in cache:
        cache[k] = o.dequant_half(P).view(np.float16).astype(np.float64).reshape(P.rows, P.cols)
    return cache[k]
def comp(c):
    if c is None: return None
    U = np.zeros((c.rows, c.rank)); V = np.zeros((c.cols, c.rank))
    gs = 64
    for g in range((c.rank + gs - 1) // gs):
        sl = slice(g * gs, min(c.rank, (g + 1) * gs))
        U[:, sl] = (c.qu_codes[:, sl].astype(np.float64) - 4) * (c.qu_scales[:, g:g+1].astype(np.float32) * np.float32(2.0 / 7.0)).astype(np.float64)
        V[:, sl] = (c.qvt_codes[:, sl].astype(np.float64) - 4) * (c.qvt_scales[:, g:g+1].astype(np.float32) * np.float32(2.0 / 7.0)).astype(np.float64)
    return U, V.T
def lin(a, P, c):
    y = a @ deq(P)
    cc = comp(c)
    if cc is not None:
        y = y + (a @ cc[0]) @ cc[1]
    return y
f64 = np.zeros((m, spec.d))
flips = []
for t in range(m):
    for k in range(spec.top_k):
        e = ids[t, k]
        if e < 0: continue
        ex = L.o_ex[e]
        a = xh[t:t+1]
        g1 = lin(a, ex["w"][0], ex["c"][0]); g3 = lin(a, ex["w"][1], ex["c"][1])
        h = (g1 / (1 + np.exp(-g1)) * g3).astype(np.float16).astype(np.float64)
        f64[t] += w[t, k] * lin(h, ex["w"][2], ex["c"][2])[0]
print(f"{name} m={m}: gpu-oracle {rel_err(got, want):.3g}  gpu-f64 {rel_err(got, f64):.3g}  oracle-f64 {rel_err(want, f64):.3g}")
pt = [rel_err(got[t], want[t]) for t in range(m)]
po = [rel_err(want[t], f64[t]) for t in range(m)]
pg = [rel_err(got[t], f64[t]) for t in range(m)]
print("per-token gpu-oracle: max %.3g med %.3g | gpu-f64 max %.3g med %.3g | oracle-f64 max %.3g med %.3g" % (max(pt), np.median(pt), max(pg), np.median(pg), max(po), np.median(po)))
