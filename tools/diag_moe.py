"""Diagnostic: where does the MoE layer's error vs fp64 come from?  Mixtral dims,
E experts (default 2) top-2 so every token hits every expert; per m: layer vs f64,
oracle vs f64, and a 'composed' GPU result (GPU linears, h rounded on the host)."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.helpers import rel_err
from tests.test_gpu_real_configs import _oracle_packed, _oracle_comp
import paper_2504_02658_b200 as mb
from paper_2504_02658_b200.synth import CONFIGS, build_host_layer
import dataclasses
from oracle.oracle import Oracle

o = Oracle("oracle")
E = int(sys.argv[1]) if len(sys.argv) > 1 else 2
d = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
f = int(sys.argv[3]) if len(sys.argv) > 3 else 14336
spec = dataclasses.replace(CONFIGS["mixtral"], experts=E, d=d, f=f)
routed, _ = build_host_layer(spec, seed=0)
dev = [mb.Expert(*(mb.Weight(P) for P in h.w), *((mb.Comp(c) if c is not None else None) for c in h.c)) for h in routed]
layer = mb.MoELayer(dev, [], top_k=2, score_mode=0)
o_ex = [{"w": [_oracle_packed(P) for P in h.w], "c": [_oracle_comp(c) for c in h.c]} for h in routed]
cache = {}
def deq(P):
    if id(P) not in cache:
        cache[id(P)] = o.dequant_half(_oracle_packed(P)).view(np.float16).astype(np.float64).reshape(P.rows, P.cols)
    return cache[id(P)]
def compf(c):
    if c is None: return None
    U = (c.qu_codes.astype(np.float64) - 4) * (c.qu_scales[:, :1] * np.float32(2 / 7)).astype(np.float64)
    V = (c.qvt_codes.astype(np.float64) - 4) * (c.qvt_scales[:, :1] * np.float32(2 / 7)).astype(np.float64)
    return U, V.T
def lin(a, P, c):
    y = a @ deq(P)
    cc = compf(c)
    return y if cc is None else y + (a @ cc[0]) @ cc[1]
for m in [int(v) for v in (sys.argv[4].split(",") if len(sys.argv) > 4 else "1,8,9,16,17,32,64,65,128".split(","))]:
    rng = np.random.default_rng(m)
    x = rng.normal(0, 1, (m, d)).astype(np.float32)
    logits = rng.normal(0, 1, (m, E)).astype(np.float32)
    ids, w = o.router_topk(logits, 2, 0)
    want = o.moe_forward(o_ex, [], x, ids, w, n_threads=os.cpu_count())
    got = layer.forward(torch.from_numpy(x).cuda(), torch.from_numpy(logits).cuda()).cpu().numpy()
    xh = x.astype(np.float16).astype(np.float64)
    f64 = np.zeros((m, d)); comp = np.zeros((m, d)); hflip = []
    xt = torch.from_numpy(x).cuda()
    for e in range(E):
        h = routed[e]
        g1 = lin(xh, h.w[0], h.c[0]); g3 = lin(xh, h.w[1], h.c[1])
        hh = (g1 / (1 + np.exp(-g1)) * g3).astype(np.float16)
        G1 = mb.gemm_w3a16(xt, dev[e].w1, dev[e].c1).cpu().numpy().astype(np.float64)
        G3 = mb.gemm_w3a16(xt, dev[e].w3, dev[e].c3).cpu().numpy().astype(np.float64)
        hg = (G1 / (1 + np.exp(-G1)) * G3).astype(np.float16)
        hflip.append(float((hg != hh).mean()))
        y = lin(hh.astype(np.float64), h.w[2], h.c[2])
        yg = mb.gemm_w3a16(torch.from_numpy(hg).cuda(), dev[e].w2, dev[e].c2).cpu().numpy()
        for t in range(m):
            for k in range(2):
                if ids[t, k] == e:
                    f64[t] += w[t, k] * y[t]; comp[t] += w[t, k] * yg[t]
    print(f"m={m:4d}: layer-f64 {rel_err(got, f64):.3g}  oracle-f64 {rel_err(want, f64):.3g}  composed-f64 {rel_err(comp, f64):.3g}  layer-composed {rel_err(got, comp):.3g}  h flips gpu-linear vs f64 {np.mean(hflip):.4f}", flush=True)
