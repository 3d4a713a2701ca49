"""Runs one MoE layer config repeatedly (for ncu): python tools/hd_run.py [config] [batch] [iters]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_02658_b200 as mb  # noqa: E402
from paper_2504_02658_b200.synth import CONFIGS, build_host_layer  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
spec = CONFIGS[name]
routed, shared = build_host_layer(spec, 0)
mk = lambda hs: [mb.Expert(*(mb.Weight(P) for P in h.w), *((mb.Comp(c) if c is not None else None) for c in h.c))
                 for h in hs]
layer = mb.MoELayer(mk(routed), mk(shared), top_k=spec.top_k, score_mode=spec.score_mode)
x = torch.randn(m, spec.d, device="cuda").half()
lg = torch.randn(m, spec.experts, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(iters):
    flush.zero_()
    layer.forward(x, lg)
torch.cuda.synchronize()
print("ok")
