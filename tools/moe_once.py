"""Runs one MoE layer call (after warm-up) at a given batch -- an ncu target.

    python tools/moe_once.py [--config mixtral] [--batch 256] [--iters 1]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_02658_b200 as mb
from paper_2504_02658_b200.synth import CONFIGS, build_host_layer

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mixtral")
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--iters", type=int, default=1)
a = ap.parse_args()
spec = CONFIGS[a.config]
routed, shared = build_host_layer(spec, 0)
mk = lambda h: mb.Expert(*(mb.Weight(P) for P in h.w), *((mb.Comp(c) if c is not None else None) for c in h.c))
layer = mb.MoELayer([mk(h) for h in routed], [mk(h) for h in shared], top_k=spec.top_k, score_mode=spec.score_mode)
x = torch.randn(a.batch, spec.d, device="cuda").half()
lg = torch.randn(a.batch, spec.experts, device="cuda")
for _ in range(a.iters):
    layer.forward(x, lg)
torch.cuda.synchronize()
