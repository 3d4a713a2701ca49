"""Kernel timeline of one MoE-layer call (torch.profiler / CUPTI timestamps).

    python tools/timeline.py [--config mixtral] [--batch 1]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_02658_b200 as mb
from paper_2504_02658_b200.synth import CONFIGS, build_host_layer

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mixtral")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
spec = CONFIGS[a.config]
routed, shared = build_host_layer(spec, 0)
ex = [mb.Expert(*(mb.Weight(P) for P in h.w), *((mb.Comp(c) if c is not None else None) for c in h.c)) for h in routed]
sh = [mb.Expert(*(mb.Weight(P) for P in h.w), *((mb.Comp(c) if c is not None else None) for c in h.c)) for h in shared]
layer = mb.MoELayer(ex, sh, top_k=spec.top_k, score_mode=spec.score_mode)
x = torch.randn(a.batch, spec.d, device="cuda").half()
lg = torch.randn(a.batch, spec.experts, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    layer.forward(x, lg)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.iters):
        flush.zero_()
        layer.forward(x, lg, out_dtype=torch.float16)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA" and "milo" in e.name]
evs.sort(key=lambda e: e.time_range.start)
# last iteration
groups, cur = [], []
for e in evs:
    if "moe_route" in e.name and cur:
        groups.append(cur); cur = []
    cur.append(e)
groups.append(cur)
g = groups[-1]
t0 = g[0].time_range.start
for e in g:
    name = e.name.split("(")[0].replace("void milo_dev::", "").replace("milo_dev::", "")
    print(f"{name:40s} start={e.time_range.start - t0:8.1f}us dur={e.time_range.end - e.time_range.start:7.1f}us end={e.time_range.end - t0:8.1f}")
print(f"layer span: {g[-1].time_range.end - t0:.1f} us")
