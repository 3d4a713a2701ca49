"""Per-step globaltimer stamps of moe_plan_kernel (one MoE prefill call).
    python tools/plan_stamps.py [--config arctic] [--batch 256]"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_02658_b200 as mb
from paper_2504_02658_b200.synth import CONFIGS, build_host_layer
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="arctic"); ap.add_argument("--batch", type=int, default=256)
a = ap.parse_args(); spec = CONFIGS[a.config]
routed, shared = build_host_layer(spec, 0)
mk = lambda h: mb.Expert(*(mb.Weight(P) for P in h.w), *((mb.Comp(c) if c is not None else None) for c in h.c))
layer = mb.MoELayer([mk(h) for h in routed], [mk(h) for h in shared], top_k=spec.top_k, score_mode=spec.score_mode)
x = torch.randn(a.batch, spec.d, device="cuda").half(); lg = torch.randn(a.batch, spec.experts, device="cuda")
for _ in range(3): layer.forward(x, lg)
dbg = torch.zeros(8192, dtype=torch.int64, device="cuda")
L = mb.lib(); L.milo_debug_timeline.argtypes = [ctypes.c_void_p]; L.milo_debug_timeline.restype = None
torch.cuda.synchronize(); L.milo_debug_timeline(ctypes.c_void_p(dbg.data_ptr())); layer.forward(x, lg); torch.cuda.synchronize(); L.milo_debug_timeline(None)
d = dbg[2 * 3232:2 * 3232 + 6].cpu().tolist()
print(a.config, a.batch, "plan steps (us):", [round((d[i + 1] - d[i]) / 1e3, 2) for i in range(5)], "total", round((d[5] - d[0]) / 1e3, 2))
