"""Layer latency at m = 16 after other calls in the same process (sweep-order check)."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_02658_b200 as mb
from paper_2504_02658_b200.synth import CONFIGS, build_host_layer
spec = CONFIGS["mixtral"]
routed, shared = build_host_layer(spec, 0)
ex = [mb.Expert(*(mb.Weight(P) for P in h.w), *((mb.Comp(c) if c is not None else None) for c in h.c)) for h in routed]
layer = mb.MoELayer(ex, [], top_k=2)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); fr = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
def t(m, host=False):
    xs = [torch.randn(m, 4096, device="cuda").half() for _ in range(8)]
    ls = [torch.randn(m, 8, device="cuda") for _ in range(8)]
    for i in range(3): layer.forward(xs[i], ls[i], out_dtype=torch.float16)
    ts = []
    for i in range(3, 8):
        flush.zero_(); torch.sum(fr)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); layer.forward(xs[i], ls[i], out_dtype=torch.float16); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return np.median(ts)
print("m=16 first:", t(16))
print("m=1:", t(1))
if len(sys.argv) > 1:
    x = np.random.randn(1, 4096).astype(np.float32); l = np.random.randn(1, 8).astype(np.float32)
    for _ in range(5): layer.forward_host(x, l)
    print("(host path ran)")
print("m=16 after:", t(16))
print("m=64:", t(64), "m=16 again:", t(16))
