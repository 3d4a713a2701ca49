"""Host-side cost of the host-buffer entry point at m = 1 (Mixtral layer):
forward_host wall time vs device-buffer call + synchronize vs the ctypes floor."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import paper_2504_02658_b200 as mb
from paper_2504_02658_b200 import synth

spec = synth.CONFIGS["mixtral"]
routed_h, shared_h = synth.build_host_layer(spec, seed=0)
ex = [mb.Expert(*(mb.Weight(P) for P in h.w), *((mb.Comp(c) if c is not None else None) for c in h.c))
      for h in routed_h]
layer = mb.MoELayer(ex, [], top_k=spec.top_k, score_mode=spec.score_mode)
m = 1
xh = torch.randn(m, spec.d).pin_memory(); lh = torch.randn(m, spec.experts).pin_memory()
xn, ln = xh.numpy(), lh.numpy()
xd, ld = xh.cuda(), lh.cuda()
out = torch.empty(m, spec.d, device="cuda")

def wall(fn, n=200):
    for _ in range(10): fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e6, np.mean(ts) * 1e6

print("forward_host             med/mean us: %.1f %.1f" % wall(lambda: layer.forward_host(xn, ln)))
def dev():
    layer.forward(xd, ld); torch.cuda.synchronize()
print("device call + sync       med/mean us: %.1f %.1f" % wall(dev))
print("torch.cuda.synchronize   med/mean us: %.1f %.1f" % wall(torch.cuda.synchronize))
print("ctypes milo_last_error   med/mean us: %.1f %.1f" % wall(lambda: mb.lib().milo_last_error()))
def launch_only():
    layer.forward(xd, ld)
print("device call (no sync)    med/mean us: %.1f %.1f" % wall(launch_only, 50)); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(50):
    s.record(); layer.forward(xd, ld); e.record(); e.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
print("device events (warm L2)  med us: %.1f" % np.median(ts))
# raw C dispatch cost (no Python wrapper): device buffers, no sync
from paper_2504_02658_b200 import _dptr
L = mb.lib()
args = (layer._h, _dptr(xd), m, 0, _dptr(ld), _dptr(out), 0, None, None, None)
def raw():
    L.milo_moe_forward(*args)
torch.cuda.synchronize()
print("raw milo_moe_forward     med/mean us: %.1f %.1f" % wall(raw, 50)); torch.cuda.synchronize()
print("torch.empty (cuda)       med/mean us: %.1f %.1f" % wall(lambda: torch.empty((m, spec.d), device="cuda")))
print("current_stream           med/mean us: %.1f %.1f" % wall(lambda: torch.cuda.current_stream()))
from paper_2504_02658_b200 import _stream_ptr
print("_stream_ptr              med/mean us: %.1f %.1f" % wall(lambda: _stream_ptr()))
print("MoELayer.forward (no sync) med/mean us: %.1f %.1f" % wall(lambda: layer.forward(xd, ld), 50)); torch.cuda.synchronize()
