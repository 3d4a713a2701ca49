"""Timeline of one hdec_kernel launch (hdec.cuh, milo_debug_timeline): per-CTA stage-0 /
end stamps, consumer warp 0's event sequence, ring wait cycles.
python tools/hd_timeline.py [config] [batch]   (config: mixtral | deepseek | arctic)"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_02658_b200 as mb  # noqa: E402
from paper_2504_02658_b200.synth import CONFIGS, build_host_layer  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = CONFIGS[name]
routed, shared = build_host_layer(spec, 0)
mk = lambda hs: [mb.Expert(*(mb.Weight(P) for P in h.w), *((mb.Comp(c) if c is not None else None) for c in h.c))
                 for h in hs]
layer = mb.MoELayer(mk(routed), mk(shared), top_k=spec.top_k, score_mode=spec.score_mode)
x = torch.randn(m, spec.d, device="cuda").half()
lg = torch.randn(m, spec.experts, device="cuda")
run = lambda: layer.forward(x, lg)
for _ in range(3):
    run()
G = 1024  # kHdDbgG (hdec.cuh): the timeline regions are sized for 1024 CTAs
dbg = torch.zeros(G * 320, dtype=torch.int64, device="cuda")
L0 = mb.lib()
L0.milo_debug_flags.argtypes = [ctypes.c_int]
L0.milo_debug_flags(int(os.environ.get("HD_FLAGS", "0")))
L = mb.lib()
L.milo_debug_timeline.argtypes = [ctypes.c_void_p]
L.milo_debug_timeline.restype = None
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
if os.environ.get("NOFLUSH") != "1":
    flush.zero_()
    flush.sum()
torch.cuda.synchronize()
L.milo_debug_timeline(ctypes.c_void_p(dbg.data_ptr()))
run()
torch.cuda.synchronize()
L.milo_debug_timeline(None)
dd = dbg.cpu().numpy()
d = dd[:G * 128].reshape(G, 128)
pr = dd[G * 128:G * 192].reshape(G, 64)
cw = dd[G * 192:G * 320].reshape(G, 64, 2)
G = int((d[:, 0] > 0).sum())  # CTAs of the launch
d, pr, cw = d[:G], pr[:G], cw[:G]
t0 = d[:, 0].min()
NAMES = {1: "T", 2: "P1", 3: "HEADPUB", 4: "FINBEGIN", 5: "FV", 6: "FINH", 7: "FU", 8: "T2DONE", 9: "HWAIT",
         10: "P2", 11: "V2"}


def st(v):
    v = np.asarray(v, dtype=np.float64) / 1e3
    return f"min {v.min():7.2f} med {np.median(v):7.2f} p90 {np.percentile(v, 90):7.2f} max {v.max():7.2f} us"


print(f"{name} m={m}: G={G}")
print("stage0 done   ", st(d[:, 1] - t0))
print("producer done ", st(d[:, 3] - t0))
print("consumer done ", st(d[:, 2] - t0))
print("producer empty-wait (us at 1.965 GHz)", st(d[:, 126] / 1.965))
print("consumer full-wait  (us at 1.965 GHz)", st(d[:, 127] / 1.965))
dur = {}
cnt = {}
for c in range(G):
    nev = int(d[c, 125])
    prev = d[c, 1]
    for i in range(min(nev, 60)):
        code, t = int(d[c, 4 + 2 * i]), d[c, 5 + 2 * i]
        ty = code & 0xFF
        dur.setdefault(NAMES.get(ty, ty), []).append(t - prev)
        prev = t
for k, v in dur.items():
    v = np.array(v) / 1e3
    print(f"  {k:9s} n={len(v):5d} mean {v.mean():6.2f} med {np.median(v):6.2f} max {v.max():6.2f} total/CTA {v.sum() / G:6.2f} us")
for c in [0, 1, G // 2, G - 1, int(np.argmax(d[:, 2]))]:
    nev = int(d[c, 125])
    seq = []
    for i in range(min(nev, 60)):
        code, t = int(d[c, 4 + 2 * i]), d[c, 5 + 2 * i]
        seq.append(f"{NAMES.get(code & 0xFF, code & 0xFF)}{(code >> 8) & 0xFF}@{(t - t0) / 1e3:.1f}")
    print(f"cta {c}: s0 {(d[c, 1] - t0) / 1e3:.1f} end {(d[c, 2] - t0) / 1e3:.1f}: " + " ".join(seq))

for c in [0, G // 2]:
    print(f"cta {c}: stage: issued -> consumer waits from .. to (us); copy latency seen = end - issue when the consumer waited")
    lat = []
    for k in range(64):
        if pr[c, k] <= 0 or cw[c, k, 1] <= 0:
            continue
        iss, w0, w1 = (pr[c, k] - t0) / 1e3, (cw[c, k, 0] - t0) / 1e3, (cw[c, k, 1] - t0) / 1e3
        waited = w1 - w0 > 0.05
        if waited:
            lat.append(w1 - iss)
        print(f"   {k:2d}: issued {iss:6.1f}  wait {w0:6.1f} -> {w1:6.1f} ({w1 - w0:4.2f})" + (f"  latency {w1 - iss:4.2f}" if waited else ""))
    if lat:
        print("   median latency when waited:", np.median(lat))

# per event kind: data wait vs processing (consumer warp 0 of every CTA; stage index = event index
# only while every event has a stage, i.e. the first 60 events)
print("per event kind (all CTAs): mean data-wait / mean processing after the wait (us)")
agg = {}
for c in range(G):
    nev = int(d[c, 125])
    for i in range(min(nev, 60)):
        code, tend = int(d[c, 4 + 2 * i]), d[c, 5 + 2 * i]
        w0, w1 = cw[c, i, 0], cw[c, i, 1]
        if w1 <= 0 or i >= 64:
            continue
        kname = NAMES.get(code & 0xFF, code & 0xFF)
        fl = (code >> 16) & 0xFF
        if kname == "P1" and fl & 4:
            kname = "P1+FINBEGIN"
        elif kname == "P1" and fl & 2:
            kname = "P1+HEADPUB"
        a_ = agg.setdefault(kname, [[], []])
        a_[0].append((w1 - w0) / 1e3)
        a_[1].append((tend - w1) / 1e3)
for k_, (wv, pv) in agg.items():
    print(f"  {k_:12s} n={len(wv):5d} wait {np.mean(wv):5.2f}  proc {np.mean(pv):5.2f} (med {np.median(pv):5.2f})")
