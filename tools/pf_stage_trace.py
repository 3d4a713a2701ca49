"""Per-stage event trace of the MoE prefill GEMMs (pf_gemm_kernel, CTA 0), one layer call.

    python tools/pf_stage_trace.py [--config mixtral] [--batch 256] [--flags 0]

Events per stage (globaltimer, us from the CTA's start): 0 packed issued, 1 A slot free
(group), 2 packed landed (group), 3 A ready (group), 4 MMA saw A, 5 MMA saw B,
6 MMA committed, 7 B issued.  Prints per-CTA role end times, the first stages and
median per-stage gaps between events.
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_02658_b200 as mb  # noqa: E402
from paper_2504_02658_b200.synth import CONFIGS, build_host_layer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mixtral")
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--flags", type=int, default=0)
a = ap.parse_args()
spec = CONFIGS[a.config]
routed, shared = build_host_layer(spec, 0)
mk = lambda h: mb.Expert(*(mb.Weight(P) for P in h.w), *((mb.Comp(c) if c is not None else None) for c in h.c))
layer = mb.MoELayer([mk(h) for h in routed], [mk(h) for h in shared], top_k=spec.top_k, score_mode=spec.score_mode)
x = torch.randn(a.batch, spec.d, device="cuda").half()
lg = torch.randn(a.batch, spec.experts, device="cuda")
for _ in range(3):
    layer.forward(x, lg)
TS, REG = 256, 148 * 8 + 256 * 8
dbg = torch.zeros(2 * REG, dtype=torch.int64, device="cuda")
L = mb.lib()
L.milo_debug_flags.argtypes = [ctypes.c_int]
L.milo_debug_timeline.argtypes = [ctypes.c_void_p]
L.milo_debug_timeline.restype = None
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush.zero_()
torch.cuda.synchronize()
L.milo_debug_flags(a.flags)
L.milo_debug_timeline(ctypes.c_void_p(dbg.data_ptr()))
layer.forward(x, lg)
torch.cuda.synchronize()
L.milo_debug_timeline(None)
L.milo_debug_flags(0)
names = ["packed issued", "A slot free", "packed landed", "A ready", "MMA saw A", "MMA saw B", "MMA committed",
         "B issued"]
for ph in range(2):
    dd = dbg[ph * REG:(ph + 1) * REG].cpu().numpy().astype(np.float64)
    d = dd[:148 * 8].reshape(-1, 8)
    tr = dd[148 * 8:].reshape(TS, 8)
    v = d[:, 0] > 0
    d = d[v]
    if not len(d):
        continue
    t0 = d[:, 0].min()
    print(f"==== phase {ph + 1}: {v.sum()} CTAs")
    for i, nm in enumerate(["start", "packed prod done", "B prod done", "dequant w0 done", "mma done", "end",
                            "epi acc_full seen"]):
        y = d[:, i][d[:, i] > 0] - t0
        if len(y):
            print(f"  {nm:18s} min={y.min() / 1e3:8.2f} med={np.median(y) / 1e3:8.2f} max={y.max() / 1e3:8.2f} us")
    c0 = d[0, 0]
    tr = np.where(tr > 0, tr - c0, np.nan) / 1e3
    print("  stage " + " ".join(f"{n[:9]:>9s}" for n in names))
    for st in list(range(0, 10)) + list(range(60, 76)) + list(range(130, 136)):
        if st < TS and not np.isnan(tr[st]).all():
            print(f"  {st:5d} " + " ".join(f"{x:9.2f}" for x in tr[st]))
    ok = ~np.isnan(tr).any(axis=1)
    t = tr[ok]
    if len(t) > 4:
        st_gap = np.diff(t[:, 6])
        print(f"  stages traced {ok.sum()}, MMA commit period med {np.median(st_gap):.3f} us")
        for a_, b_, lbl in [(1, 2, "slot free -> packed landed"), (2, 3, "packed landed -> A ready (dequant)"),
                            (3, 4, "A ready -> MMA saw A"), (4, 5, "MMA saw A -> saw B"),
                            (5, 6, "saw B -> committed"), (0, 2, "packed issued -> landed"),
                            (7, 5, "B issued -> MMA saw B"), (1, 3, "slot free -> A ready")]:
            g = t[:, b_] - t[:, a_]
            print(f"  {lbl:36s} med {np.median(g):7.3f}  p90 {np.percentile(g, 90):7.3f} us")
    if os.environ.get("MILO_B200_LIB_VARIANT"):  # PF_PROF build: per-role cycle split of CTA 0
        roles = [("MMA issuer 0", ["wait stage", "MMAs", "commits"]), ("ring waiter", ["wait A", "wait B", "publish"]),
                 ("B producer", ["wait slot", "copy"]), ("packed producer", ["wait slot", "copies"]),
                 ("dequant w0", ["wait A slot", "wait packed", "dequant+st", "tail/idle"]),
                 ("epilogue w0", ["wait acc", "drain", "item setup"])]
        for r, (nm, parts) in enumerate(roles):
            raw = dd[148 * 8 + (TS - 1 - r) * 8:148 * 8 + (TS - 1 - r) * 8 + 4]
            tot = raw.sum()
            if tot > 0:
                print(f"  {nm:16s} {tot / 1e6:6.3f} Mcyc: " + ", ".join(f"{p_} {v / tot * 100:.0f}%" for p_, v in zip(parts, raw)))
