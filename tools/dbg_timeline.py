"""Per-warp timeline of one decode launch (milo_debug_timeline)."""
import sys, os, ctypes, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_02658_b200 as mb
from paper_2504_02658_b200.synth import CONFIGS, build_host_layer
m = int(sys.argv[1]) if len(sys.argv) > 1 else 1
mode = sys.argv[2] if len(sys.argv) > 2 else "moe"
if mode == "moe" or mode in CONFIGS:
    spec = CONFIGS["mixtral" if mode == "moe" else mode]
    routed, shared = build_host_layer(spec, 0)
    mk = lambda hs: [mb.Expert(*(mb.Weight(P) for P in h.w), *((mb.Comp(c) if c is not None else None) for c in h.c)) for h in hs]
    layer = mb.MoELayer(mk(routed), mk(shared), top_k=spec.top_k, score_mode=spec.score_mode)
    x = torch.randn(m, spec.d, device="cuda").half(); lg = torch.randn(m, spec.experts, device="cuda")
    run = lambda: layer.forward(x, lg)
else:
    from paper_2504_02658_b200.synth import packed_random_words
    from paper_2504_02658_b200.pack import random_compensator
    rng = np.random.default_rng(0)
    W = mb.Weight(packed_random_words(4096, 14336, rng)); Cm = mb.Comp(random_compensator(4096, 14336, 32, rng))
    x = torch.randn(m, 4096, device="cuda").half()
    run = lambda: mb.gemm_w3a16(x, W, Cm)
for _ in range(3): run()
dbg = torch.zeros(148 * 16 * 16, dtype=torch.int64, device="cuda")
L = mb.lib(); L.milo_debug_flags.argtypes = [ctypes.c_int]; L.milo_debug_flags(int(os.environ.get("DEC_FLAGS", "0")))
L.milo_debug_timeline.argtypes = [ctypes.c_void_p]; L.milo_debug_timeline.restype = None
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush.zero_() if os.environ.get("NOFLUSH") != "1" else None
L.milo_debug_timeline(ctypes.c_void_p(dbg.data_ptr()))
run(); torch.cuda.synchronize()
L.milo_debug_timeline(None)
d = dbg.cpu().numpy().reshape(-1, 16).astype(np.float64)
t0 = d[:, 0][d[:, 0] > 0].min()
names = ["start", "stage0 done", "p1 start", "p1 units end", "p1 done", "p2 start", "p2 units end", "end",
         "F enter", "F atomic", "F summed", "F tflag", "F tv done", "F h stored", "F h st issued", "xrep done"]
for i in [0, 15, 1, 2, 3, 8, 9, 10, 11, 12, 14, 13, 4, 5, 6, 7]:
    nm = names[i]
    v = d[:, i][d[:, i] > 0] - t0
    if len(v): print(f"{nm:14s} n={len(v):5d} min={v.min()/1e3:7.2f} med={np.median(v)/1e3:7.2f} p90={np.percentile(v,90)/1e3:7.2f} max={v.max()/1e3:7.2f} us")

v = d[:, 14]
for a_, b_ in [(3, 8), (8, 9), (9, 10), (10, 11), (11, 12), (12, 14), (14, 13), (13, 4), (3, 4)]:
    ok = (d[:, a_] > 0) & (d[:, b_] > 0)
    v = d[ok, b_] - d[ok, a_]
    if len(v): print(f"  {names[a_]:>12s} -> {names[b_]:<12s} n={len(v):5d} med={np.median(v)/1e3:6.2f} p90={np.percentile(v,90)/1e3:6.2f} max={v.max()/1e3:6.2f} us")
d_all = d
d = d[d[:, 0] > 0]
for i, nm in ([(11, "wait cyc"), (12, "finish cyc"), (13, "issue cyc"), (14, "units"), (10, "compute cyc"), (8, "compute p1 cyc"), (9, "wait_h cyc")] if os.environ.get("TIMERS") else []):
    v = d[:, i]
    print(f"{nm:12s} min={v.min():10.0f} med={np.median(v):10.0f} p90={np.percentile(v,90):10.0f} max={v.max():10.0f}  (us at 1.965GHz: med {np.median(v)/1965:.2f})")
ue = d[:, 3] - t0; dn = d[:, 4] - t0
order = np.argsort(-dn)[:12]
print("latest p1-done warps (gw, cta, warp, units_end us, done us):")
for w in order:
    print(f"  gw={w:5d} cta={w // 12 if mode == 'linear' else w // 8:4d} units_end={ue[w]/1e3:7.2f} done={dn[w]/1e3:7.2f}")
order = np.argsort(-ue)[:8]
print("latest units-end warps:", [(int(w), round(ue[w]/1e3, 1)) for w in order])
