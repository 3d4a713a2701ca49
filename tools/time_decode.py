"""Times the decode kernel: single linear (C1) and the Mixtral layer, m = 1 / 16."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_02658_b200 as mb
from paper_2504_02658_b200.synth import CONFIGS, build_host_layer, packed_random_words
from paper_2504_02658_b200.pack import random_compensator

NOFLUSH = os.environ.get("NOFLUSH") == "1"
def timeit(fn, n=20):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3): fn()
    ts = []
    for _ in range(n):
        if not NOFLUSH: flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return float(np.median(ts)), float(np.min(ts))

import ctypes
L = mb.lib(); L.milo_debug_flags.argtypes = [ctypes.c_int]; L.milo_debug_flags.restype = None
L.milo_debug_flags(int(os.environ.get("DEC_FLAGS", "0")))
rng = np.random.default_rng(0)
only = sys.argv[1] if len(sys.argv) > 1 else "all"
if only in ("all", "linear"):
    P = packed_random_words(4096, 14336, rng)
    c = random_compensator(4096, 14336, 32, rng)
    W, Cm = mb.Weight(P), mb.Comp(c)
    for m in (1, 16):
        A = torch.randn(m, 4096, device="cuda").half()
        out = torch.empty(m, 14336, device="cuda")
        med, mn = timeit(lambda: mb.gemm_w3a16(A, W, Cm, out=out))
        print(f"linear 4096x14336 r32 m={m}: median {med:.1f} us  min {mn:.1f} us  -> {25.95e6/med/1e3:.0f} GB/s")
if only in ("all", "moe"):
    spec = CONFIGS["mixtral"]
    routed, shared = build_host_layer(spec, 0)
    ex = [mb.Expert(*(mb.Weight(P) for P in h.w), *((mb.Comp(c) if c is not None else None) for c in h.c)) for h in routed]
    layer = mb.MoELayer(ex, [], top_k=2)
    for m in (1, 16):
        x = torch.randn(m, 4096, device="cuda").half()
        lg = torch.randn(m, 8, device="cuda")
        med, mn = timeit(lambda: layer.forward(x, lg, out_dtype=torch.float16))
        print(f"mixtral layer m={m}: median {med:.1f} us  min {mn:.1f} us")
