import sys, os, ctypes, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_02658_b200 as mb
from paper_2504_02658_b200.synth import packed_random_words
m = int(sys.argv[1]) if len(sys.argv) > 1 else 128
rng = np.random.default_rng(0)
W = mb.Weight(packed_random_words(4096, 14336, rng))
A = torch.randn(m, 4096, device="cuda").half(); out = torch.empty(m, 14336, device="cuda", dtype=torch.float16)
for _ in range(3): mb.gemm_w3a16(A, W, None, out=out)
dbg = torch.zeros(148 * 8 + 64 * 4, dtype=torch.int64, device="cuda")
L = mb.lib(); L.milo_debug_flags.argtypes = [ctypes.c_int]; L.milo_debug_flags(int(os.environ.get("PF_FLAGS", "0")))
L.milo_debug_timeline.argtypes = [ctypes.c_void_p]; L.milo_debug_timeline.restype = None
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); fl.zero_(); torch.cuda.synchronize()
L.milo_debug_timeline(ctypes.c_void_p(dbg.data_ptr())); mb.gemm_w3a16(A, W, None, out=out); torch.cuda.synchronize(); L.milo_debug_timeline(None)
dd = dbg.cpu().numpy().astype(np.float64); d = dd[:148*8].reshape(-1, 8); tr = dd[148*8:].reshape(64, 4); v = d[:, 0] > 0; d = d[v]; t0 = d[:, 0].min()
for i, nm in enumerate(["start", "packed prod done", "B prod done", "dequant w0 done", "mma done", "epi/end", "epi acc_full seen", "deq first packed"]):
    x = d[:, i][d[:, i] > 0] - t0
    if len(x): print(f"{nm:22s} n={len(x):4d} min={x.min()/1e3:7.2f} med={np.median(x)/1e3:7.2f} max={x.max()/1e3:7.2f} us")

tr = np.where(tr > 0, tr - t0, np.nan) / 1e3
print("stage: packed_issued [flags32: commit issued] a_full_seen [flags32: commit landed] (us, CTA 0)")
for st in list(range(0, 12)) + list(range(30, 34)) + list(range(60, 64)):
    print(st, " ".join(f"{x:7.2f}" for x in tr[st]))
