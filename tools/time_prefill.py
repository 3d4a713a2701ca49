import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_02658_b200 as mb
from paper_2504_02658_b200.synth import packed_random_words
rng = np.random.default_rng(0)
W = mb.Weight(packed_random_words(4096, 14336, rng))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); fr = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
for m in [int(x) for x in (sys.argv[1:] or ["64", "128", "256", "512", "1024", "2048"])]:
    A = torch.randn(m, 4096, device="cuda").half(); out = torch.empty(m, 14336, device="cuda", dtype=torch.float16)
    for _ in range(3): mb.gemm_w3a16(A, W, None, out=out)
    ts = []
    for _ in range(10):
        flush.zero_(); torch.sum(fr)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); mb.gemm_w3a16(A, W, None, out=out); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    us = float(np.median(ts)); fl = 2 * m * 4096 * 14336
    print(f"m={m:5d}: {us:8.1f} us  {fl / us / 1e6:7.1f} TFLOP/s  {(25.7e6 + 2*m*(4096+14336)) / us / 1e3:7.1f} GB/s")
