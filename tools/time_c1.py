"""C1 timing: the 4096 x 14336 linear at m = 1 / 8 / 16, with and without the rank-32
compensator (L2 flushed).  MILO_GEMV_SLAB=0 selects the decode megakernel."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_02658_b200 as mb
from paper_2504_02658_b200.synth import packed_random_words
from paper_2504_02658_b200.pack import random_compensator
rng = np.random.default_rng(0)
W = mb.Weight(packed_random_words(4096, 14336, rng)); Cm = mb.Comp(random_compensator(4096, 14336, 32, rng))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for comp in (None, Cm):
    for m in (1, 8, 16):
        A = torch.randn(m, 4096, device="cuda").half()
        out = torch.empty(m, 14336, device="cuda")
        for _ in range(3): mb.gemm_w3a16(A, W, comp, out=out)
        ts = []
        for _ in range(20):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); mb.gemm_w3a16(A, W, comp, out=out); e.record(); torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        us = float(np.median(ts))
        print(f"4096x14336 {'r32' if comp else 'r0 '} m={m:2d}: {us:7.1f} us  {25.7e6 / us / 1e3:6.0f} GB/s")
