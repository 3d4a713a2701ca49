"""Runs the C1 single linear (4096x14336, r=32) a few times for ncu capture."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_02658_b200 as mb
from paper_2504_02658_b200.synth import packed_random_words
from paper_2504_02658_b200.pack import random_compensator
rng = np.random.default_rng(0)
k, n = int(os.environ.get("K", 4096)), int(os.environ.get("N", 14336))
m = int(os.environ.get("M", 1))
W = mb.Weight(packed_random_words(k, n, rng))
C = mb.Comp(random_compensator(k, n, 32, rng)) if os.environ.get("COMP", "0") == "1" else None
A = torch.randn(m, k, device="cuda").half()
for _ in range(int(os.environ.get("ITERS", 5))):
    mb.gemm_w3a16(A, W, C, out_dtype=torch.float16)
torch.cuda.synchronize()
print("done")
