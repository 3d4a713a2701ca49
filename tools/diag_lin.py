"""Diagnostic: single W3A16(+LoRC) linear on the GPU vs fp64 vs the oracle across the
decode (m <= 16), decode NT=2 and tcgen05 (m >= 64) paths.  python tools/diag_lin.py"""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.helpers import rel_err
from tests.test_gpu_real_configs import _oracle_packed, _oracle_comp
import paper_2504_02658_b200 as mb
from paper_2504_02658_b200.synth import packed_random_words
from paper_2504_02658_b200.pack import random_compensator
from oracle.oracle import Oracle

o = Oracle("oracle")
rng = np.random.default_rng(5)
k, n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096, int(sys.argv[2]) if len(sys.argv) > 2 else 14336
P = packed_random_words(k, n, rng)
c = random_compensator(k, n, 32, rng)
W = mb.Weight(P); Cd = mb.Comp(c)
wd = o.dequant_half(_oracle_packed(P)).view(np.float16).astype(np.float64).reshape(k, n)
def compf(c):
    U = (c.qu_codes.astype(np.float64) - 4) * (c.qu_scales[:, :1] * np.float32(2 / 7)).astype(np.float64)
    V = (c.qvt_codes.astype(np.float64) - 4) * (c.qvt_scales[:, :1] * np.float32(2 / 7)).astype(np.float64)
    return U, V.T
U, V = compf(c)
for m in (1, 2, 16, 17, 40, 64, 256):
    A = np.random.default_rng(m).normal(0, 1, (m, k)).astype(np.float32)
    Ah = A.astype(np.float16).astype(np.float64)
    for withc in (False, True):
        ref = Ah @ wd + ((Ah @ U) @ V if withc else 0)
        got = mb.gemm_w3a16(torch.from_numpy(A).cuda(), W, Cd if withc else None).cpu().numpy()
        rows = list(range(min(m, 4)))
        orc = o.gemm_w3a16(A[rows], _oracle_packed(P), _oracle_comp(c) if withc else None)
        print(f"m={m:4d} comp={int(withc)}: gpu-f64 {rel_err(got, ref):.3g}  oracle-f64(rows<4) {rel_err(orc, ref[rows]):.3g}  gpu-oracle(rows<4) {rel_err(got[rows], orc):.3g}", flush=True)
