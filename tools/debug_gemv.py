import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_02658_b200 as mb
from oracle.oracle import Oracle, GemmCfg
from tests.helpers import random_quantized, rel_err
o = Oracle("oracle")
for (k, n, m, tk, tn) in [(256, 64, 1, 256, 64), (64, 256, 1, 64, 256), (128, 128, 1, 128, 128), (128, 128, 3, 128, 128), (128, 128, 16, 128, 128), (128, 128, 128, 128, 128), (4096, 4096, 1, 128, 128)]:
    P, _ = random_quantized(o, k, n, seed=1)
    A = np.random.default_rng(2).normal(0, 1, (m, k)).astype(np.float32)
    want = o.gemm_w3a16(A, P, cfg=GemmCfg(tile_k=tk, tile_n=tn))
    W = mb.Weight(P)
    try:
        got = mb.gemm_w3a16(torch.from_numpy(A).cuda(), W, cfg=mb.GemmConfig(tile_shape=(tk, tn))).cpu().numpy()
    except Exception as e:
        print(k, n, m, "ERR", e); continue
    if want is not None:
        print(k, n, m, "rel", rel_err(got, want), "got", got[0, :4], "want", want[0, :4], flush=True)
from torch.profiler import profile, ProfilerActivity
P, _ = random_quantized(o, 4096, 14336, seed=7)
W = mb.Weight(P)
A = torch.randn(1, 4096, device="cuda")
for _ in range(3): mb.gemm_w3a16(A, W)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(5): mb.gemm_w3a16(A, W)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
