"""MoE-layer parity cases run in a fresh process, so that process-wide switches read once
by the library (MILO_LEGACY=1: the round-1 multi-launch path; MILO_HDEC=1: the h-local
decode kernel, hdec.cuh) take effect.  Invoked by tests/test_gpu_env_paths.py; prints
one line per case and exits non-zero on the first failure.

    python tests/env_parity_main.py <case> ...   cases: mixtral, deepseek, nonpf, linear
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2504_02658_b200 as mb  # noqa: E402
from oracle.oracle import GemmCfg, Oracle  # noqa: E402
from tests.helpers import random_comp, random_quantized, rel_err  # noqa: E402

TOL = 1e-4


def experts(o, E, d, f, ranks, seed):
    o_ex, g_ex = [], []
    for e in range(E):
        ws, cs, gw, gc = [], [], [], []
        for j, (k, n) in enumerate([(d, f), (d, f), (f, d)]):
            P, _ = random_quantized(o, k, n, seed=seed + 31 * e + j)
            r = ranks[e][j]
            c = random_comp(o, k, n, r, seed=seed + 977 * e + j) if r else None
            ws.append(P)
            cs.append(c)
            gw.append(mb.Weight(P))
            gc.append(mb.Comp(c) if c is not None else None)
        o_ex.append({"w": ws, "c": cs})
        g_ex.append(mb.Expert(gw[0], gw[1], gw[2], gc[0], gc[1], gc[2]))
    return o_ex, g_ex


def layer_case(o, name, E, K, S, d, f, ranks, sranks, score, ms, seed):
    o_ex, g_ex = experts(o, E, d, f, ranks, seed)
    o_sh, g_sh = experts(o, S, d, f, sranks, seed + 5000) if S else ([], [])
    layer = mb.MoELayer(g_ex, g_sh, top_k=K, score_mode=score)
    for m in ms:
        rng = np.random.default_rng(seed + m)
        x = rng.normal(0, 1, (m, d)).astype(np.float32)
        logits = rng.normal(0, 1, (m, E)).astype(np.float32)
        ids, w = o.router_topk(logits, K, score)
        want = o.moe_forward(o_ex, o_sh, x, ids, w)
        out, gids, _ = layer.forward(torch.from_numpy(x).cuda(), torch.from_numpy(logits).cuda(),
                                     return_routing=True)
        assert (gids.cpu().numpy() == ids).all(), f"{name} m={m}: routing ids differ"
        err = rel_err(out.cpu().numpy(), want)
        # binary16 activations, f16 output
        out16 = layer.forward(torch.from_numpy(x).cuda().half(), torch.from_numpy(logits).cuda(),
                              out_dtype=torch.float16).float().cpu().numpy()
        err16 = rel_err(out16, want)
        print(f"{name} m={m}: rel_err {err:.3g} (f16 in/out {err16:.3g})", flush=True)
        assert err <= TOL and err16 <= 1e-3, f"{name} m={m}: {err} / {err16}"


def linear_case(o):
    for (k, n, m, r, tile) in [(256, 512, 40, 32, (128, 128)), (512, 384, 23, 0, (128, 128)),
                               (768, 192, 100, 8, (256, 64))]:
        P, _ = random_quantized(o, k, n, seed=k + n + m)
        c = random_comp(o, k, n, r, seed=7 + r) if r else None
        rng = np.random.default_rng(m)
        A = rng.normal(0, 1, (m, k)).astype(np.float32)
        want = o.gemm_w3a16(A, P, c, cfg=GemmCfg(tile_k=tile[0], tile_n=tile[1], mode=1))
        got = mb.gemm_w3a16(torch.from_numpy(A).cuda(), mb.Weight(P), mb.Comp(c) if c is not None else None,
                            cfg=mb.GemmConfig(tile_shape=tile, mode=1))
        err = rel_err(got.cpu().numpy(), want)
        print(f"linear {k}x{n} r{r} m={m}: rel_err {err:.3g}", flush=True)
        assert err <= 1e-5, err


def main():
    os.chdir(ROOT)
    o = Oracle("oracle")
    mb.device_check()
    for case in sys.argv[1:]:
        if case == "mixtral":
            ranks = [[(8 * ((e + j) % 4)) for j in range(3)] for e in range(8)]
            layer_case(o, "mixtral-like", 8, 2, 0, 256, 512, ranks, [], 0, [1, 3, 8, 13, 16], 100)
        elif case == "deepseek":
            ranks = [[(0, 8, 16)[(e + j) % 3] for j in range(3)] for e in range(16)]
            layer_case(o, "deepseek-like", 16, 6, 2, 256, 128, ranks, [[96, 64, 80], [16, 0, 32]], 1,
                       [1, 2, 9, 16], 300)
        elif case == "nonpf":  # f % 128 == 64: no prefill kernel; m > 64
            ranks = [[(0, 16, 8)[(e + j) % 3] for j in range(3)] for e in range(8)]
            layer_case(o, "non-prefill", 8, 2, 1, 256, 192, ranks, [[8, 0, 16]], 0, [5, 150], 700)
        elif case == "linear":
            linear_case(o)
        else:
            raise SystemExit(f"unknown case {case}")
    print("ok")


if __name__ == "__main__":
    main()
