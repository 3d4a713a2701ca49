"""Generates tests/golden/golden_v1.npz from the REFERENCE itself.

Runs only where oracle/_ref/libmilo_ref.so exists (built by oracle/build_ref.sh
from the unmodified /root/reference/proj/src sources).  Every array here is an
input or an output of a reference function; tests/test_oracle_golden.py then
pins our C restatement (oracle/milo_oracle.c) against them bit for bit, on any
machine, without /root/reference.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Comp, GemmCfg, Oracle, OracleError  # noqa: E402

OUT = os.path.join(HERE, "golden_v1.npz")


def main():
    r = Oracle("ref")
    g = {}
    rng = np.random.default_rng(2024)

    # ---- binary16 boundary (half.hpp:47-158) --------------------------------
    pats = np.arange(65536, dtype=np.uint32)
    g["h2f_all"] = np.array([r.half_to_float(int(h)) for h in pats], np.float32)
    f = np.concatenate([
        rng.uniform(-70000, 70000, 4000), rng.normal(0, 1, 4000), rng.normal(0, 1e-5, 2000),
        np.array([0.0, -0.0, 1.0, 1024.0, 1028.0, 0.125, -132.0, -128.0, 65504.0, 65520.0, 1e30,
                  5.96046448e-8, 1.0 + 0.00048828125, 1.0 + 3 * 0.00048828125, np.inf, -np.inf,
                  np.nan, 2.98e-8, 6.1e-5, 6.09e-5])]).astype(np.float32)
    g["f2h_in"] = f
    g["f2h_out"] = np.array([r.float_to_half(float(x)) for x in f], np.uint16)
    d = np.concatenate([rng.normal(0, 100, 2000), rng.uniform(-1, 1, 1000) * 1e-6,
                        np.array([1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11, 65519.99, 65520.0])])
    g["d2h_in"] = d
    g["d2h_out"] = np.array([r.double_to_half(float(x)) for x in d], np.uint16)
    abc = rng.integers(0, 65536, (5000, 3), dtype=np.uint32).astype(np.uint16)
    # keep finite operands
    fin = np.array([[np.isfinite(g["h2f_all"][v]) for v in row] for row in abc]).all(1)
    abc = abc[fin]
    g["hops_in"] = abc
    g["hops_out"] = np.array([[r.half_add(int(a), int(b)), r.half_sub(int(a), int(b)),
                               r.half_mul(int(a), int(b)), r.half_fma(int(a), int(b), int(c))]
                              for a, b, c in abc], np.uint16)
    sz = np.array([[int(r.float_to_half(float(s))), int(r.float_to_half(float(z)))]
                   for s, z in zip(np.abs(rng.normal(0, 1, 400)) + 0.01, rng.normal(3, 2, 400))],
                  np.uint16)
    g["scale_zero_in"] = sz
    g["step_off_out"] = np.array([[r.symmetric_step(int(s)), r.asymmetric_offset(int(s), int(z))]
                                  for s, z in sz], np.uint16)

    # ---- pack32 / unpack32 / fast_dequant_pair (pack.cpp:33-68,224-234) -----
    codes32 = rng.integers(0, 8, (2000, 32), dtype=np.uint8)
    codes32[0] = 0
    codes32[1] = 7
    codes32[2] = np.arange(32) % 8
    g["pack32_in"] = codes32
    g["pack32_out"] = np.stack([r.pack32(c) for c in codes32])
    words = rng.integers(0, 2 ** 32, 500, dtype=np.uint64).astype(np.uint32)
    g["fdp_in"] = words
    g["fdp_out"] = np.array([[r.fast_dequant_pair(int(w), p, m) for p in range(4) for m in (0, 1)]
                             for w in words], np.uint16)

    # ---- matrix packing (pack.cpp:97-211,244-302) ----------------------------
    for name, (rows, cols, seed) in {"pm0": (32, 128, 21), "pm1": (48, 128, 22),
                                     "pm2": (64, 192, 23)}.items():
        rs = np.random.default_rng(seed)
        codes = rs.integers(0, 8, (rows, cols), dtype=np.uint8)
        sc = (np.abs(rs.normal(0, 1, rows * cols // 64)) + 0.1).astype(np.float32)
        ze = (3.5 + rs.normal(0, 1, rows * cols // 64)).astype(np.float32)
        g[name + "_codes"], g[name + "_scales"], g[name + "_zeros"] = codes, sc, ze
        for tiled in (0, 1):
            for split in (0, 1):
                P = r.pack_matrix(codes, sc, ze, tiled=bool(tiled), split=bool(split))
                key = f"{name}_t{tiled}s{split}"
                if split:
                    g[key + "_pa"], g[key + "_pb"] = P.plane_a, P.plane_b
                else:
                    g[key + "_words"] = P.words
                g[key + "_sh"], g[key + "_zh"] = P.scales, P.zeros
                g[key + "_unpack"] = r.unpack_codes(P)
                g[key + "_dq_asym"] = r.dequant_half(P, 1)
        Ps = r.pack_matrix(codes, sc, None)
        g[name + "_sym_words"], g[name + "_sym_sh"] = Ps.words, Ps.scales
        g[name + "_sym_dq"] = r.dequant_half(Ps, 0)

    # ---- quantizers (quant.cpp:23-76, lowrank.cpp:89-134) ---------------------
    wq = np.random.default_rng(31).normal(0, 0.05, (64, 128)).astype(np.float32)
    wq[3, :64] = 0.0  # degenerate group -> floor scale
    g["quant_in"] = wq
    c, s, z = r.quantize_minmax(wq)
    g["quant_codes"], g["quant_scales"], g["quant_zeros"] = c, s, z
    sv = np.random.default_rng(32).normal(0, 1, (16, 70)).astype(np.float32)
    sv[0, :3] = [2.0, -1.0, 0.5]
    sv[1, :] = 0.0
    g["symm_in"] = sv
    qc, qs = r.symm_int3_quantize(sv, 16, 70)
    g["symm_codes"], g["symm_scales"] = qc, qs
    g["symm_deq"] = r.symm_int3_dequantize(qc, qs)

    # ---- the hot path: gemm_w3a16 (gemm.cpp:117-199) --------------------------
    gemm_cases = []
    for ci, (k, n, m, mode, rank, storage, tile, mat) in enumerate([
            (128, 256, 5, 1, 0, 1, (128, 128), 0), (128, 256, 17, 0, 0, 1, (64, 256), 0),
            (256, 256, 16, 1, 4, 0, (128, 128), 0), (256, 256, 16, 1, 4, 0, (128, 128), 1),
            (256, 512, 3, 1, 32, 1, (256, 64), 0), (640, 256, 8, 1, 0, 1, (128, 128), 0),
            (256, 128, 1, 0, 70, 1, (128, 128), 0)]):
        seed = r.fnv1a64(f"gemm-{k}x{n}") + ci
        P = r.random_packed(k, n, mode, seed)
        A = r.fill_normal(seed ^ 0xA5A5A5A5, m * k).reshape(m, k)
        comp = None
        if rank:
            U = r.fill_normal(seed + 1, k * rank, 0.0, 0.1).reshape(k, rank)
            V = r.fill_normal(seed + 2, rank * n, 0.0, 0.1).reshape(rank, n)
            comp = Comp(k, n, rank, 0, U, V) if storage == 0 else r.quantize_comp(U, V)
        cfg = GemmCfg(tile[0], tile[1], 64, mode, 4, bool(mat))
        C = r.gemm_w3a16(A, P, comp, cfg)
        key = f"gemm{ci}"
        g[key + "_words"], g[key + "_sh"] = P.words, P.scales
        if P.zeros is not None:
            g[key + "_zh"] = P.zeros
        g[key + "_A"], g[key + "_C"] = A, C
        g[key + "_meta"] = np.array([k, n, m, mode, rank, storage, tile[0], tile[1], mat], np.int64)
        if comp is not None:
            if storage == 0:
                g[key + "_U"], g[key + "_V"] = comp.U, comp.V
            else:
                g[key + "_qu"], g[key + "_qus"] = comp.qu_codes, comp.qu_scales
                g[key + "_qvt"], g[key + "_qvts"] = comp.qvt_codes, comp.qvt_scales
        gemm_cases.append(ci)
    g["gemm_cases"] = np.array(gemm_cases, np.int64)

    # error categories (pipeline.cpp:440-474, test_gemm.cpp:209-233)
    P = r.random_packed(128, 256, 1, 7)
    A = np.zeros((4, 128), np.float32)
    errs = []
    for cfg, a in [(GemmCfg(128, 128, 32, 1), A), (GemmCfg(256, 64, 64, 1), A),
                   (GemmCfg(32, 32, 64, 1), A), (GemmCfg(128, 128, 64, 0), A),
                   (GemmCfg(128, 128, 64, 1, 0), A), (GemmCfg(128, 128, 64, 1), A[:, :64])]:
        try:
            r.gemm_w3a16(a, P, None, cfg)
            errs.append(0)
        except OracleError as e:
            errs.append(e.status)
    g["gemm_err_status"] = np.array(errs, np.int64)

    g["tail_sched"] = np.array([len(r.pipeline_tail_check(kk, GemmCfg())) for kk in
                                (512, 640, 1408, 4096)], np.int64)
    g["mmb"] = np.array([r.matrix_memory_bytes(rr, cc, rk) for rr, cc, rk in
                         [(4096, 14336, 32), (4096, 14336, 0), (2048, 1408, 16), (1408, 2048, 512),
                          (7168, 4864, 16)]], np.uint64)

    # ---- MoE composition over the reference gemm_w3a16 ------------------------
    d, fdim, E, K, mtok = 128, 256, 4, 2, 6
    rs = np.random.default_rng(77)
    experts = []
    for e in range(E + 1):
        ws, cs = [], []
        for j, (kk, nn) in enumerate([(d, fdim), (d, fdim), (fdim, d)]):
            P = r.random_packed(kk, nn, 1, 1000 + 10 * e + j)
            rank = [8, 4, 16][j] if e % 2 == 0 else 0
            comp = None
            if rank:
                comp = r.quantize_comp(rs.normal(0, 0.05, (kk, rank)).astype(np.float32),
                                       rs.normal(0, 0.05, (rank, nn)).astype(np.float32))
                g[f"moe_e{e}_{j}_qu"], g[f"moe_e{e}_{j}_qus"] = comp.qu_codes, comp.qu_scales
                g[f"moe_e{e}_{j}_qvt"], g[f"moe_e{e}_{j}_qvts"] = comp.qvt_codes, comp.qvt_scales
            g[f"moe_e{e}_{j}_words"], g[f"moe_e{e}_{j}_sh"] = P.words, P.scales
            g[f"moe_e{e}_{j}_zh"] = P.zeros
            ws.append(P)
            cs.append(comp)
        experts.append({"w": ws, "c": cs})
    x = rs.normal(0, 1, (mtok, d)).astype(np.float32)
    logits = rs.normal(0, 1, (mtok, E)).astype(np.float32)
    o = Oracle("oracle")
    ids, wts = o.router_topk(logits, K, 0)
    g["moe_x"], g["moe_logits"], g["moe_ids"], g["moe_w"] = x, logits, ids, wts
    g["moe_out"] = r.moe_forward(experts[:E], experts[E:], x, ids, wts)
    g["moe_meta"] = np.array([d, fdim, E, K, mtok, 1], np.int64)

    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes,", len(g), "arrays")


if __name__ == "__main__":
    main()
