"""Pins the C restatement (oracle/milo_oracle.c) to the reference's own outputs.

tests/golden/golden_v1.npz was produced by tests/golden/make_golden.py from
the reference sources compiled unmodified (oracle/build_ref.sh); every check
here is bit-exact.  Runs on CPU anywhere (no /root/reference needed).
"""
import os

import numpy as np
import pytest

from oracle.oracle import Comp, GemmCfg, OracleError, Packed

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_v1.npz")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def g():
    return np.load(GOLD)


def test_half_decode_all_patterns(oracle, g):
    got = np.array([oracle.half_to_float(h) for h in range(65536)], np.float32)
    want = g["h2f_all"]
    nan = np.isnan(want)
    assert (np.isnan(got) == nan).all()
    assert (got.view(np.uint32)[~nan] == want.view(np.uint32)[~nan]).all()


def test_half_encode_and_ops(oracle, g):
    got = np.array([oracle.float_to_half(float(x)) for x in g["f2h_in"]], np.uint16)
    assert (got == g["f2h_out"]).all()
    got = np.array([oracle.double_to_half(float(x)) for x in g["d2h_in"]], np.uint16)
    assert (got == g["d2h_out"]).all()
    ops = np.array([[oracle.half_add(int(a), int(b)), oracle.half_sub(int(a), int(b)),
                     oracle.half_mul(int(a), int(b)), oracle.half_fma(int(a), int(b), int(c))]
                    for a, b, c in g["hops_in"]], np.uint16)
    assert (ops == g["hops_out"]).all()
    so = np.array([[oracle.symmetric_step(int(s)), oracle.asymmetric_offset(int(s), int(z))]
                   for s, z in g["scale_zero_in"]], np.uint16)
    assert (so == g["step_off_out"]).all()


def test_known_encodings(oracle):
    # test_half.cpp:48-71
    f2h = oracle.float_to_half
    assert [f2h(x) for x in (0.0, -0.0, 1.0, 1024.0, 1028.0, 0.125, -132.0, -128.0)] == \
        [0x0000, 0x8000, 0x3C00, 0x6400, 0x6404, 0x3000, 0xD820, 0xD800]
    assert f2h(65504.0) == 0x7BFF and f2h(65520.0) == 0x7C00 and f2h(1e30) == 0x7C00
    assert f2h(5.96046448e-8) == 0x0001
    assert f2h(1.0 + 0.00048828125) == 0x3C00 and f2h(1.0 + 3 * 0.00048828125) == 0x3C02
    assert oracle.half_add(f2h(2048.0), 0x3C00) == f2h(2048.0)


def test_pack32_unpack32(oracle, g):
    for c, w in zip(g["pack32_in"], g["pack32_out"]):
        assert (oracle.pack32(c) == w).all()
        assert (oracle.unpack32(w) == c).all()
    assert (g["pack32_out"][0] == 0).all() and (g["pack32_out"][1] == 0xFFFFFFFF).all()
    bad = np.zeros(32, np.uint8)
    bad[3] = 8
    with pytest.raises(OracleError) as e:
        oracle.pack32(bad)
    assert e.value.category == "range"
    with pytest.raises(OracleError) as e:
        oracle.pack32(np.zeros(31, np.uint8))
    assert e.value.category == "shape"


def test_fast_dequant_pair(oracle, g):
    got = np.array([[oracle.fast_dequant_pair(int(w), p, m) for p in range(4) for m in (0, 1)]
                    for w in g["fdp_in"]], np.uint16)
    assert (got == g["fdp_out"]).all()


@pytest.mark.parametrize("name", ["pm0", "pm1", "pm2"])
def test_pack_matrix_layouts(oracle, g, name):
    codes, sc, ze = g[name + "_codes"], g[name + "_scales"], g[name + "_zeros"]
    for tiled in (0, 1):
        for split in (0, 1):
            key = f"{name}_t{tiled}s{split}"
            P = oracle.pack_matrix(codes, sc, ze, tiled=bool(tiled), split=bool(split))
            if split:
                assert (P.plane_a == g[key + "_pa"]).all() and (P.plane_b == g[key + "_pb"]).all()
            else:
                assert (P.words == g[key + "_words"]).all()
            assert (P.scales == g[key + "_sh"]).all() and (P.zeros == g[key + "_zh"]).all()
            assert (oracle.unpack_codes(P) == g[key + "_unpack"]).all()
            assert (oracle.unpack_codes(P) == codes).all()
            assert (oracle.dequant_half(P, 1) == g[key + "_dq_asym"]).all()
    Ps = oracle.pack_matrix(codes, sc, None)
    assert (Ps.words == g[name + "_sym_words"]).all() and (Ps.scales == g[name + "_sym_sh"]).all()
    assert (oracle.dequant_half(Ps, 0) == g[name + "_sym_dq"]).all()


def test_quantizers(oracle, g):
    c, s, z = oracle.quantize_minmax(g["quant_in"])
    assert (c == g["quant_codes"]).all()
    assert (s.view(np.uint32) == g["quant_scales"].view(np.uint32)).all()
    assert (z.view(np.uint32) == g["quant_zeros"].view(np.uint32)).all()
    qc, qs = oracle.symm_int3_quantize(g["symm_in"], 16, 70)
    assert (qc == g["symm_codes"]).all() and (qs == g["symm_scales"]).all()
    c3, s3 = oracle.symm_int3_quantize(np.array([2.0, -1.0, 0.5], np.float32), 1, 3)
    assert list(c3[0]) == [7, 2, 5] and s3[0, 0] == 2.0  # test_lowrank.cpp:94-99 (code wins)
    assert (oracle.symm_int3_dequantize(qc, qs) == g["symm_deq"]).all()


def _packed(g, key, k, n, mode):
    return Packed(k, n, 0, False, mode, 64, g[key + "_words"], None, None, g[key + "_sh"],
                  g[key + "_zh"] if (key + "_zh") in g.files else None)


def test_gemm_w3a16_bit_exact(oracle, g):
    for ci in g["gemm_cases"]:
        key = f"gemm{ci}"
        k, n, m, mode, rank, storage, tk, tn, mat = (int(x) for x in g[key + "_meta"])
        P = _packed(g, key, k, n, mode)
        comp = None
        if rank:
            if storage == 0:
                comp = Comp(k, n, rank, 0, g[key + "_U"], g[key + "_V"])
            else:
                comp = Comp(k, n, rank, 1, None, None, g[key + "_qu"], g[key + "_qus"],
                            g[key + "_qvt"], g[key + "_qvts"])
        C = oracle.gemm_w3a16(g[key + "_A"], P, comp, GemmCfg(tk, tn, 64, mode, 4, bool(mat)))
        assert (C.view(np.uint32) == g[key + "_C"].view(np.uint32)).all(), key


def test_gemm_error_categories(oracle, g):
    from tests.helpers import random_quantized
    P, _ = random_quantized(oracle, 128, 256, seed=7)
    A = np.zeros((4, 128), np.float32)
    got = []
    for cfg, a in [(GemmCfg(128, 128, 32, 1), A), (GemmCfg(256, 64, 64, 1), A),
                   (GemmCfg(32, 32, 64, 1), A), (GemmCfg(128, 128, 64, 0), A),
                   (GemmCfg(128, 128, 64, 1, 0), A), (GemmCfg(128, 128, 64, 1), A[:, :64])]:
        try:
            oracle.gemm_w3a16(a, P, None, cfg)
            got.append(0)
        except OracleError as e:
            got.append(e.status)
    assert got == list(g["gemm_err_status"])


def test_schedule_and_accounting(oracle, g):
    assert [len(oracle.pipeline_tail_check(k, GemmCfg())) for k in (512, 640, 1408, 4096)] == \
        list(g["tail_sched"])
    assert oracle.pipeline_tail_check(5 * 128, GemmCfg()) == [4, 1]
    assert oracle.pipeline_tail_check(11 * 128, GemmCfg()) == [4, 4, 3]
    got = [oracle.matrix_memory_bytes(r, c, k) for r, c, k in
           [(4096, 14336, 32), (4096, 14336, 0), (2048, 1408, 16), (1408, 2048, 512),
            (7168, 4864, 16)]]
    assert got == [int(x) for x in g["mmb"]]
    assert got[0] == 25_690_112 + 258_048


def _moe_experts(g):
    d, f, E, K, m, _ = (int(x) for x in g["moe_meta"])
    experts = []
    for e in range(E + 1):
        ws, cs = [], []
        for j, (kk, nn) in enumerate([(d, f), (d, f), (f, d)]):
            key = f"moe_e{e}_{j}"
            ws.append(Packed(kk, nn, 0, False, 1, 64, g[key + "_words"], None, None,
                             g[key + "_sh"], g[key + "_zh"]))
            if key + "_qu" in g.files:
                cs.append(Comp(kk, nn, g[key + "_qu"].shape[1], 1, None, None, g[key + "_qu"],
                               g[key + "_qus"], g[key + "_qvt"], g[key + "_qvts"]))
            else:
                cs.append(None)
        experts.append({"w": ws, "c": cs})
    return experts[:E], experts[E:]


def test_moe_composition_matches_reference(oracle, g):
    routed, shared = _moe_experts(g)
    ids, w = oracle.router_topk(g["moe_logits"], int(g["moe_meta"][3]), 0)
    assert (ids == g["moe_ids"]).all()
    out = oracle.moe_forward(routed, shared, g["moe_x"], ids, w)
    assert (out.view(np.uint32) == g["moe_out"].view(np.uint32)).all()
    out4 = oracle.moe_forward(routed, shared, g["moe_x"], ids, w, n_threads=4)
    assert (out4 == out).all()


def test_router_topk_ties_and_modes(oracle):
    logits = np.array([[1.0, 3.0, 3.0, 0.5], [2.0, 2.0, 2.0, 2.0]], np.float32)
    ids, w = oracle.router_topk(logits, 2, 0)
    assert ids.tolist() == [[1, 2], [0, 1]]
    assert np.allclose(w, 0.5)
    ids, w = oracle.router_topk(logits, 2, 1)
    p = np.exp(logits[0] - 3.0)
    assert np.allclose(w[0], p[[1, 2]] / p.sum(), rtol=1e-6)


def test_restatement_matches_compiled_reference_directly(oracle, ref):
    """Where oracle/_ref exists (this container), also cross-check live."""
    from tests.helpers import random_quantized, random_comp
    for mode in (1, 0):
        P, _ = random_quantized(oracle, 256, 512, seed=3 + mode, mode=mode)
        comp = random_comp(oracle, 256, 512, 16, seed=5)
        A = np.random.default_rng(4).normal(0, 1, (9, 256)).astype(np.float32)
        cfg = GemmCfg(mode=mode)
        a = oracle.gemm_w3a16(A, P, comp, cfg)
        b = ref.gemm_w3a16(A, P, comp, cfg)
        assert (a.view(np.uint32) == b.view(np.uint32)).all()


def test_reference_moe_column_slices_are_bit_identical(oracle, ref, g):
    """bench.py's reference arm cuts every matrix into column slices so all host
    threads work at batch 1 (oracle/ref/ref_capi.cpp ref_moe_forward); the
    reference's columns are independent, so any slice count must give the same
    bits as the unsliced composition, which equals the golden MoE output."""
    from oracle.oracle import RefMoE
    routed, shared = _moe_experts(g)
    ids, w = oracle.router_topk(g["moe_logits"], int(g["moe_meta"][3]), 0)
    outs = []
    for workers in (1, 2, 3, 8):
        h = RefMoE(ref, routed, shared, workers)
        outs.append(h.forward(g["moe_x"], ids, w))
        h.close()
    for o in outs:
        assert (o.view(np.uint32) == g["moe_out"].view(np.uint32)).all()


def test_router_gemm_restatement_is_a_dot_product(oracle):
    """or_router_gemm (the MoE gate in the device's fixed fp32 order) is the
    product half(x) W_gate^T up to fp32 summation: checked against float64."""
    rng = np.random.default_rng(12)
    for m, d, E in [(1, 4096, 8), (5, 2048, 64), (3, 96, 4)]:
        x = rng.normal(0, 1, (m, d)).astype(np.float32)
        gate = (rng.normal(0, 0.02, (E, d))).astype(np.float16)
        got = oracle.router_gemm(x, gate.view(np.uint16))
        want = x.astype(np.float16).astype(np.float64) @ gate.astype(np.float64).T
        assert np.allclose(got, want, rtol=1e-5, atol=1e-6 * np.abs(want).max())
        # lane-order arithmetic: exactly reproducible
        assert np.array_equal(got, oracle.router_gemm(x, gate.view(np.uint16)))


def test_frozen_rank_plans_are_the_references():
    """paper_2504_02658_b200/plans/*.plan.json (the benchmark layers' ranks) are what the
    reference's plan_ranks gives (tools/make_rank_plans.py); re-derived here when the
    compiled reference is present (Mixtral: 24 matrices of 4096 x 14336 synthetic weights)."""
    import json
    from paper_2504_02658_b200.artifacts import load_plan
    from paper_2504_02658_b200.synth import CONFIGS, PLAN_DIR
    for name, spec in CONFIGS.items():
        path = os.path.join(PLAN_DIR, f"{spec.plan}.plan.json")
        plan = load_plan(path)
        routed = [plan.ranks[f"layer0.expert{e}.{w}"] for e in range(spec.experts) for w in ("w1", "w3", "w2")]
        assert abs(np.mean(routed) - 16.0) < 1e-9, name  # Kurtosis-16: total = 16 x #expert matrices
        assert plan.policy.endswith("Kurtosis-16")
        if spec.shared:
            assert all(plan.ranks[f"layer0.shared_expert{s}.{w}"] == 512
                       for s in range(spec.shared) for w in ("w1", "w3", "w2"))
    lib_path = os.path.join(ROOT, "oracle", "_ref", "libmilo_ref.so")
    if not os.path.exists(lib_path):
        return
    import ctypes
    lib = ctypes.CDLL(lib_path)
    f = lib.ref_plan_synth
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                  ctypes.c_uint64, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_void_p, ctypes.c_void_p]
    spec = CONFIGS["mixtral"]
    ranks = np.zeros(spec.experts * 3, np.int32)
    kurt = np.zeros(spec.experts * 3, np.float64)
    assert f(spec.experts, 0, spec.d, spec.f, 0, 0, 0, b"Kurtosis-16", ranks.ctypes.data, kurt.ctypes.data) == 0
    frozen = json.load(open(os.path.join(PLAN_DIR, "mixtral.plan.json")))["ranks"]
    want = [frozen[f"layer0.expert{e}.{w}"] for e in range(spec.experts) for w in ("w1", "w3", "w2")]
    assert ranks.tolist() == want
