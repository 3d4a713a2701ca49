"""GPU: the C++ host API (include/milo_b200.hpp) end to end, compiled from
tests/cpp/gpu_run.cpp against the in-tree library: a symm-INT3-compensated GEMM
(DeviceWeight / DeviceCompensator / gemm_w3a16 with host WeightMatrix buffers, the
reference's gemm.hpp:43-48 form) and a MoE layer forward from host buffers, checked
against the CPU oracle (1e-5 GEMM, 1e-4 layer, as the Python-binding tests)."""
import os
import subprocess

import numpy as np
import pytest

from tests.helpers import random_comp, random_quantized, rel_err

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _write_packed(prefix, P):
    P.words.astype(np.uint32).tofile(prefix + ".words")
    P.scales.astype(np.uint16).tofile(prefix + ".scales")
    if P.zeros is not None:
        P.zeros.astype(np.uint16).tofile(prefix + ".zeros")


def test_cpp_api_gemm_and_moe_on_gpu(gpu, oracle, tmp_path):
    from oracle.oracle import GemmCfg
    from paper_2504_02658_b200 import LIB_PATH
    k, n, m, rank = 512, 1024, 3, 32
    d, f, E, K, m2 = 256, 512, 4, 2, 5
    d_ = str(tmp_path)
    P, _ = random_quantized(oracle, k, n, seed=41)
    c = random_comp(oracle, k, n, rank, seed=42)
    _write_packed(d_ + "/lin", P)
    c.qu_codes.astype(np.uint8).tofile(d_ + "/lin.qu_codes")
    c.qu_scales.astype(np.float32).tofile(d_ + "/lin.qu_scales")
    c.qvt_codes.astype(np.uint8).tofile(d_ + "/lin.qvt_codes")
    c.qvt_scales.astype(np.float32).tofile(d_ + "/lin.qvt_scales")
    rng = np.random.default_rng(43)
    A = rng.normal(0, 1, (m, k)).astype(np.float32)
    A.tofile(d_ + "/A.f32")
    o_ex = []
    for e in range(E):
        ws = []
        for j, (kk, nn) in enumerate([(d, f), (d, f), (f, d)]):
            Pe, _ = random_quantized(oracle, kk, nn, seed=500 + 7 * e + j)
            _write_packed(f"{d_}/e{e}_{j}", Pe)
            ws.append(Pe)
        o_ex.append({"w": ws, "c": [None, None, None]})
    x = rng.normal(0, 1, (m2, d)).astype(np.float32)
    logits = rng.normal(0, 1, (m2, E)).astype(np.float32)
    x.tofile(d_ + "/x.f32")
    logits.tofile(d_ + "/logits.f32")
    with open(d_ + "/meta.txt", "w") as fh:
        fh.write(f"{k} {n} {m} {P.mode} {rank} {d} {f} {E} {K} {m2}\n")

    exe = str(tmp_path / "gpu_run")
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "gpu_run.cpp"), LIB_PATH,
                           "-Wl,-rpath," + os.path.dirname(LIB_PATH), "-o", exe])
    res = subprocess.run([exe, d_], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "gpu_run ok" in res.stdout

    C = np.fromfile(d_ + "/C.f32", np.float32).reshape(m, n)
    want = oracle.gemm_w3a16(A, P, c, cfg=GemmCfg(mode=P.mode))
    assert rel_err(C, want) <= 1e-5
    got = np.fromfile(d_ + "/moe.f32", np.float32).reshape(m2, d)
    ids, w = oracle.router_topk(logits, K, 0)
    assert rel_err(got, oracle.moe_forward(o_ex, [], x, ids, w)) <= 1e-4


def test_integration_binding_against_compiled_reference(gpu):
    """INTEGRATION.md section 2, compiled (oracle/ref/b200_binding_check.cpp, built by
    oracle/build_ref.sh into oracle/_ref): the reference's own gemm_w3a16 and the B200
    library through to_b200 copies of the reference's types, on the same inputs."""
    exe = os.path.join(ROOT, "oracle", "_ref", "b200_binding_check")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/b200_binding_check not built (needs /root/reference sources)")
    res = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "binding check ok" in res.stdout
