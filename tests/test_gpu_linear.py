"""GPU parity of the single-linear W3A16 path against the CPU oracle.

Mirrors the reference's own hot-path tests: test_pack.cpp (bit-exact
unpack/dequant), test_gemm.cpp (identity, tiles, linearity, compensator,
errors, padding) and the gemm_correctness gate (acceptance_main.cpp:50-66).
Tolerances: de-quantized weights and codes bit-exact;
fp32 GEMM output <= 1e-5 relative Frobenius vs the oracle; fp16 output <= 5e-4.
"""
import numpy as np
import pytest

from tests.helpers import rel_err, random_comp, random_quantized

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-5
TOL_F16 = 5e-4


def _cfg(mb, mode, tile=(128, 128)):
    return mb.GemmConfig(tile_shape=tile, mode=mode)


@pytest.mark.parametrize("mode,tiled,split", [(1, False, False), (1, True, False), (1, False, True),
                                              (1, True, True), (0, False, False), (0, False, True)])
def test_device_unpack_and_dequant_bit_exact(gpu, oracle, mode, tiled, split):
    P, codes = random_quantized(oracle, 96, 192, seed=21 + mode, mode=mode, tiled=tiled, split=split)
    W = gpu.Weight(P)
    assert W.device_bytes == 96 * 192 * 7 // 16  # 0.4375 B/weight
    got = W.unpack_codes().cpu().numpy()
    assert (got == oracle.unpack_codes(P)).all()
    assert (got == codes).all()
    dq = W.dequant_half().cpu().view(__import__("torch").int16).numpy().view(np.uint16)
    want = oracle.dequant_half(P)
    assert (dq == want).all()


def test_dequant_extreme_scales_bit_exact(gpu, oracle):
    # scales spanning subnormal..large binary16 and zeros in [-3, 10]
    rng = np.random.default_rng(5)
    k, n = 64, 128
    codes = rng.integers(0, 8, (k, n), dtype=np.uint8)
    sc = np.exp(rng.uniform(np.log(1e-6), np.log(500.0), k * n // 64)).astype(np.float32)
    ze = rng.uniform(-3, 10, k * n // 64).astype(np.float32)
    P = oracle.pack_matrix(codes, sc, ze)
    W = gpu.Weight(P)
    import torch
    dq = W.dequant_half().cpu().view(torch.int16).numpy().view(np.uint16)
    assert (dq == oracle.dequant_half(P)).all()
    Ps = oracle.pack_matrix(codes, sc, None)
    Ws = gpu.Weight(Ps)
    dqs = Ws.dequant_half().cpu().view(torch.int16).numpy().view(np.uint16)
    assert (dqs == oracle.dequant_half(Ps)).all()


def test_identity_activations_reproduce_weights(gpu, oracle):
    # test_gemm.cpp:55-79: weights on the grid, A = I -> C == dequant exactly
    import torch
    k = n = 128
    rng = np.random.default_rng(3)
    codes = rng.integers(0, 8, (k, n), dtype=np.uint8)
    P = oracle.pack_matrix(codes, np.full(k * n // 64, 0.25, np.float32),
                           np.full(k * n // 64, 4.0, np.float32))
    W = gpu.Weight(P)
    A = torch.eye(k, dtype=torch.float32, device="cuda")
    C = gpu.gemm_w3a16(A, W, cfg=_cfg(gpu, 1)).cpu().numpy()
    want = np.array([oracle.half_to_float(int(h)) for h in oracle.dequant_half(P).ravel()],
                    np.float32).reshape(k, n)
    assert (C == want).all()


@pytest.mark.parametrize("k,n", [(128, 256), (512, 512), (640, 256)])
@pytest.mark.parametrize("m", [1, 5, 16, 17, 40])
@pytest.mark.parametrize("mode", [1, 0])
def test_gemm_matches_oracle(gpu, oracle, k, n, m, mode):
    import torch
    P, _ = random_quantized(oracle, k, n, seed=k * 7 + n + mode, mode=mode)
    rng = np.random.default_rng(m + 100)
    A = rng.normal(0, 1, (m, k)).astype(np.float32)
    want = oracle.gemm_w3a16(A, P, cfg=_oc(mode))
    W = gpu.Weight(P)
    got = gpu.gemm_w3a16(torch.from_numpy(A).cuda(), W, cfg=_cfg(gpu, mode)).cpu().numpy()
    assert rel_err(got, want) <= TOL_F32
    got16 = gpu.gemm_w3a16(torch.from_numpy(A).cuda().half(), W, cfg=_cfg(gpu, mode),
                           out_dtype=torch.float16).float().cpu().numpy()
    assert rel_err(got16, want) <= TOL_F16


def _oc(mode, materialize=False):
    from oracle.oracle import GemmCfg
    return GemmCfg(mode=mode, materialize_compensator=materialize)


@pytest.mark.parametrize("storage", [1, 0])
@pytest.mark.parametrize("rank", [4, 32, 70])
@pytest.mark.parametrize("m", [1, 8, 16, 19])
def test_gemm_with_compensator(gpu, oracle, storage, rank, m):
    import torch
    k, n = 256, 512
    P, _ = random_quantized(oracle, k, n, seed=31)
    comp = random_comp(oracle, k, n, rank, seed=rank, storage=storage)
    A = np.random.default_rng(32).normal(0, 1, (m, k)).astype(np.float32)
    want = oracle.gemm_w3a16(A, P, comp, _oc(1))
    got = gpu.gemm_w3a16(torch.from_numpy(A).cuda(), gpu.Weight(P), gpu.Comp(comp),
                         cfg=_cfg(gpu, 1)).cpu().numpy()
    assert rel_err(got, want) <= TOL_F32
    # and the materialized form of the reference agrees (test_gemm.cpp:152-159)
    want_mat = oracle.gemm_w3a16(A, P, comp, _oc(1, True))
    assert rel_err(got, want_mat) <= 1e-4


def test_padding_rows_are_bit_identical(gpu, oracle):
    # test_gemm.cpp:235-261 / pipeline.cpp:476-493
    import torch
    k, n = 256, 256
    P, _ = random_quantized(oracle, k, n, seed=11)
    comp = random_comp(oracle, k, n, 16, seed=12)
    W, Cp = gpu.Weight(P), gpu.Comp(comp)
    a5 = np.random.default_rng(13).normal(0, 1, (5, k)).astype(np.float32)
    a16 = np.zeros((16, k), np.float32)
    a16[:5] = a5
    c5 = gpu.gemm_w3a16(torch.from_numpy(a5).cuda(), W, Cp, _cfg(gpu, 1)).cpu().numpy()
    c16 = gpu.gemm_w3a16(torch.from_numpy(a16).cuda(), W, Cp, _cfg(gpu, 1)).cpu().numpy()
    assert (c5 == c16[:5]).all()


def test_tile_configs_and_determinism(gpu, oracle):
    import torch
    k, n = 512, 512
    P, _ = random_quantized(oracle, k, n, seed=41)
    W = gpu.Weight(P)
    A = torch.from_numpy(np.random.default_rng(42).normal(0, 1, (16, k)).astype(np.float32)).cuda()
    want = oracle.gemm_w3a16(A.cpu().numpy(), P, cfg=_oc(1))
    outs = [gpu.gemm_w3a16(A, W, cfg=_cfg(gpu, 1, t)).cpu().numpy()
            for t in [(64, 256), (128, 128), (256, 64)]]
    for o in outs:
        assert rel_err(o, want) <= TOL_F32
        assert (o == outs[0]).all()  # tile shape is validation-only: same kernel, same bits
    again = gpu.gemm_w3a16(A, W, cfg=_cfg(gpu, 1)).cpu().numpy()
    assert (again == outs[0]).all()


def test_error_conditions_match_reference_categories(gpu, oracle):
    # test_gemm.cpp:209-233, pipeline.cpp:440-474
    import torch
    P, _ = random_quantized(oracle, 256, 256, seed=51)
    W = gpu.Weight(P)
    A = torch.zeros((4, 256), device="cuda")
    with pytest.raises(gpu.ConfigError):
        gpu.gemm_w3a16(A, W, cfg=gpu.GemmConfig(group_size=32))
    with pytest.raises(gpu.ConfigError):
        gpu.gemm_w3a16(A, W, cfg=gpu.GemmConfig(tile_shape=(100, 100)))
    with pytest.raises(gpu.ConfigError):
        gpu.gemm_w3a16(A, W, cfg=gpu.GemmConfig(tile_shape=(32, 32)))
    with pytest.raises(gpu.ConfigError):
        gpu.gemm_w3a16(A, W, cfg=gpu.GemmConfig(mode=0))
    with pytest.raises(gpu.ConfigError):
        gpu.gemm_w3a16(A, W, cfg=gpu.GemmConfig(pipeline_depth=0))
    Podd, _ = random_quantized(oracle, 192, 256, seed=53)
    with pytest.raises(gpu.ShapeError):
        gpu.gemm_w3a16(torch.zeros((4, 192), device="cuda"), gpu.Weight(Podd))
    with pytest.raises(gpu.ShapeError):
        gpu.gemm_w3a16(torch.zeros((4, 128), device="cuda"), W)
    comp = random_comp(oracle, 128, 256, 4, seed=1)
    with pytest.raises(gpu.ShapeError):
        gpu.gemm_w3a16(A, W, gpu.Comp(comp))
    Pz = random_quantized(oracle, 256, 256, seed=54)[0]
    Pz.zeros = None
    with pytest.raises(gpu.ConfigError):
        gpu.gemm_w3a16(A, gpu.Weight(Pz))
    # ordering: bad tile (config) wins over bad A shape (shape)
    with pytest.raises(gpu.ConfigError):
        gpu.gemm_w3a16(torch.zeros((4, 128), device="cuda"), W,
                       cfg=gpu.GemmConfig(tile_shape=(32, 32)))


def test_host_entry_point(gpu, oracle):
    k, n = 256, 512
    P, _ = random_quantized(oracle, k, n, seed=61)
    comp = random_comp(oracle, k, n, 8, seed=62)
    A = np.random.default_rng(63).normal(0, 1, (3, k)).astype(np.float32)
    got = gpu.gemm_w3a16_host(A, gpu.Weight(P), gpu.Comp(comp))
    assert rel_err(got, oracle.gemm_w3a16(A, P, comp, _oc(1))) <= TOL_F32


@pytest.mark.parametrize("m", [1, 16])
def test_c1_shape_with_rank32(gpu, oracle, m):
    # configs[0]: single INT3 linear 4096x14336, g64, rank-32 compensator
    import torch
    k, n = 4096, 14336
    P, _ = random_quantized(oracle, k, n, seed=7)
    comp = random_comp(oracle, k, n, 32, seed=8)
    A = np.random.default_rng(9).normal(0, 1, (m, k)).astype(np.float32)
    want = oracle.gemm_w3a16(A, P, comp, _oc(1))
    got = gpu.gemm_w3a16(torch.from_numpy(A).cuda(), gpu.Weight(P), gpu.Comp(comp),
                         _cfg(gpu, 1)).cpu().numpy()
    assert rel_err(got, want) <= TOL_F32


# ---------------------------------------------------------------------------
# tcgen05 prefill path (m >= 64 tokens): same contract as the decode path
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("k,n,m", [(128, 128, 64), (512, 1024, 200), (640, 256, 130), (1024, 384, 512)])
@pytest.mark.parametrize("mode", [1, 0])
def test_prefill_gemm_matches_oracle(gpu, oracle, k, n, m, mode):
    import torch
    P, _ = random_quantized(oracle, k, n, seed=k + n + m + mode, mode=mode)
    A = np.random.default_rng(m).normal(0, 1, (m, k)).astype(np.float32)
    want = oracle.gemm_w3a16(A, P, cfg=_oc(mode))
    W = gpu.Weight(P)
    got = gpu.gemm_w3a16(torch.from_numpy(A).cuda(), W, cfg=_cfg(gpu, mode)).cpu().numpy()
    assert rel_err(got, want) <= TOL_F32
    got16 = gpu.gemm_w3a16(torch.from_numpy(A).cuda().half(), W, cfg=_cfg(gpu, mode),
                           out_dtype=torch.float16).float().cpu().numpy()
    assert rel_err(got16, want) <= TOL_F16


@pytest.mark.parametrize("storage", [1, 0])
@pytest.mark.parametrize("rank", [4, 32, 70])
def test_prefill_gemm_with_compensator(gpu, oracle, storage, rank):
    import torch
    k, n, m = 512, 256, 150
    P, _ = random_quantized(oracle, k, n, seed=41)
    comp = random_comp(oracle, k, n, rank, seed=rank + 1, storage=storage)
    A = np.random.default_rng(42).normal(0, 1, (m, k)).astype(np.float32)
    want = oracle.gemm_w3a16(A, P, comp, _oc(1))
    got = gpu.gemm_w3a16(torch.from_numpy(A).cuda(), gpu.Weight(P), gpu.Comp(comp),
                         cfg=_cfg(gpu, 1)).cpu().numpy()
    assert rel_err(got, want) <= TOL_F32


def test_prefill_identity_reproduces_weights(gpu, oracle):
    # test_gemm.cpp:55-79 on the tensor-core path: A = I (128 rows) -> C == dequant exactly
    import torch
    k = n = 128
    codes = np.random.default_rng(9).integers(0, 8, (k, n), dtype=np.uint8)
    P = oracle.pack_matrix(codes, np.full(k * n // 64, 0.25, np.float32), np.full(k * n // 64, 4.0, np.float32))
    C = gpu.gemm_w3a16(torch.eye(k, device="cuda"), gpu.Weight(P), cfg=_cfg(gpu, 1)).cpu().numpy()
    want = np.array([oracle.half_to_float(int(h)) for h in oracle.dequant_half(P).ravel()],
                    np.float32).reshape(k, n)
    assert (C == want).all()


@pytest.mark.gpu
@pytest.mark.parametrize("m", [4, 96])
def test_out_buffer_defines_output_dtype(gpu, m):
    """A caller-provided output buffer fixes the output type (decode and prefill paths)."""
    import torch
    rng = np.random.default_rng(m)
    from paper_2504_02658_b200.synth import packed_random_words
    W = gpu.Weight(packed_random_words(256, 512, rng))
    A = torch.from_numpy(rng.normal(0, 1, (m, 256)).astype(np.float32)).cuda()
    ref = gpu.gemm_w3a16(A, W)
    out16 = torch.full((m, 512), float("nan"), dtype=torch.float16, device="cuda")
    got = gpu.gemm_w3a16(A, W, out=out16)
    assert got is out16 and torch.isfinite(out16).all()
    assert torch.allclose(out16.float(), ref, rtol=2e-3, atol=2e-3)
    with pytest.raises(gpu.ArgumentError):
        gpu.gemm_w3a16(A, W, out=out16, out_dtype=torch.float32)


@pytest.mark.gpu
def test_empty_batch(gpu, oracle):
    """m = 0: pad_batch keeps 0 rows (gemm.cpp:49-60), so C is 0 x n; shape errors
    still come first (gemm.cpp:131-139)."""
    import torch
    k, n = 128, 256
    P, _ = random_quantized(oracle, k, n, seed=71)
    W = gpu.Weight(P)
    got = gpu.gemm_w3a16(torch.empty((0, k), device="cuda"), W, cfg=_cfg(gpu, 1))
    assert tuple(got.shape) == (0, n)
    assert gpu.gemm_w3a16_host(np.empty((0, k), np.float32), W, cfg=_cfg(gpu, 1)).shape == (0, n)
    with pytest.raises(gpu.ShapeError):
        gpu.gemm_w3a16_host(np.empty((0, k + 64), np.float32), W, cfg=_cfg(gpu, 1))
