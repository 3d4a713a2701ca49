"""GPU parity of the top-k routed grouped-expert layer against the CPU oracle.

The reference has no MoE layer; its semantics are
defined in oracle/milo_oracle.h (or_router_topk / or_moe_forward) as a
composition of per-expert gemm_w3a16 calls, and pinned against the same
composition over the compiled reference (tests/test_oracle_golden.py).
Tolerances: routing indices bit-exact; routing weights 1e-6 relative;
layer output 1e-4 relative Frobenius (fp32 out) — the intermediate h is
rounded to binary16 on both sides (gemm.cpp:144-146), so a 1e-6 difference
in fp32 can flip a rare h element by one binary16 ulp.
"""
import numpy as np
import pytest

from tests.helpers import rel_err

pytestmark = pytest.mark.gpu

TOL_MOE = 1e-4


def _experts(oracle, gpu, E, d, f, ranks, seed, mode=1, storage=None):
    from tests.helpers import random_comp, random_quantized
    o_ex, g_ex = [], []
    for e in range(E):
        ws, cs, gw, gc = [], [], [], []
        for j, (k, n) in enumerate([(d, f), (d, f), (f, d)]):
            P, _ = random_quantized(oracle, k, n, seed=seed + 31 * e + j, mode=mode)
            r = ranks[e][j]
            st = 1 if storage is None else storage[e][j]
            c = random_comp(oracle, k, n, r, seed=seed + 977 * e + j, storage=st) if r else None
            ws.append(P)
            cs.append(c)
            gw.append(gpu.Weight(P))
            gc.append(gpu.Comp(c) if c is not None else None)
        o_ex.append({"w": ws, "c": cs})
        g_ex.append(gpu.Expert(gw[0], gw[1], gw[2], gc[0], gc[1], gc[2]))
    return o_ex, g_ex


@pytest.mark.parametrize("m", [1, 3, 8, 16, 33, 64, 100, 300])
def test_mixtral_like_layer(gpu, oracle, m):
    import torch
    E, K, d, f = 8, 2, 256, 512
    ranks = [[(8 * ((e + j) % 4)) for j in range(3)] for e in range(E)]  # ragged, incl. 0
    o_ex, g_ex = _experts(oracle, gpu, E, d, f, ranks, seed=100)
    rng = np.random.default_rng(m)
    x = rng.normal(0, 1, (m, d)).astype(np.float32)
    logits = rng.normal(0, 1, (m, E)).astype(np.float32)
    ids, w = oracle.router_topk(logits, K, 0)
    want = oracle.moe_forward(o_ex, [], x, ids, w)
    layer = gpu.MoELayer(g_ex, [], top_k=K, score_mode=0)
    out, gids, gw = layer.forward(torch.from_numpy(x).cuda(), torch.from_numpy(logits).cuda(),
                                  return_routing=True)
    assert (gids.cpu().numpy() == ids).all()
    assert np.allclose(gw.cpu().numpy(), w, rtol=1e-6, atol=1e-7)
    assert rel_err(out.cpu().numpy(), want) <= TOL_MOE
    # routed entry point with the oracle's routing, fp16 in / fp16 out
    out16 = layer.forward_routed(torch.from_numpy(x).cuda().half(), torch.from_numpy(ids).cuda(),
                                 torch.from_numpy(w).cuda(), out_dtype=torch.float16)
    assert rel_err(out16.float().cpu().numpy(), want) <= 1e-3


@pytest.mark.parametrize("m", [1, 7, 40, 150])
def test_deepseek_like_layer_with_shared_experts(gpu, oracle, m):
    import torch
    E, K, d, f = 16, 6, 256, 128
    ranks = [[(0, 8, 16)[(e + j) % 3] for j in range(3)] for e in range(E)]
    o_ex, g_ex = _experts(oracle, gpu, E, d, f, ranks, seed=300)
    o_sh, g_sh = _experts(oracle, gpu, 2, d, f, [[64, 64, 64], [32, 0, 96]], seed=900)
    rng = np.random.default_rng(10 + m)
    x = rng.normal(0, 1, (m, d)).astype(np.float32)
    logits = rng.normal(0, 1, (m, E)).astype(np.float32)
    ids, w = oracle.router_topk(logits, K, 1)
    want = oracle.moe_forward(o_ex, o_sh, x, ids, w)
    layer = gpu.MoELayer(g_ex, g_sh, top_k=K, score_mode=1)
    out = layer.forward(torch.from_numpy(x).cuda(), torch.from_numpy(logits).cuda())
    assert rel_err(out.cpu().numpy(), want) <= TOL_MOE


def test_skewed_routing_and_host_entry(gpu, oracle):
    import torch
    E, K, d, f = 4, 2, 128, 256
    o_ex, g_ex = _experts(oracle, gpu, E, d, f, [[16, 16, 16]] * E, seed=500)
    m = 50
    rng = np.random.default_rng(1)
    x = rng.normal(0, 1, (m, d)).astype(np.float32)
    logits = rng.normal(0, 1, (m, E)).astype(np.float32)
    logits[:, 2] += 5.0  # every token picks expert 2 -> one expert with 50 rows
    ids, w = oracle.router_topk(logits, K, 0)
    want = oracle.moe_forward(o_ex, [], x, ids, w)
    layer = gpu.MoELayer(g_ex, [], top_k=K)
    got = layer.forward_host(x, logits)
    assert rel_err(got, want) <= TOL_MOE
    # determinism: same inputs -> same bits
    a = layer.forward(torch.from_numpy(x).cuda(), torch.from_numpy(logits).cuda())
    b = layer.forward(torch.from_numpy(x).cuda(), torch.from_numpy(logits).cuda())
    assert torch.equal(a, b)


@pytest.mark.parametrize("m", [1, 16, 600])
def test_host_entry_matches_device_call(gpu, oracle, m):
    """milo_moe_forward_host: the host-buffer entry point must equal the
    device-buffer call.  Decode batches run the h-local kernel, whose output is
    accumulated with fp32 reductions in arrival order, so two calls agree to
    fp32 reassociation (<= 1e-6 relative); the other paths bit for bit."""
    import torch
    E, K, d, f = 4, 2, 128, 256
    o_ex, g_ex = _experts(oracle, gpu, E, d, f, [[16, 8, 0]] * E, seed=510)
    rng = np.random.default_rng(20 + m)
    x = rng.normal(0, 1, (m, d)).astype(np.float32)
    logits = rng.normal(0, 1, (m, E)).astype(np.float32)
    layer = gpu.MoELayer(g_ex, [], top_k=K)
    host = layer.forward_host(x, logits)
    host2 = layer.forward_host(x, logits)  # the stage is reused across calls
    dev = layer.forward(torch.from_numpy(x).cuda(), torch.from_numpy(logits).cuda()).cpu().numpy()
    if m <= 16:
        assert rel_err(host, dev) <= 1e-6 and rel_err(host2, dev) <= 1e-6
    else:
        assert np.array_equal(host, dev) and np.array_equal(host2, dev)
    ids, w = oracle.router_topk(logits, K, 0)
    assert rel_err(host, oracle.moe_forward(o_ex, [], x, ids, w)) <= TOL_MOE


def test_router_ties_prefer_lower_expert(gpu):
    import torch
    logits = torch.tensor([[1.0, 3.0, 3.0, 0.5], [2.0, 2.0, 2.0, 2.0]], device="cuda")
    ids, w = gpu.router_topk(logits, 2)
    assert ids.cpu().tolist() == [[1, 2], [0, 1]]
    assert torch.allclose(w, torch.full_like(w, 0.5))


def test_expert_parallel_layer_world1_matches_layer(gpu, oracle):
    """MiloEPLayer (NCCL all-to-all dispatch / combine) on a world of 1 equals
    the single-GPU layer; the 2-rank exchange logic is tests/test_ep.py (gloo)."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_2504_02658_b200.ep import MiloEPLayer
    E, K, d, f = 8, 2, 256, 512
    ranks = [[(8 * ((e + j) % 4)) for j in range(3)] for e in range(E)]
    o_ex, g_ex = _experts(oracle, gpu, E, d, f, ranks, seed=700)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        ep = MiloEPLayer(g_ex, [], E, K, 0)
        ref = gpu.MoELayer(g_ex, [], top_k=K)
        for m in (1, 9, 70):
            rng = np.random.default_rng(m)
            x = torch.from_numpy(rng.normal(0, 1, (m, d)).astype(np.float32)).cuda()
            lg = torch.from_numpy(rng.normal(0, 1, (m, E)).astype(np.float32)).cuda()
            a = ep.forward(x, lg)
            b = ref.forward(x, lg)
            assert rel_err(a.cpu().numpy(), b.cpu().numpy()) <= 1e-5
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("m", [20, 64])
def test_hot_expert_token_chunks(gpu, oracle, m):
    """Decode megakernel with m <= 64: an expert routed more than 16 tokens is split into
    16-row blocks (chunks), combined in k order like the oracle."""
    import torch
    E, K, d, f = 8, 2, 256, 512
    ranks = [[(8 * ((e + j) % 4)) for j in range(3)] for e in range(E)]
    o_ex, g_ex = _experts(oracle, gpu, E, d, f, ranks, seed=1300)
    rng = np.random.default_rng(7 + m)
    x = rng.normal(0, 1, (m, d)).astype(np.float32)
    logits = rng.normal(0, 1, (m, E)).astype(np.float32)
    logits[:, 3] += 10.0  # every token routes to expert 3 (m rows: several chunks)
    ids, w = oracle.router_topk(logits, K, 0)
    assert (ids[:, 0] == 3).all()
    want = oracle.moe_forward(o_ex, [], x, ids, w)
    layer = gpu.MoELayer(g_ex, [], top_k=K, score_mode=0)
    out, gids, _ = layer.forward(torch.from_numpy(x).cuda(), torch.from_numpy(logits).cuda(),
                                 return_routing=True)
    assert (gids.cpu().numpy() == ids).all()
    assert rel_err(out.cpu().numpy(), want) <= TOL_MOE


@pytest.mark.gpu
@pytest.mark.parametrize("world,m,K", [(4, 3, 2), (8, 5, 2), (2, 16, 6)])
def test_ep_dispatch_combine_kernels_multi_rank_layout(gpu, world, m, K):
    """The EP exchange kernels for world > 1 (the multi-GPU scaling path, which a
    1-GPU box cannot run end to end): every routed entry lands in its owner's
    capacity block in entry order with its local expert id, unused rows carry
    id -1 and zeros, and the combine sums the returned rows in k order."""
    import torch
    E, d = 4 * world, 64
    per = E // world
    C = m * K
    rng = np.random.default_rng(world * 100 + m)
    ids = np.stack([rng.choice(E, K, replace=False) for _ in range(m)]).astype(np.int32)
    ids[0, -1] = -1  # an unused routing slot
    x = rng.normal(0, 1, (m, d)).astype(np.float32)
    send, _, slot = gpu.ep_dispatch(torch.from_numpy(ids).cuda(), torch.from_numpy(x).cuda(), world, per, C,
                                    packed=True)
    send = send.cpu()
    slot = slot.cpu().numpy()
    rows = send[:, :d].float().numpy()
    lid = send[:, d:d + 2].contiguous().view(torch.int32).view(-1).numpy()
    used = np.zeros(world * C, bool)
    for dest in range(world):
        pos = 0
        for t in range(m):
            for k in range(K):
                e = ids[t, k]
                if e < 0 or e // per != dest:
                    continue
                r = dest * C + pos
                assert slot[t * K + k] == r
                assert lid[r] == e - dest * per
                assert np.array_equal(rows[r], x[t].astype(np.float16).astype(np.float32))
                used[r] = True
                pos += 1
    assert slot[0 * K + K - 1] == -1
    assert (lid[~used] == -1).all() and (rows[~used] == 0).all()
    # combine: y rows returned per slot, weighted in k order
    y = rng.normal(0, 1, (world * C, d)).astype(np.float32)
    w = rng.random((m, K)).astype(np.float32)
    out = gpu.ep_combine(torch.from_numpy(y).cuda(), torch.from_numpy(slot).cuda(),
                         torch.from_numpy(w).cuda()).cpu().numpy()
    want = np.zeros((m, d), np.float32)
    for t in range(m):
        for k in range(K):
            if slot[t * K + k] >= 0:
                want[t] += w[t, k] * y[slot[t * K + k]]
    assert np.allclose(out, want, rtol=1e-6, atol=1e-6)


@pytest.mark.gpu
@pytest.mark.parametrize("m", [1, 40, 130])
def test_arctic_like_layer_128_experts(gpu, oracle, m):
    """Arctic-480B-shaped routing (128 experts, top-2; reduced hidden sizes): decode
    megakernel (m <= 64) and tcgen05 prefill path (m = 130) against the oracle."""
    import torch
    E, K, d, f = 128, 2, 256, 256
    ranks = [[(0, 8, 16, 32)[(e + j) % 4] for j in range(3)] for e in range(E)]
    o_ex, g_ex = _experts(oracle, gpu, E, d, f, ranks, seed=2100)
    rng = np.random.default_rng(300 + m)
    x = rng.normal(0, 1, (m, d)).astype(np.float32)
    logits = rng.normal(0, 1, (m, E)).astype(np.float32)
    ids, w = oracle.router_topk(logits, K, 0)
    want = oracle.moe_forward(o_ex, [], x, ids, w)
    layer = gpu.MoELayer(g_ex, [], top_k=K, score_mode=0)
    out, gids, _ = layer.forward(torch.from_numpy(x).cuda(), torch.from_numpy(logits).cuda(),
                                 return_routing=True)
    assert (gids.cpu().numpy() == ids).all()
    assert rel_err(out.cpu().numpy(), want) <= TOL_MOE


def test_empty_token_batch(gpu, oracle):
    import torch
    E, K, d, f = 4, 2, 128, 256
    _, g_ex = _experts(oracle, gpu, E, d, f, [[16, 0, 8]] * E, seed=520)
    layer = gpu.MoELayer(g_ex, [], top_k=K)
    out = layer.forward(torch.empty((0, d), device="cuda"), torch.empty((0, E), device="cuda"))
    assert tuple(out.shape) == (0, d)
    assert layer.forward_host(np.empty((0, d), np.float32), np.empty((0, E), np.float32)).shape == (0, d)


@pytest.mark.parametrize("m", [12, 16, 48, 64])
def test_decode_path_beyond_64_blocks(gpu, oracle, m):
    """64 routed experts, top-6, 2 shared: 66 .. 92 (expert, chunk) blocks and up to
    384 routed entries in one decode launch (the DeepSeek-like shape;
    kDecMaxBlocks = 96, kDecMaxEntries = 384)."""
    import torch
    E, K, d, f = 64, 6, 128, 128
    ranks = [[(0, 8, 16)[(e + j) % 3] for j in range(3)] for e in range(E)]
    o_ex, g_ex = _experts(oracle, gpu, E, d, f, ranks, seed=1300)
    o_sh, g_sh = _experts(oracle, gpu, 2, d, f, [[64, 32, 64], [16, 0, 32]], seed=1900)
    rng = np.random.default_rng(40 + m)
    x = rng.normal(0, 1, (m, d)).astype(np.float32)
    logits = rng.normal(0, 1, (m, E)).astype(np.float32)
    for t in range(m):  # token t prefers experts 6t .. 6t + 5 (mod 64): all 64 touched
        logits[t, (np.arange(K) + K * t) % E] += 8.0
    ids, w = oracle.router_topk(logits, K, 1)
    assert len(np.unique(ids)) == E  # 64 routed blocks + 2 shared-expert blocks
    want = oracle.moe_forward(o_ex, o_sh, x, ids, w)
    layer = gpu.MoELayer(g_ex, g_sh, top_k=K, score_mode=1)
    l0 = gpu.launch_count()
    out = layer.forward(torch.from_numpy(x).cuda(), torch.from_numpy(logits).cuda())
    torch.cuda.synchronize()
    # one decode kernel (+ the f32 -> binary16 row rounding of x), not the multi-launch
    # legacy or prefill paths
    assert gpu.launch_count() - l0 <= 2
    assert rel_err(out.cpu().numpy(), want) <= TOL_MOE


def test_host_entry_shape_errors(gpu, oracle):
    """milo_moe_forward_host checks x's and the logits' column counts against the
    layer (d, E) before touching any buffer: ShapeError, as the reference's
    gemm_w3a16 throws for A.cols != k (gemm.cpp:135-136)."""
    E, K, d, f = 4, 2, 128, 256
    _, g_ex = _experts(oracle, gpu, E, d, f, [[0, 0, 0]] * E, seed=520)
    layer = gpu.MoELayer(g_ex, [], top_k=K)
    x = np.zeros((3, d), np.float32)
    lg = np.zeros((3, E), np.float32)
    with pytest.raises(gpu.ShapeError):
        layer.forward_host(np.zeros((3, d - 64), np.float32), lg)
    with pytest.raises(gpu.ShapeError):
        layer.forward_host(x, np.zeros((3, E - 1), np.float32))
    with pytest.raises(gpu.ShapeError):
        layer.forward_host(x, np.zeros((2, E), np.float32))
    assert layer.forward_host(x, lg).shape == (3, d)


@pytest.mark.parametrize("m,x16", [(1, False), (7, True), (40, False), (130, True)])
def test_router_gemm_bit_exact_and_forward_x(gpu, oracle, m, x16):
    """The MoE gate on the device (router_gemm_kernel) gives the oracle's logits
    bit for bit (same fixed fp32 order), so the routing ids of forward_x are
    the oracle's; the layer output matches the oracle's composition."""
    import torch
    E, K, d, f = 8, 2, 256, 512
    ranks = [[(8 * ((e + j) % 4)) for j in range(3)] for e in range(E)]
    o_ex, g_ex = _experts(oracle, gpu, E, d, f, ranks, seed=140)
    rng = np.random.default_rng(900 + m)
    x = rng.normal(0, 1, (m, d)).astype(np.float32)
    gate = rng.normal(0, 0.05, (E, d)).astype(np.float16)
    want_logits = oracle.router_gemm(x, gate.view(np.uint16))
    xt = torch.from_numpy(x).cuda()
    if x16:
        xt = xt.half()
    got_logits = gpu.router_gemm(xt, torch.from_numpy(gate).cuda()).cpu().numpy()
    assert np.array_equal(got_logits.view(np.uint32), want_logits.view(np.uint32))
    ids, w = oracle.router_topk(want_logits, K, 0)
    want = oracle.moe_forward(o_ex, [], x, ids, w)
    layer = gpu.MoELayer(g_ex, [], top_k=K, score_mode=0)
    with pytest.raises(gpu.ConfigError):
        layer.forward_x(xt)
    with pytest.raises(gpu.ShapeError):
        layer.set_gate(gate[:, :64])
    layer.set_gate(gate)
    out, gids, gw = layer.forward_x(xt, return_routing=True)
    assert np.array_equal(gids.cpu().numpy(), ids)
    assert rel_err(out.cpu().numpy(), want) <= 2.5e-4


@pytest.mark.parametrize("m", [96, 200])
def test_prefill_mixed_compensators(gpu, oracle, m):
    """The tcgen05 prefill path with every LoRC t variant in one layer: symm-INT3
    factors of one rank chunk (contiguous code runs), of several chunks with
    rank % 16 == 0 (16-byte code rows) and != 0 (byte loads), real-valued factors
    (the CUDA-core t kernel), and a rank-0 matrix; the shared expert's t on all
    tokens.  f = 256: k % 128 == 0 on both phases."""
    import torch
    E, K, d, f = 4, 2, 256, 256
    ranks = [[8, 70, 96], [32, 0, 64], [80, 16, 40], [128, 24, 4]]
    storage = [[1, 1, 1], [0, 1, 0], [1, 0, 1], [1, 1, 0]]
    o_ex, g_ex = _experts(oracle, gpu, E, d, f, ranks, 900, storage=storage)
    o_sh, g_sh = _experts(oracle, gpu, 1, d, f, [[96, 70, 8]], 1900, storage=[[1, 0, 1]])
    layer = gpu.MoELayer(g_ex, g_sh, top_k=K)
    rng = np.random.default_rng(m)
    x = rng.normal(0, 1, (m, d)).astype(np.float32)
    logits = rng.normal(0, 1, (m, E)).astype(np.float32)
    ids, w = oracle.router_topk(logits, K, 0)
    want = oracle.moe_forward(o_ex, o_sh, x, ids, w)
    got = layer.forward(torch.from_numpy(x).cuda(), torch.from_numpy(logits).cuda()).cpu().numpy()
    assert rel_err(got, want) <= TOL_MOE
