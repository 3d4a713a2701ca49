"""Expert-parallel dispatch / combine (paper_2504_02658_b200/ep.py) on CPU with
gloo, world size 2: the EP layer must equal the single-process layer.  The
experts here are plain fp32 reference FFNs (test infrastructure); on GPUs the
same class binds the MiLo kernels (tests/test_gpu_moe.py covers those)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

E, K, D, F = 6, 2, 32, 48


def _experts(seed=0):
    g = torch.Generator().manual_seed(seed)
    return [(torch.randn(D, F, generator=g) * 0.1, torch.randn(D, F, generator=g) * 0.1,
             torch.randn(F, D, generator=g) * 0.1) for _ in range(E)]


def _ffn(w, x):
    w1, w3, w2 = w
    return (torch.nn.functional.silu(x @ w1) * (x @ w3)) @ w2


def _route(logits):
    v, i = torch.topk(logits, K, dim=-1)  # distinct logits in the test: no ties
    return i.to(torch.int32), torch.softmax(v, dim=-1)


def _reference(x, logits, experts, shared):
    ids, w = _route(logits)
    out = torch.zeros(x.shape[0], D)
    for t in range(x.shape[0]):
        for k in range(K):
            out[t] += w[t, k] * _ffn(experts[ids[t, k]], x[t:t + 1].half().float())[0]
    return out + _ffn(shared, x)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_02658_b200.ep import ExpertParallelMoE
    experts = _experts()
    shared = _experts(7)[0]
    per = (E + world - 1) // world
    own = experts[rank * per:(rank + 1) * per]

    def local_fn(rows, local_ids):  # rows with id -1 are padding (fixed-capacity exchange)
        rows = rows.float()
        return torch.stack([_ffn(own[int(e)], rows[i:i + 1])[0] if int(e) >= 0 else torch.zeros(D)
                            for i, e in enumerate(local_ids)]) if rows.shape[0] else torch.zeros(0, D)

    layer = ExpertParallelMoE(E, K, D, local_fn, shared_fn=lambda x: _ffn(shared, x), router_fn=_route)
    layer.capacity = 8 * K  # ragged m per rank: the fixed exchange uses the largest m K
    g = torch.Generator().manual_seed(100 + rank)
    m = 5 + 3 * rank  # ragged token counts per rank
    x = torch.randn(m, D, generator=g)
    logits = torch.randn(m, E, generator=g)
    logits[:, 0] += 2.0 * rank  # skew: rank 1 sends most tokens to rank 0's expert 0
    out = layer.forward(x, logits)
    ref = _reference(x, logits, experts, shared)
    err = float((out - ref).norm() / ref.norm())
    # routed-entry point with explicit ids (including an unused -1 slot)
    ids, w = _route(logits)
    ids[0, 1] = -1
    out2 = layer.forward(x, ids=ids, weights=w)
    # the exact all-to-all-v path (prefill-sized batches) agrees with the fixed-capacity one
    layer.fixed_cap_max = 0
    out3 = layer.forward(x, logits)
    q.put((rank, err, max(float((out2[1:] - out[1:]).abs().max()), float((out3 - out).abs().max()))))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(120)
def test_expert_parallel_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in range(2)]
    for p in procs:
        p.join(30)
    for rank, err, drift in res:
        assert err < 1e-5, (rank, err)
        assert drift < 1e-5, (rank, drift)
