#!/usr/bin/env python3
"""C4: the Mixtral-8x7B 32-layer MoE stack at prefill 2048 tokens,
1 GPU or expert-parallel over N GPUs (torchrun, one rank per GPU, weak scaling: 2048
tokens per rank).  Every layer has its own device copy of the INT3+LoRC weights (the host
packing of one synthetic layer is reused, so 32 x 617 MB of distinct device weights stream
from HBM every step); layer l's output (plus the residual, RMS-normalised) feeds layer l+1.

    python tools/bench_stack.py [--layers 32] [--tokens 2048] [--steps 3] [--warmup 1]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/bench_stack.py

Prints one JSON line (rank 0): ms per step (max over ranks, CUDA events), tokens/s, TFLOP/s.
"""
import argparse, json, os, sys
import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_02658_b200 as mb  # noqa: E402
from paper_2504_02658_b200.synth import CONFIGS, build_host_layer, layer_traffic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--tokens", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()
    ws, rank = int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec = CONFIGS["mixtral"]
    routed_h, shared_h = build_host_layer(spec, seed=0)

    def dev(h):
        return mb.Expert(*(mb.Weight(P) for P in h.w), *((mb.Comp(c) if c is not None else None) for c in h.c))

    layers = []
    per = (spec.experts + ws - 1) // ws
    for _ in range(args.layers):
        if ws > 1:
            from paper_2504_02658_b200.ep import MiloEPLayer
            layers.append(MiloEPLayer([dev(h) for h in routed_h[rank * per:(rank + 1) * per]], [],
                                      spec.experts, spec.top_k, spec.score_mode))
        else:
            layers.append(mb.MoELayer([dev(h) for h in routed_h], [], top_k=spec.top_k,
                                      score_mode=spec.score_mode))
    g = torch.Generator(device="cuda").manual_seed(1000 + rank)
    m = args.tokens
    x0 = torch.randn(m, spec.d, device="cuda", generator=g).half()
    logits = [torch.randn(m, spec.experts, device="cuda", generator=g) for _ in range(args.layers)]
    w_norm = torch.ones(spec.d, device="cuda", dtype=torch.float32)
    ids_seen = []

    def step(record=False):
        x = x0
        for l, layer in enumerate(layers):
            y, ids, _ = layer.forward(x, logits[l], out_dtype=torch.float32, return_routing=True)
            if record:
                ids_seen.append(ids)
            x = torch.nn.functional.rms_norm(x.float() + y, (spec.d,), w_norm).half()
        return x

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i, (s, e) in enumerate(evs):
        s.record()
        out = step(record=(i == 0))
        e.record()
    torch.cuda.synchronize()
    ms = float(np.mean([s.elapsed_time(e) for s, e in evs]))
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    flops = 0.0
    for ids in ids_seen:  # this rank's tokens, all experts (EP: executed across ranks)
        flops += layer_traffic(spec, routed_h, shared_h, ids.cpu().numpy())["total_flops"]
    if ws > 1:
        t = torch.tensor([flops], device="cuda", dtype=torch.float64)
        dist.all_reduce(t)
        flops = float(t.item())
    if rank == 0:
        print(json.dumps({
            "metric": "Mixtral-8x7B 32-layer INT3+LoRC MoE stack, prefill (C4)", "value": round(ms, 3),
            "unit": "ms per step", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "tokens_per_s": round(m * ws / (ms * 1e-3), 1), "tflops": round(flops / (ms * 1e-3) / 1e12, 1),
            "finite": bool(torch.isfinite(out).all().item()),
            "config": {"workload": "mixtral-8x7b-moe-stack", "layers": args.layers, "tokens_per_rank": m,
                       "parallelism": f"ep{ws}" if ws > 1 else "single GPU", "scaling": "weak",
                       "data": "synthetic (one packed layer replicated into distinct device copies)"}}), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
