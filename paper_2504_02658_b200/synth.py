"""Synthetic MoE layers of the benchmark configurations (BASELINE.json).

Random-init packed INT3 weights (every 96-bit group is a valid packed group,
pack.cpp:56-68, so random words give uniformly random codes), binary16
scales/zero-points with the reference generators' statistics
(pipeline.cpp:408-426), and symm-int3 compensators with ragged per-expert
ranks.  Shapes: public Mixtral-8x7B / DeepSeek-MoE-16B / Arctic configs in
the reference's k x n orientation (synth.cpp:37-39), SURVEY.md section 8.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import ASYMMETRIC, Compensator, PackedInt3Matrix
from .pack import float_to_half_bits, random_compensator


@dataclass
class ConfigSpec:
    name: str
    d: int
    f: int
    experts: int
    top_k: int
    score_mode: int
    shared: int = 0
    f_shared: int = 0
    rank_shared: int = 0
    routed_ranks: tuple = (16,)
    plan: Optional[str] = None  # frozen rank plan (plans/<plan>.plan.json), else routed_ranks / rank_shared


# Ranks: frozen plans made by the reference's own plan_ranks (tools/make_rank_plans.py:
# Kurtosis-16 over the reference's synthetic StudentTMix experts; DeepSeek adds
# Dense-512 for the shared experts) -- adaptive, ragged per matrix (0 .. 54 for Mixtral).
CONFIGS = {
    # configs[1]: Mixtral-8x7B MoE layer, 8 experts top-2
    "mixtral": ConfigSpec("mixtral-8x7b-layer", 4096, 14336, 8, 2, 0,
                          routed_ranks=(16, 32, 8, 24, 16, 0, 32, 16), plan="mixtral"),
    # configs[2]: DeepSeek-MoE-16B layer, 64 routed (f=1408) top-6 + 2 shared
    "deepseek": ConfigSpec("deepseek-moe-16b-layer", 2048, 1408, 64, 6, 1, shared=2,
                           f_shared=1408, rank_shared=512, routed_ranks=(16, 0, 32, 8, 16, 24), plan="deepseek"),
    # configs[4]: Arctic-480B-shaped layer, 128 experts top-2
    "arctic": ConfigSpec("arctic-480b-layer", 7168, 4864, 128, 2, 0, routed_ranks=(16, 8, 32, 16),
                         plan="arctic"),
}

PLAN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "plans")


def load_rank_plan(spec: ConfigSpec):
    """The config's frozen plan (policy, {matrix name: rank}) or None."""
    if spec.plan is None:
        return None
    from .artifacts import load_plan
    return load_plan(os.path.join(PLAN_DIR, spec.plan + ".plan.json"))


def packed_random_words(rows: int, cols: int, rng: np.random.Generator,
                        mode: int = ASYMMETRIC) -> PackedInt3Matrix:
    groups = rows * cols // 32
    words = rng.integers(0, 2 ** 32, groups * 3, dtype=np.uint64).astype(np.uint32)
    ng = rows * cols // 64
    scales = (np.abs(rng.normal(0.0, 0.05, ng)) + 0.01).astype(np.float32)
    zeros = (3.5 + rng.normal(0.0, 1.0, ng)).astype(np.float32) if mode == ASYMMETRIC else None
    return PackedInt3Matrix(rows, cols, 0, False, mode, 64, words, None, None,
                            float_to_half_bits(scales),
                            None if zeros is None else float_to_half_bits(zeros))


@dataclass
class HostExpert:
    w: List[PackedInt3Matrix]              # w1 (d x f), w3 (d x f), w2 (f x d)
    c: List[Optional[Compensator]]
    ranks: List[int] = field(default_factory=list)


def expert_ranks(spec: ConfigSpec, e: int, plan=None) -> List[int]:
    """Ranks of w1, w3, w2 of routed expert e (plan names: synth.cpp:32-48)."""
    if plan is not None:
        return [plan.ranks[f"layer0.expert{e}.{w}"] for w in ("w1", "w3", "w2")]
    r = spec.routed_ranks
    return [r[(3 * e + j) % len(r)] for j in range(3)]


def build_host_layer(spec: ConfigSpec, seed: int = 0):
    """Host-side packed experts (routed, shared) for a config."""
    rng = np.random.default_rng(seed)
    plan = load_rank_plan(spec)
    routed, shared = [], []
    for e in range(spec.experts):
        ranks = expert_ranks(spec, e, plan)
        dims = [(spec.d, spec.f), (spec.d, spec.f), (spec.f, spec.d)]
        routed.append(HostExpert([packed_random_words(k, n, rng) for k, n in dims],
                                 [random_compensator(k, n, r, rng) for (k, n), r in zip(dims, ranks)],
                                 ranks))
    for s in range(spec.shared):
        dims = [(spec.d, spec.f_shared), (spec.d, spec.f_shared), (spec.f_shared, spec.d)]
        ranks = ([plan.ranks[f"layer0.shared_expert{s}.{w}"] for w in ("w1", "w3", "w2")] if plan is not None
                 else [spec.rank_shared] * 3)
        shared.append(HostExpert([packed_random_words(k, n, rng) for k, n in dims],
                                 [random_compensator(k, n, r, rng) for (k, n), r in zip(dims, ranks)],
                                 ranks))
    return routed, shared


def matrix_memory_bytes(rows: int, cols: int, rank: int, bits: int = 3, group_size: int = 64,
                        comp_bits: int = 3) -> int:
    """The reference's accounting (tensor_store.cpp:247-266)."""
    n = rows * cols
    comp_groups = 0 if rank == 0 else (rows + cols) * ((rank + group_size - 1) // group_size)
    return (n * bits // 8 + 2 * (n // group_size) * 2 + (rows + cols) * rank * comp_bits // 8
            + comp_groups * 2)


def layer_traffic(spec: ConfigSpec, routed: List[HostExpert], shared: List[HostExpert],
                  ids: np.ndarray):
    """Algorithmic bytes and flops of one layer call for a given routing
    (SURVEY.md section 8d): weights of every touched expert counted once
    (matrix_memory_bytes), fp16 activations in and out of every matrix
    invocation, flops 2 m_e k n + 2 m_e r (k + n) per matrix.
    Returns dict(total_bytes, total_flops, phase1_bytes, phase1_flops, ...)."""
    m = ids.shape[0]
    counts = np.bincount(ids[ids >= 0].ravel(), minlength=spec.experts)
    out = dict(phase1_bytes=0, phase2_bytes=0, phase1_flops=0, phase2_flops=0)
    entries = [(routed[e], int(counts[e])) for e in range(spec.experts) if counts[e] > 0]
    entries += [(s, m) for s in shared]
    for ex, me in entries:
        for j, P in enumerate(ex.w):
            k, n, r = P.rows, P.cols, ex.ranks[j]
            b = matrix_memory_bytes(k, n, r) + 2 * me * k + 2 * me * n
            fl = 2 * me * k * n + 2 * me * r * (k + n)
            key = "phase1" if j < 2 else "phase2"
            out[key + "_bytes"] += b
            out[key + "_flops"] += fl
    out["total_bytes"] = out["phase1_bytes"] + out["phase2_bytes"]
    out["total_flops"] = out["phase1_flops"] + out["phase2_flops"]
    out["touched_experts"] = len(entries)
    return out
