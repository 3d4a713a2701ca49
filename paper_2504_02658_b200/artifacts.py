"""Serving a MoE layer from the reference's offline artifacts (SURVEY.md section 8f
row 3): the model manifest, the rank plan and the per-matrix files `quantize` /
`pack` write go straight onto the device.

Reference formats read here:
  * manifest.json   -- tensor_store.cpp:172-193 (layers[].matrices[] with name, rows,
                       cols, structure_tag, expert_index), validated like
                       ModelManifest::validate (tensor_store.cpp:36-50);
  * plan.json       -- pipeline.cpp:179-192 (policy, ranks{name: r}, avg_sparse_rank,
                       memory_bytes), with load_plan's error categories;
  * artifacts       -- pipeline.cpp:318-320: <dir>/<name>.q.milo (packed-i3, linear) and,
                       for r > 0, <dir>/<name>.u.milo / .v.milo (compensator factors);
                       `pack` (pipeline.cpp:375-400) writes <out>/packed/<name>.packed.milo.

Expert matrices follow the reference's naming (synth.cpp:32-48):
layer<l>.expert<x>.w1 | .w3 (d x f) and .w2 (f x d); shared experts (structure tag
"shared_expert") are grouped by the name prefix before .w1/.w2/.w3.  Every expert's
compensator rank must equal the plan's rank for that matrix (a PlanError otherwise,
as quantize raises for a matrix the plan lacks, pipeline.cpp:315-317).
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass
from typing import Dict, List, Optional

from . import (Comp, ConfigError, Expert, FormatError, IoError, MoELayer, PlanError, ShapeError,
               Weight)

STRUCTURE_TAGS = ("attention", "shared_expert", "dense_ffn", "expert")


@dataclass
class MatrixEntry:
    name: str
    rows: int
    cols: int
    structure_tag: str
    expert_index: Optional[int] = None


@dataclass
class RankPlan:
    policy: str
    ranks: Dict[str, int]
    avg_sparse_rank: float = 0.0
    memory_bytes: int = 0


def _read_json(path: str, missing_exc, what: str):
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise missing_exc(f"cannot open {what} '{path}'") from None
    try:
        return json.loads(text)
    except ValueError:
        raise FormatError(f"{what} '{path}' is not valid JSON") from None


def load_manifest(path: str) -> Dict[int, List[MatrixEntry]]:
    """layer_index -> matrices (tensor_store.cpp:172-193 + validate 36-50)."""
    j = _read_json(path, IoError, "manifest")
    layers: Dict[int, List[MatrixEntry]] = {}
    names = set()
    try:
        for jl in j["layers"]:
            mats = []
            for jm in jl["matrices"]:
                tag = jm["structure_tag"]
                if tag not in STRUCTURE_TAGS:
                    raise FormatError(f"unknown structure_tag '{tag}'")
                e = MatrixEntry(jm["name"], int(jm["rows"]), int(jm["cols"]), tag,
                                int(jm["expert_index"]) if "expert_index" in jm else None)
                if e.name in names:
                    raise FormatError(f"duplicate matrix name '{e.name}' in manifest")
                names.add(e.name)
                if (tag == "expert") != (e.expert_index is not None):
                    raise FormatError(f"matrix '{e.name}': expert_index must be present exactly for expert tag")
                if e.rows == 0 or e.cols == 0:
                    raise FormatError(f"matrix '{e.name}': zero dimension")
                mats.append(e)
            layers[int(jl["layer_index"])] = mats
    except (KeyError, TypeError) as exc:
        raise FormatError(f"manifest '{path}': missing or mistyped field {exc}") from None
    return layers


def load_plan(path: str) -> RankPlan:
    """pipeline.cpp:179-192: a missing file is a ConfigError, bad JSON a FormatError."""
    j = _read_json(path, ConfigError, "plan file")
    try:
        ranks = {str(k): int(v) for k, v in j["ranks"].items()}
        if any(r < 0 for r in ranks.values()):
            raise FormatError(f"plan file '{path}': negative rank")
        return RankPlan(str(j["policy"]), ranks, float(j.get("avg_sparse_rank", 0.0)),
                        int(j.get("memory_bytes", 0)))
    except (KeyError, TypeError, AttributeError, ValueError) as exc:
        raise FormatError(f"plan file '{path}': missing or mistyped field {exc}") from None


def _weight_path(name: str, artifact_dir: str, packed_dir: Optional[str]) -> str:
    if packed_dir is not None:
        p = os.path.join(packed_dir, name + ".packed.milo")
        if os.path.exists(p):
            return p
    p = os.path.join(artifact_dir, name + ".q.milo")
    if not os.path.exists(p):
        raise ConfigError(f"missing quantized artifact '{p}'")  # like run_pack, pipeline.cpp:379
    return p


def _load_matrix(e: MatrixEntry, artifact_dir: str, packed_dir: Optional[str], plan: Optional[RankPlan]):
    W = Weight.load(_weight_path(e.name, artifact_dir, packed_dir))
    if (W.rows, W.cols) != (e.rows, e.cols):
        raise ShapeError(f"artifact '{e.name}' is {W.rows} x {W.cols}, manifest says {e.rows} x {e.cols}")
    u = os.path.join(artifact_dir, e.name + ".u.milo")
    v = os.path.join(artifact_dir, e.name + ".v.milo")
    if plan is not None:
        if e.name not in plan.ranks:
            raise PlanError(f"plan has no rank for matrix '{e.name}'")
        r = plan.ranks[e.name]
        if r == 0:
            return W, None
        if not (os.path.exists(u) and os.path.exists(v)):
            raise ConfigError(f"plan rank {r} for '{e.name}' but no compensator files")
        C = Comp.load(u, v)
        if C.rank != r:
            raise PlanError(f"compensator of '{e.name}' has rank {C.rank}, the plan says {r}")
        return W, C
    if os.path.exists(u) and os.path.exists(v):
        return W, Comp.load(u, v)
    return W, None


def _triplet(group: Dict[str, MatrixEntry], what: str, artifact_dir, packed_dir, plan) -> Expert:
    missing = [p for p in ("w1", "w2", "w3") if p not in group]
    if missing:
        raise FormatError(f"{what}: missing matrices {missing}")
    (w1, c1), (w2, c2), (w3, c3) = (_load_matrix(group[p], artifact_dir, packed_dir, plan)
                                    for p in ("w1", "w2", "w3"))
    if not (w1.rows == w3.rows == w2.cols and w1.cols == w3.cols == w2.rows):
        raise ShapeError(f"{what}: w1/w3 must be d x f and w2 f x d")
    return Expert(w1=w1, w3=w3, w2=w2, c1=c1, c3=c3, c2=c2)


def load_moe_layer(manifest, layer_index: int, artifact_dir: str, plan=None,
                   packed_dir: Optional[str] = None, top_k: int = 2, score_mode: int = 0) -> MoELayer:
    """The routed (tag "expert", ordered by expert_index) and shared experts of one
    manifest layer as a device MoELayer.  `manifest` / `plan`: paths or the parsed
    objects; `packed_dir`: the output of `milo pack` (preferred when present)."""
    layers = load_manifest(manifest) if isinstance(manifest, str) else manifest
    plan = load_plan(plan) if isinstance(plan, str) else plan
    if layer_index not in layers:
        raise ConfigError(f"manifest has no layer {layer_index}")
    routed: Dict[int, Dict[str, MatrixEntry]] = {}
    shared: Dict[str, Dict[str, MatrixEntry]] = {}
    for e in layers[layer_index]:
        prefix, _, proj = e.name.rpartition(".")
        if e.structure_tag == "expert" and proj in ("w1", "w2", "w3"):
            routed.setdefault(e.expert_index, {})[proj] = e
        elif e.structure_tag == "shared_expert" and proj in ("w1", "w2", "w3"):
            shared.setdefault(prefix, {})[proj] = e
    if not routed and not shared:
        raise ConfigError(f"layer {layer_index} has no expert matrices")
    idx = sorted(routed)
    if idx != list(range(len(idx))):
        raise FormatError(f"layer {layer_index}: expert indices {idx} are not 0..E-1")
    experts = [_triplet(routed[x], f"layer {layer_index} expert {x}", artifact_dir, packed_dir, plan) for x in idx]
    shared_ex = [_triplet(shared[p], p, artifact_dir, packed_dir, plan) for p in sorted(shared)]
    return MoELayer(experts, shared_ex, top_k=top_k, score_mode=score_mode)
