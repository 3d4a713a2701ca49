"""Serving from the reference's offline artifacts:
manifest.json / plan.json parsing with the reference's error categories
(tensor_store.cpp:36-50,172-193; pipeline.cpp:179-192) on the CPU, and (GPU) a MoE
layer assembled from quantize-style artifacts -- packed-i3 files written by the
reference's own save_packed, symm-i3 compensator factor files -- against the oracle."""
import json
import struct

import numpy as np
import pytest

from tests.helpers import rel_err


@pytest.fixture(scope="module")
def art():
    from paper_2504_02658_b200 import artifacts
    return artifacts


def _dump(path, obj):
    path.write_text(json.dumps(obj))
    return str(path)


def _manifest(d=128, f=256, E=2):
    mats = [{"name": "layer0.attn.q", "rows": d, "cols": d, "structure_tag": "attention"}]
    for x in range(E):
        for proj, k, n in (("w1", d, f), ("w3", d, f), ("w2", f, d)):
            mats.append({"name": f"layer0.expert{x}.{proj}", "rows": k, "cols": n,
                         "structure_tag": "expert", "expert_index": x})
    return {"layers": [{"layer_index": 0, "matrices": mats}]}


def test_manifest_and_plan_parsing(art, tmp_path):
    layers = art.load_manifest(_dump(tmp_path / "m.json", _manifest()))
    assert [e.name for e in layers[0]][:2] == ["layer0.attn.q", "layer0.expert0.w1"]
    assert layers[0][1].expert_index == 0 and layers[0][0].expert_index is None
    plan = art.load_plan(_dump(tmp_path / "p.json", {"policy": "Dense-8+Frequency-16",
                                                        "ranks": {"a": 8, "b": 0}, "memory_bytes": 7}))
    assert plan.ranks == {"a": 8, "b": 0} and plan.memory_bytes == 7 and plan.avg_sparse_rank == 0.0


def test_manifest_and_plan_error_categories(art, tmp_path):
    import paper_2504_02658_b200 as mb
    with pytest.raises(mb.ConfigError):  # load_plan: missing file (pipeline.cpp:180)
        art.load_plan(str(tmp_path / "none.json"))
    (tmp_path / "bad.json").write_text("{ranks:")
    with pytest.raises(mb.FormatError):
        art.load_plan(str(tmp_path / "bad.json"))
    with pytest.raises(mb.IoError):  # load_manifest: cannot open (tensor_store.cpp:174)
        art.load_manifest(str(tmp_path / "none.json"))
    m = _manifest()
    m["layers"][0]["matrices"].append(dict(m["layers"][0]["matrices"][1]))
    with pytest.raises(mb.FormatError):  # duplicate name
        art.load_manifest(_dump(tmp_path / "dup.json", m))
    m = _manifest()
    del m["layers"][0]["matrices"][1]["expert_index"]
    with pytest.raises(mb.FormatError):  # expert tag without expert_index
        art.load_manifest(_dump(tmp_path / "idx.json", m))
    m = _manifest()
    m["layers"][0]["matrices"][0]["structure_tag"] = "mlp"
    with pytest.raises(mb.FormatError):
        art.load_manifest(_dump(tmp_path / "tag.json", m))
    # a missing quantized artifact is a ConfigError (run_pack, pipeline.cpp:378-379)
    with pytest.raises(mb.ConfigError):
        art.load_moe_layer(_dump(tmp_path / "m.json", _manifest()), 0, str(tmp_path))


def _write_symm_i3(prefix, k, n, r, rng):
    """A compensator factor pair in the layout quantize writes (pipeline.cpp:258-282)."""
    gpr = (r + 63) // 64
    for rows, role, tr, suf in ((k, "compensator-U", False, ".u.milo"), (n, "compensator-V", True, ".v.milo")):
        codes = rng.integers(0, 8, (rows, r), dtype=np.uint8)
        sc = (np.abs(rng.normal(0, 0.05, (rows, gpr))) + 0.01).astype(np.float16)
        h = json.dumps(dict(name="x." + role[-1], rows=rows, cols=r, dtype="symm-i3", role=role, rank=r,
                            storage="symm-int3", group_size=64, transposed=tr)).encode()
        with open(prefix + suf, "wb") as fh:
            fh.write(b"MILO1" + struct.pack("<I", len(h)) + h + codes.tobytes() + sc.view(np.uint16).tobytes())


@pytest.mark.gpu
def test_layer_from_artifacts_matches_oracle(gpu, oracle, ref, art, tmp_path):
    import torch
    from tests.helpers import random_quantized
    from tests.test_containers import _oracle_comp
    E, K, d, f = 4, 2, 128, 256
    adir = tmp_path / "artifacts"
    adir.mkdir()
    rng = np.random.default_rng(77)
    ranks, o_ex = {"layer0.attn.q": 8}, []
    for x in range(E):
        ws, cs = [], []
        for j, (proj, k, n) in enumerate((("w1", d, f), ("w3", d, f), ("w2", f, d))):
            name = f"layer0.expert{x}.{proj}"
            P, _ = random_quantized(oracle, k, n, seed=700 + 31 * x + j, mode=1)
            ref.save_packed(P, name, str(adir / f"{name}.q.milo"))
            r = (0, 8, 16, 24)[(x + j) % 4]
            ranks[name] = r
            c = None
            if r:
                _write_symm_i3(str(adir / name), k, n, r, rng)
                c = _oracle_comp(str(adir / name))
            ws.append(P)
            cs.append(c)
        o_ex.append({"w": ws, "c": cs})
    mpath = _dump(tmp_path / "manifest.json", _manifest(d, f, E))
    ppath = _dump(tmp_path / "plan.json", {"policy": "Dense-8+Frequency-16", "ranks": ranks})
    layer = art.load_moe_layer(mpath, 0, str(adir), plan=ppath, top_k=K)
    for m in (1, 40, 130):  # decode and prefill paths
        x = rng.normal(0, 1, (m, d)).astype(np.float32)
        logits = rng.normal(0, 1, (m, E)).astype(np.float32)
        ids, w = oracle.router_topk(logits, K, 0)
        want = oracle.moe_forward(o_ex, [], x, ids, w)
        got = layer.forward(torch.from_numpy(x).cuda(), torch.from_numpy(logits).cuda()).cpu().numpy()
        assert rel_err(got, want) <= 1e-4
    # the plan must agree with the artifacts
    bad = dict(ranks, **{"layer0.expert0.w3": 16})  # the file holds rank 8
    with pytest.raises(gpu.PlanError):
        art.load_moe_layer(mpath, 0, str(adir), plan=_dump(tmp_path / "bad.json", {"policy": "p", "ranks": bad}))
    missing = {k: v for k, v in ranks.items() if k != "layer0.expert2.w2"}
    with pytest.raises(gpu.PlanError):
        art.load_moe_layer(mpath, 0, str(adir), plan=_dump(tmp_path / "miss.json", {"policy": "p", "ranks": missing}))
