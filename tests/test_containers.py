"""MILO1 container loaders: the B200 library's C++
readers against the reference's own writer/reader on committed fixtures
(tests/golden/make_containers.py), error categories like milo::load_packed, and
(GPU) loaded weights / compensators through the kernels against the oracle."""
import json
import os
import struct

import numpy as np
import pytest

from tests.helpers import rel_err

FIX = os.path.join(os.path.dirname(__file__), "golden", "containers")
PACKED = ["asym_linear.packed.milo", "sym_linear_split.packed.milo", "asym_tiled_split.packed.milo"]


@pytest.fixture(scope="module")
def mb():
    import paper_2504_02658_b200 as m
    m.lib()
    return m


def _eq(a, b):
    if a is None or b is None:
        return a is None and b is None
    return np.array_equal(np.asarray(a).ravel(), np.asarray(b).ravel())


@pytest.mark.parametrize("name", PACKED)
def test_packed_loader_matches_reference_reader(mb, ref, name):
    path = os.path.join(FIX, name)
    got = mb.load_packed_host(path)
    want = ref.load_packed(path)
    assert (got.rows, got.cols, got.layout, got.split, got.mode, got.group_size) == \
        (want.rows, want.cols, want.layout, want.split, want.mode, want.group_size)
    for f in ("words", "plane_a", "plane_b", "scales", "zeros"):
        assert _eq(getattr(got, f), getattr(want, f)), f


def _write(path, header, payload: bytes, magic=b"MILO1"):
    h = json.dumps(header).encode()
    with open(path, "wb") as f:
        f.write(magic + struct.pack("<I", len(h)) + h + payload)


def test_packed_loader_error_categories(mb, tmp_path):
    src = os.path.join(FIX, "asym_linear.packed.milo")
    raw = open(src, "rb").read()
    hlen = struct.unpack("<I", raw[5:9])[0]
    header = json.loads(raw[9:9 + hlen])
    payload = raw[9 + hlen:]
    with pytest.raises(mb.IoError):
        mb.load_packed_host(str(tmp_path / "missing.milo"))
    p = tmp_path / "magic.milo"
    _write(p, header, payload, magic=b"MILO2")
    with pytest.raises(mb.FormatError):
        mb.load_packed_host(str(p))
    p = tmp_path / "short.milo"
    _write(p, header, payload[:-2])
    with pytest.raises(mb.FormatError):
        mb.load_packed_host(str(p))
    p = tmp_path / "dtype.milo"
    _write(p, dict(header, dtype="f32"), payload)
    with pytest.raises(mb.FormatError):
        mb.load_packed_host(str(p))
    p = tmp_path / "layout.milo"
    _write(p, dict(header, layout="tiled32x32"), payload)
    with pytest.raises(mb.FormatError):
        mb.load_packed_host(str(p))
    p = tmp_path / "header.milo"
    with open(p, "wb") as f:
        f.write(b"MILO1" + struct.pack("<I", 7) + b"{rows:1")
    with pytest.raises(mb.FormatError):
        mb.load_packed_host(str(p))
    # a header with extra / reordered keys (nlohmann writes sorted keys) still loads
    p = tmp_path / "reordered.milo"
    _write(p, dict(reversed(list(header.items())), extra={"a": [1, 2]}), payload)
    got = mb.load_packed_host(str(p))
    assert (got.rows, got.cols) == (header["rows"], header["cols"])


def _read_factor(path):
    raw = open(path, "rb").read()
    hlen = struct.unpack("<I", raw[5:9])[0]
    h = json.loads(raw[9:9 + hlen])
    return h, raw[9 + hlen:]


def _oracle_comp(prefix):
    """The factor pair as the oracle's Comp (symm-i3 scales as stored: binary16)."""
    from oracle.oracle import Comp
    hu, pu = _read_factor(prefix + ".u.milo")
    hv, pv = _read_factor(prefix + ".v.milo")
    r = hu["rank"]
    if hu["dtype"] == "f32":
        U = np.frombuffer(pu, np.float32).reshape(hu["rows"], hu["cols"])
        V = np.frombuffer(pv, np.float32).reshape(hv["rows"], hv["cols"])
        return Comp(hu["rows"], hv["cols"], r, 0, U=U.copy(), V=V.copy())
    def fac(h, p):
        n = h["rows"] * h["cols"]
        codes = np.frombuffer(p[:n], np.uint8).reshape(h["rows"], h["cols"]).copy()
        sc = np.frombuffer(p[n:], np.uint16).view(np.float16).astype(np.float32).reshape(h["rows"], -1)
        return codes, sc
    qu, qus = fac(hu, pu)
    qv, qvs = fac(hv, pv)
    return Comp(hu["rows"], hv["rows"], r, 1, qu_codes=qu, qu_scales=qus, qvt_codes=qv, qvt_scales=qvs,
                group_size=hu["group_size"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", PACKED)
def test_loaded_weight_unpacks_and_dequantizes_bit_exact(gpu, oracle, ref, name):
    import torch
    path = os.path.join(FIX, name)
    W = gpu.Weight.load(path)
    P = ref.load_packed(path)
    assert (W.rows, W.cols) == (P.rows, P.cols)
    assert np.array_equal(W.unpack_codes().cpu().numpy(), oracle.unpack_codes(P))
    dq = W.dequant_half().cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(dq, oracle.dequant_half(P))


@pytest.mark.gpu
@pytest.mark.parametrize("comp", ["comp_r16_i3", "comp_r8_real"])
def test_loaded_compensator_gemm_matches_oracle(gpu, oracle, ref, comp):
    from oracle.oracle import GemmCfg
    path = os.path.join(FIX, "asym_linear.packed.milo")
    P = ref.load_packed(path)
    W = gpu.Weight.load(path)
    C = gpu.Comp.load(os.path.join(FIX, comp + ".u.milo"), os.path.join(FIX, comp + ".v.milo"))
    oc = _oracle_comp(os.path.join(FIX, comp))
    for m in (1, 5):
        A = np.random.default_rng(m).normal(0, 1, (m, P.rows)).astype(np.float32)
        want = oracle.gemm_w3a16(A, P, oc, GemmCfg(tile_k=128, tile_n=128, mode=1))
        import torch
        got = gpu.gemm_w3a16(torch.from_numpy(A).cuda(), W, C,
                             gpu.GemmConfig(tile_shape=(128, 128), mode=1)).cpu().numpy()
        assert rel_err(got, want) <= 1e-5
