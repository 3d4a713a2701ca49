"""MILO1 container fixtures for the loader tests (tests/test_containers.py).

packed-i3 files are written by the REFERENCE's own milo::save_packed
(pack.cpp:306-343, compiled into oracle/_ref/libmilo_ref.so by oracle/build_ref.sh),
in the three layouts the reference produces.  Compensator factor files follow the
format the reference's quantize writes (pipeline.cpp:233-283: symm-i3 = u8 codes +
binary16 scales per (row, 64-group), U k x r and V^T n x r "transposed"; real = f32
U k x r and V r x n); that writer sits in an anonymous namespace of the reference,
so it is restated here (json.dumps with the same keys; the reader ignores key order).

    python tests/golden/make_containers.py      # needs oracle/_ref/libmilo_ref.so
"""
import json, os, struct, sys
import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Oracle  # noqa: E402

OUT = os.path.join(HERE, "containers")


def container(path, header: dict, payload: bytes):
    h = json.dumps(header, separators=(",", ":")).encode()
    with open(path, "wb") as f:
        f.write(b"MILO1" + struct.pack("<I", len(h)) + h + payload)


def half_bits(x: np.ndarray) -> np.ndarray:
    return np.asarray(x, np.float32).astype(np.float16).view(np.uint16)


def main():
    ref = Oracle("ref")
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(2504)
    # 1. asymmetric linear (the shape quantize writes, pipeline.cpp:324), unsplit
    P = ref.random_packed(128, 256, 1, 11)
    ref.save_packed(P, "layer0.w1", os.path.join(OUT, "asym_linear.packed.milo"))
    # 2. symmetric linear, split planes
    codes = rng.integers(0, 8, (32, 256), dtype=np.uint8)
    scales = (np.abs(rng.normal(0, 0.05, 32 * 256 // 64)) + 0.01).astype(np.float32)
    P = ref.pack_matrix(codes, scales, None, split=True)
    ref.save_packed(P, "layer0.w3", os.path.join(OUT, "sym_linear_split.packed.milo"))
    # 3. asymmetric tiled16x64, split planes
    codes = rng.integers(0, 8, (64, 128), dtype=np.uint8)
    scales = (np.abs(rng.normal(0, 0.05, 64 * 128 // 64)) + 0.01).astype(np.float32)
    zeros = (3.5 + rng.normal(0, 1, 64 * 128 // 64)).astype(np.float32)
    P = ref.pack_matrix(codes, scales, zeros, tiled=True, split=True)
    ref.save_packed(P, "layer0.w2", os.path.join(OUT, "asym_tiled_split.packed.milo"))
    # compensators for the 128 x 256 matrix (file 1): rank 16 symm-i3, rank 8 real
    k, n = 128, 256
    for r, storage in ((16, "symm-int3"), (8, "real")):
        base = os.path.join(OUT, f"comp_r{r}_{'i3' if storage != 'real' else 'real'}")
        if storage == "real":
            U = rng.normal(0, 0.05, (k, r)).astype(np.float32)
            V = rng.normal(0, 0.05, (r, n)).astype(np.float32)
            hu = dict(name="layer0.w1.U", rows=k, cols=r, dtype="f32", role="compensator-U", rank=r, storage="real")
            hv = dict(hu, name="layer0.w1.V", rows=r, cols=n, role="compensator-V")
            container(base + ".u.milo", hu, U.tobytes())
            container(base + ".v.milo", hv, V.tobytes())
        else:
            for rows, role, tr, suf in ((k, "compensator-U", False, ".u.milo"), (n, "compensator-V", True, ".v.milo")):
                codes = rng.integers(0, 8, (rows, r), dtype=np.uint8)
                sc = (np.abs(rng.normal(0, 0.05, (rows, (r + 63) // 64))) + 0.01).astype(np.float32)
                h = dict(name="layer0.w1." + role[-1], rows=rows, cols=r, dtype="symm-i3", role=role, rank=r,
                         storage="symm-int3", group_size=64, transposed=tr)
                container(base + suf, h, codes.tobytes() + half_bits(sc).tobytes())
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
