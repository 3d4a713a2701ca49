"""Shared synthetic-input helpers for the parity tests (numpy, seeded)."""
import numpy as np


def rel_err(c, ref):
    c = np.asarray(c, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.sqrt((ref * ref).sum())
    num = np.sqrt(((c - ref) ** 2).sum())
    return num / den if den > 0 else num


def random_quantized(oracle, k, n, seed, mode=1, tiled=False, split=False, sigma=0.05):
    """Weights ~ N(0, sigma) -> min/max INT3 g64 (quant.cpp:23-76) -> packed.
    Symmetric: codes U[0,7], scales |N(0,.05)|+0.01 (pipeline.cpp:418-424)."""
    rng = np.random.default_rng(seed)
    if mode == 1:
        w = rng.normal(0.0, sigma, (k, n)).astype(np.float32)
        codes, sc, ze = oracle.quantize_minmax(w)
        return oracle.pack_matrix(codes, sc, ze, tiled=tiled, split=split), codes
    codes = rng.integers(0, 8, (k, n), dtype=np.uint8)
    sc = (np.abs(rng.normal(0.0, 0.05, k * n // 64)) + 0.01).astype(np.float32)
    return oracle.pack_matrix(codes, sc, None, tiled=False, split=split), codes


def random_comp(oracle, k, n, rank, seed, storage=1, sigma=0.05):
    rng = np.random.default_rng(seed)
    U = rng.normal(0.0, sigma, (k, rank)).astype(np.float32)
    V = rng.normal(0.0, sigma, (rank, n)).astype(np.float32)
    if storage == 1:
        return oracle.quantize_comp(U, V)
    from oracle.oracle import Comp
    return Comp(k, n, rank, 0, U, V)
