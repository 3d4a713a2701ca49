"""Host-side packed-INT3 format utilities (numpy), mirroring the reference's
storage API so callers can build PackedInt3Matrix inputs without the C++
library.  These are format conversions run once on the host (the reference's
offline `milo pack` stage), not the hot path, which is on the device only.

    pack32 / unpack32        proj/src/pack.cpp:33-68
    pack_linear(_symmetric)  proj/src/pack.cpp:97-131
    tiled_position           proj/src/pack.cpp:133-139
    reshuffle_tiled          proj/src/pack.cpp:141-161
    split_planes             proj/src/pack.cpp:163-178
    unpack_codes             proj/src/pack.cpp:196-211
    float_to_half            proj/include/milo/half.hpp:47-78 (IEEE RNE == numpy)

Canonical 32-code group (pack.hpp:6-24): word j bits [3k, 3k+3) = e_{8j+k};
bits [24, 32) of word j = byte j of the 24-bit `rest` holding e24..e31.
"""
from __future__ import annotations

from typing import Optional

import numpy as np

from . import ASYMMETRIC, LINEAR, SYMMETRIC, TILED16X64, Compensator, PackedInt3Matrix, \
    RangeError, ShapeError


def float_to_half_bits(x) -> np.ndarray:
    """binary16 RNE of float32 values (== milo::float_to_half)."""
    return np.asarray(x, np.float32).astype(np.float16).view(np.uint16)


def pack_groups(codes: np.ndarray) -> np.ndarray:
    """(G, 32) codes in [0, 7] -> (G, 3) uint32 words (vectorized pack32)."""
    c = np.ascontiguousarray(codes, dtype=np.uint8)
    if c.ndim != 2 or c.shape[1] != 32:
        raise ShapeError("pack32 takes exactly 32 codes per group")
    if (c > 7).any():
        raise RangeError("pack32 code outside [0, 7]")
    c = c.astype(np.uint32)
    shifts = (3 * np.arange(8, dtype=np.uint32))
    w = np.zeros((c.shape[0], 3), np.uint32)
    for j in range(3):
        w[:, j] = (c[:, 8 * j:8 * j + 8] << shifts).sum(axis=1, dtype=np.uint64).astype(np.uint32)
    rest = (c[:, 24:32] << shifts).sum(axis=1, dtype=np.uint64).astype(np.uint32)
    for j in range(3):
        w[:, j] |= ((rest >> np.uint32(8 * j)) & np.uint32(0xFF)) << np.uint32(24)
    return w


def unpack_groups(words: np.ndarray) -> np.ndarray:
    """(G, 3) uint32 -> (G, 32) uint8 codes (vectorized unpack32)."""
    w = np.ascontiguousarray(words, dtype=np.uint32).reshape(-1, 3)
    shifts = (3 * np.arange(8, dtype=np.uint32))
    out = np.zeros((w.shape[0], 32), np.uint8)
    for j in range(3):
        out[:, 8 * j:8 * j + 8] = ((w[:, j:j + 1] >> shifts) & 7).astype(np.uint8)
    rest = (w[:, 0] >> 24) | ((w[:, 1] >> 24) << 8) | ((w[:, 2] >> 24) << 16)
    out[:, 24:32] = ((rest[:, None] >> shifts) & 7).astype(np.uint8)
    return out


def pack32(codes) -> np.ndarray:
    return pack_groups(np.asarray(codes, np.uint8).reshape(1, -1))[0]


def unpack32(words) -> np.ndarray:
    return unpack_groups(np.asarray(words, np.uint32).reshape(1, 3))[0]


def tiled_order(rows: int, cols: int) -> np.ndarray:
    """Stream position of every logical (i, j) in the tiled16x64 layout."""
    i = np.arange(rows)[:, None]
    j = np.arange(cols)[None, :]
    return ((i // 16) * (cols // 64) + j // 64) * 1024 + (i % 16) * 64 + j % 64


def pack_matrix(codes: np.ndarray, scales, zeros=None, group_size: int = 64,
                tiled: bool = False, split: bool = False) -> PackedInt3Matrix:
    """Logical row-major codes (rows x cols) + per-group scales/zeros (float)
    -> PackedInt3Matrix.  zeros=None selects symmetric mode
    (pack_linear_symmetric); otherwise asymmetric (pack_linear /
    reshuffle_tiled).  Optional plane split (split_planes)."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    rows, cols = codes.shape
    if rows == 0 or cols == 0:
        raise ShapeError("cannot pack an empty matrix")
    if cols % 32:
        raise ShapeError(f"cols {cols} not a multiple of 32")
    if zeros is None and cols % group_size:
        raise ShapeError("group_size does not divide cols")
    if tiled and (rows % 16 or cols % 64):
        raise ShapeError("tiled layout needs rows % 16 == 0 and cols % 64 == 0")
    stream = codes.ravel()
    if tiled:
        s = np.empty_like(stream)
        s[tiled_order(rows, cols).ravel()] = stream
        stream = s
    w = pack_groups(stream.reshape(-1, 32))
    p = PackedInt3Matrix(rows, cols, TILED16X64 if tiled else LINEAR, split,
                         SYMMETRIC if zeros is None else ASYMMETRIC, group_size)
    if split:
        p.plane_a = np.ascontiguousarray(w[:, :2]).ravel()
        p.plane_b = np.ascontiguousarray(w[:, 2])
    else:
        p.words = w.ravel()
    p.scales = float_to_half_bits(np.asarray(scales, np.float32).ravel())
    p.zeros = None if zeros is None else float_to_half_bits(np.asarray(zeros, np.float32).ravel())
    return p


def unpack_codes(p: PackedInt3Matrix) -> np.ndarray:
    if p.split:
        w = np.stack([p.plane_a.reshape(-1, 2)[:, 0], p.plane_a.reshape(-1, 2)[:, 1],
                      p.plane_b], axis=1)
    else:
        w = p.words.reshape(-1, 3)
    stream = unpack_groups(w).ravel()
    if p.layout == LINEAR:
        return stream.reshape(p.rows, p.cols)
    return stream[tiled_order(p.rows, p.cols)]


def random_packed(rows: int, cols: int, rng: np.random.Generator, mode: int = ASYMMETRIC,
                  scale_sigma: float = 0.05) -> PackedInt3Matrix:
    """Seeded synthetic packed weights with the reference generators' statistics
    (pipeline.cpp:408-426): codes U[0,7]; scales |N(0, sigma)| + 0.01; asymmetric
    zero-points N(3.5, 1)."""
    codes = rng.integers(0, 8, (rows, cols), dtype=np.uint8)
    ng = rows * cols // 64
    scales = (np.abs(rng.normal(0.0, scale_sigma, ng)) + 0.01).astype(np.float32)
    zeros = None if mode == SYMMETRIC else (3.5 + rng.normal(0.0, 1.0, ng)).astype(np.float32)
    return pack_matrix(codes, scales, zeros)


def random_compensator(rows: int, cols: int, rank: int, rng: np.random.Generator,
                       sigma: float = 0.02) -> Optional[Compensator]:
    """Synthetic symm-int3 compensator (lowrank.hpp:19-50 storage): codes
    U[0,7], per-64-group float scales along the rank axis."""
    if rank <= 0:
        return None
    gpr = (rank + 63) // 64
    return Compensator(
        rows, cols, rank, 1, None, None,
        rng.integers(0, 8, (rows, rank), dtype=np.uint8),
        (np.abs(rng.normal(0.0, sigma, (rows, gpr))) + 1e-3).astype(np.float32),
        rng.integers(0, 8, (cols, rank), dtype=np.uint8),
        (np.abs(rng.normal(0.0, sigma, (cols, gpr))) + 1e-3).astype(np.float32), 64)
