"""numpy/ctypes front end for the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Two interchangeable backends with the same Python API:
  * ``Oracle("oracle")`` — oracle/libmilo_oracle.so, our C restatement
    (oracle/milo_oracle.c) of the reference hot path;
  * ``Oracle("ref")``    — oracle/_ref/libmilo_ref.so, the reference's own
    sources compiled by oracle/build_ref.sh (exists only where it was built).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module.  The product path (paper_2504_02658_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libmilo_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmilo_ref.so")

u8p = C.POINTER(C.c_uint8)
u16p = C.POINTER(C.c_uint16)
u32p = C.POINTER(C.c_uint32)
i32p = C.POINTER(C.c_int32)
f32p = C.POINTER(C.c_float)

STATUS_NAMES = {0: "ok", 1: "format", 2: "data", 3: "io", 4: "shape", 5: "rank",
                6: "numeric", 7: "stat", 8: "plan", 9: "range", 10: "config"}


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        self.status = status
        self.category = STATUS_NAMES.get(status, "unknown")
        super().__init__(f"{self.category} error ({status}) {msg}")


def build_oracle() -> str:
    """Compiles the C restatement (make -C oracle)."""
    import subprocess
    subprocess.check_call(["make", "-s", "-C", HERE, "libmilo_oracle.so"])
    return ORACLE_SO


def _p(a, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


@dataclass
class Packed:
    """Mirror of milo::PackedInt3Matrix (proj/include/milo/pack.hpp:45-66)."""
    rows: int
    cols: int
    layout: int = 0          # 0 linear, 1 tiled16x64
    split: bool = False
    mode: int = 1            # 0 symmetric, 1 asymmetric
    group_size: int = 64
    words: Optional[np.ndarray] = None
    plane_a: Optional[np.ndarray] = None
    plane_b: Optional[np.ndarray] = None
    scales: Optional[np.ndarray] = None   # uint16 binary16
    zeros: Optional[np.ndarray] = None    # uint16 binary16, None = empty

    def arrays(self):
        return (_p(self.words, u32p), _p(self.plane_a, u32p), _p(self.plane_b, u32p),
                _p(self.scales, u16p), _p(self.zeros, u16p))


@dataclass
class Comp:
    """Mirror of milo::Compensator (proj/include/milo/lowrank.hpp:31-50)."""
    rows: int
    cols: int
    rank: int
    storage: int = 1  # 0 real, 1 symm-int3
    U: Optional[np.ndarray] = None
    V: Optional[np.ndarray] = None
    qu_codes: Optional[np.ndarray] = None    # rows x rank uint8
    qu_scales: Optional[np.ndarray] = None   # rows x ceil(rank/g) f32
    qvt_codes: Optional[np.ndarray] = None   # cols x rank uint8
    qvt_scales: Optional[np.ndarray] = None  # cols x ceil(rank/g) f32
    group_size: int = 64


@dataclass
class GemmCfg:
    """Mirror of milo::GemmConfig (proj/include/milo/gemm.hpp:17-25)."""
    tile_k: int = 128
    tile_n: int = 128
    group_size: int = 64
    mode: int = 1
    pipeline_depth: int = 4
    materialize_compensator: bool = False


class _ORPacked(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("layout", C.c_int),
                ("split", C.c_int), ("mode", C.c_int), ("group_size", C.c_uint64),
                ("words", u32p), ("plane_a", u32p), ("plane_b", u32p), ("scales", u16p),
                ("zeros", u16p)]


class _ORComp(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("rank", C.c_uint64),
                ("storage", C.c_int), ("U", f32p), ("V", f32p), ("qu_codes", u8p),
                ("qu_scales", f32p), ("qvt_codes", u8p), ("qvt_scales", f32p),
                ("group_size", C.c_uint64)]


class _ORCfg(C.Structure):
    _fields_ = [("tile_k", C.c_int), ("tile_n", C.c_int), ("group_size", C.c_uint64),
                ("mode", C.c_int), ("pipeline_depth", C.c_int),
                ("materialize_compensator", C.c_int)]


class _ORExpert(C.Structure):
    _fields_ = [("w", _ORPacked * 3), ("c", _ORComp * 3), ("has_comp", C.c_int * 3)]


def _or_packed(P: Packed) -> _ORPacked:
    w, a, b, s, z = P.arrays()
    return _ORPacked(P.rows, P.cols, P.layout, int(P.split), P.mode, P.group_size, w, a, b, s, z)


def _or_comp(c: Comp) -> _ORComp:
    return _ORComp(c.rows, c.cols, c.rank, c.storage, _p(c.U, f32p), _p(c.V, f32p),
                   _p(c.qu_codes, u8p), _p(c.qu_scales, f32p), _p(c.qvt_codes, u8p),
                   _p(c.qvt_scales, f32p), c.group_size)


def _or_cfg(g: GemmCfg) -> _ORCfg:
    return _ORCfg(g.tile_k, g.tile_n, g.group_size, g.mode, g.pipeline_depth,
                  int(g.materialize_compensator))


class Oracle:
    def __init__(self, which: str = "oracle"):
        self.which = which
        path = ORACLE_SO if which == "oracle" else REF_SO
        if which == "oracle" and not os.path.exists(path):
            build_oracle()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self._pre = "or_" if which == "oracle" else "ref_"
        self._setup()

    @staticmethod
    def available(which: str) -> bool:
        return os.path.exists(ORACLE_SO if which == "oracle" else REF_SO)

    def _f(self, name, restype, argtypes):
        fn = getattr(self.lib, self._pre + name)
        fn.restype = restype
        fn.argtypes = argtypes
        return fn

    def _setup(self):
        u16, u32, u64, i, f, d = C.c_uint16, C.c_uint32, C.c_uint64, C.c_int, C.c_float, C.c_double
        self.float_to_half = self._f("float_to_half", u16, [f])
        self.half_to_float = self._f("half_to_float", f, [u16])
        self.double_to_half = self._f("double_to_half", u16, [d])
        self.half_add = self._f("half_add", u16, [u16, u16])
        self.half_sub = self._f("half_sub", u16, [u16, u16])
        self.half_mul = self._f("half_mul", u16, [u16, u16])
        self.half_fma = self._f("half_fma", u16, [u16, u16, u16])
        self.symmetric_step = self._f("symmetric_step", u16, [u16])
        self.asymmetric_offset = self._f("asymmetric_offset", u16, [u16, u16])
        self.tiled_position = self._f("tiled_position", u64, [u64, u64, u64, u64])
        self._pack32 = self._f("pack32", i, [u8p, C.c_size_t if self.which == "oracle" else u64, u32p])
        self._unpack32 = self._f("unpack32", None, [u32p, u8p])
        self._fdp = self._f("fast_dequant_pair", None, [u32, i, i, u16p])
        self._pack_matrix = self._f("pack_matrix", i, [u64, u64, u8p, f32p, f32p, u64, i, i,
                                                       u32p, u32p, u32p, u16p, u16p])
        self._quant = self._f("quantize_minmax", i, ([u64, u64, u64] if self.which == "oracle" else [u64, u64]) + [f32p, u8p, f32p, f32p])
        self._sq = self._f("symm_int3_quantize", i, [f32p, u64, u64, u64, u8p, f32p])
        self._mmb = self._f("matrix_memory_bytes", u64, [u64, u64, u64, i, u64, i])
        if self.which == "oracle":
            self._unpack_codes = self._f("unpack_codes", i, [u64, u64, i, i, u32p, u32p, u32p, u8p])
            self._dq = self._f("dequant_packed_half", i, [u64, u64, i, i, u64, u32p, u32p, u32p,
                                                          u16p, u16p, i, u16p])
            self._sdq = self._f("symm_int3_dequantize", None, [u64, u64, u64, u8p, f32p, f32p])
            self._gemm = self._f("gemm_w3a16", i, [f32p, u64, u64, C.POINTER(_ORPacked),
                                                   C.POINTER(_ORComp), C.POINTER(_ORCfg), f32p])
            self._ptc = self._f("pipeline_tail_check", i, [u64, C.POINTER(_ORCfg), i32p, i, i32p])
            self._router = self._f("router_topk", None, [f32p, u64, i, i, i, i32p, f32p])
            self._rgemm = self._f("router_gemm", None, [f32p, u64, u64, u16p, i, f32p])
            self._moe = self._f("moe_forward", i, [C.POINTER(_ORExpert), i, C.POINTER(_ORExpert), i,
                                                   f32p, u64, u64, i, i32p, f32p, i, f32p])
        else:
            self._unpack_codes = self._f("unpack_codes", i, [u64, u64, i, i, i, u64, u32p, u32p,
                                                             u32p, u16p, u16p, u8p])
            self._dq = self._f("dequant_packed_half", i, [u64, u64, i, i, i, u64, u32p, u32p, u32p,
                                                          u16p, u16p, i, u16p])
            self._sdq = self._f("symm_int3_dequantize", i, [u64, u64, u64, u8p, f32p, f32p])
            self._gemm = self._f("gemm_w3a16", i, [f32p, u64, u64, u64, i, i, i, u64, u32p, u32p,
                                                   u32p, u16p, u16p, i, u64, u64, u64, i, f32p,
                                                   f32p, u8p, f32p, u8p, f32p, u64, i, i, u64, i,
                                                   i, i, u64, f32p])
            self._ptc = self._f("pipeline_tail_check", i, [u64, i, i, i, i32p, i, i32p])
            self._rp = self._f("random_packed", i, [u64, u64, i, u64, u32p, u16p, u16p])
            self._fill_normal = self._f("fill_normal", None, [u64, u64, f, f, f32p])
            self._fnv = self._f("fnv1a64", u64, [C.c_char_p])
            self._cq = self._f("comp_quantize", i, [u64, u64, u64, f32p, f32p, u64, u8p, f32p,
                                                    u8p, f32p])
            self._save_packed = self._f("save_packed", i, [u64, u64, i, i, i, u64, u32p, u32p, u32p, u16p,
                                                           u16p, C.c_char_p, C.c_char_p])
            self._load_info = self._f("load_packed_info", i, [C.c_char_p, C.POINTER(u64)])
            self._load_packed = self._f("load_packed", i, [C.c_char_p, u32p, u32p, u32p, u16p, u16p])
            self.lib.ref_last_error.restype = C.c_char_p
            self.lib.ref_moe_create.restype = C.c_void_p
            self.lib.ref_moe_create.argtypes = [i]
            self.lib.ref_moe_destroy.argtypes = [C.c_void_p]
            self.lib.ref_moe_set_linear.restype = i
            self.lib.ref_moe_set_linear.argtypes = [C.c_void_p, i, i, u64, u64, u32p, u16p, u16p,
                                                    u64, u8p, f32p, u8p, f32p]
            self.lib.ref_moe_prepare.restype = i
            self.lib.ref_moe_prepare.argtypes = [C.c_void_p, i]
            self.lib.ref_moe_forward.restype = i
            self.lib.ref_moe_forward.argtypes = [C.c_void_p, f32p, u64, u64, i, i32p, f32p, i, f32p]

    def _check(self, st):
        if st:
            msg = self.lib.ref_last_error().decode() if self.which == "ref" else ""
            raise OracleError(st, msg)

    # ---- pack.hpp ----------------------------------------------------------
    def pack32(self, codes) -> np.ndarray:
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        out = np.zeros(3, np.uint32)
        self._check(self._pack32(_p(codes, u8p), codes.size, _p(out, u32p)))
        return out

    def unpack32(self, w3) -> np.ndarray:
        w3 = np.ascontiguousarray(w3, dtype=np.uint32)
        out = np.zeros(32, np.uint8)
        self._unpack32(_p(w3, u32p), _p(out, u8p))
        return out

    def fast_dequant_pair(self, word: int, pair: int, mode: int):
        out = np.zeros(2, np.uint16)
        self._fdp(word, pair, mode, _p(out, u16p))
        return int(out[0]), int(out[1])

    def pack_matrix(self, codes, scales, zeros=None, group_size=64, tiled=False,
                    split=False) -> Packed:
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        rows, cols = codes.shape
        scales = np.ascontiguousarray(scales, dtype=np.float32).ravel()
        zeros_a = None if zeros is None else np.ascontiguousarray(zeros, dtype=np.float32).ravel()
        groups = rows * cols // 32
        words = None if split else np.zeros(groups * 3, np.uint32)
        pa = np.zeros(groups * 2, np.uint32) if split else None
        pb = np.zeros(groups, np.uint32) if split else None
        qg = rows * cols // group_size
        sh = np.zeros(qg, np.uint16)
        zh = None if zeros is None else np.zeros(qg, np.uint16)
        self._check(self._pack_matrix(rows, cols, _p(codes, u8p), _p(scales, f32p),
                                      _p(zeros_a, f32p), group_size, int(tiled), int(split),
                                      _p(words, u32p), _p(pa, u32p), _p(pb, u32p), _p(sh, u16p),
                                      _p(zh, u16p)))
        return Packed(rows, cols, 1 if tiled else 0, split, 0 if zeros is None else 1,
                      group_size, words, pa, pb, sh, zh)

    def unpack_codes(self, P: Packed) -> np.ndarray:
        out = np.zeros((P.rows, P.cols), np.uint8)
        w, a, b, s, z = P.arrays()
        if self.which == "oracle":
            self._check(self._unpack_codes(P.rows, P.cols, P.layout, int(P.split), w, a, b,
                                           _p(out, u8p)))
        else:
            self._check(self._unpack_codes(P.rows, P.cols, P.layout, int(P.split), P.mode,
                                           P.group_size, w, a, b, s, z, _p(out, u8p)))
        return out

    def dequant_half(self, P: Packed, mode: Optional[int] = None) -> np.ndarray:
        mode = P.mode if mode is None else mode
        out = np.zeros((P.rows, P.cols), np.uint16)
        w, a, b, s, z = P.arrays()
        if self.which == "oracle":
            st = self._dq(P.rows, P.cols, P.layout, int(P.split), P.group_size, w, a, b, s, z,
                          mode, _p(out, u16p))
        else:
            st = self._dq(P.rows, P.cols, P.layout, int(P.split), P.mode, P.group_size, w, a, b,
                          s, z, mode, _p(out, u16p))
        self._check(st)
        return out

    # ---- quant / lowrank ----------------------------------------------------
    def quantize_minmax(self, w: np.ndarray, group_size=64):
        w = np.ascontiguousarray(w, dtype=np.float32)
        rows, cols = w.shape
        codes = np.zeros((rows, cols), np.uint8)
        qg = rows * cols // group_size
        sc = np.zeros(qg, np.float32)
        ze = np.zeros(qg, np.float32)
        if self.which == "oracle":
            st = self._quant(rows, cols, group_size, _p(w, f32p), _p(codes, u8p), _p(sc, f32p),
                             _p(ze, f32p))
        else:
            st = self._quant(rows, cols, _p(w, f32p), _p(codes, u8p), _p(sc, f32p), _p(ze, f32p))
        self._check(st)
        return codes, sc, ze

    def symm_int3_quantize(self, values, rows, cols, group_size=64):
        values = np.ascontiguousarray(values, dtype=np.float32).ravel()
        codes = np.zeros(rows * cols, np.uint8)
        gpr = (cols + group_size - 1) // group_size
        sc = np.zeros(rows * gpr, np.float32)
        self._check(self._sq(_p(values, f32p), rows, cols, group_size, _p(codes, u8p),
                             _p(sc, f32p)))
        return codes.reshape(rows, cols), sc.reshape(rows, gpr)

    def symm_int3_dequantize(self, codes, scales, group_size=64):
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        scales = np.ascontiguousarray(scales, dtype=np.float32)
        rows, cols = codes.shape
        out = np.zeros((rows, cols), np.float32)
        st = self._sdq(rows, cols, group_size, _p(codes, u8p), _p(scales, f32p), _p(out, f32p))
        if self.which == "ref":
            self._check(st)
        return out

    def quantize_comp(self, U: np.ndarray, V: np.ndarray, group_size=64) -> Comp:
        """Compensator::quantize_symm_int3 (lowrank.cpp:34-50) from real factors."""
        rows, rank = U.shape
        cols = V.shape[1]
        qu, qus = self.symm_int3_quantize(U, rows, rank, group_size)
        qvt, qvts = self.symm_int3_quantize(np.ascontiguousarray(V.T), cols, rank, group_size)
        return Comp(rows, cols, rank, 1, None, None, qu, qus, qvt, qvts, group_size)

    def matrix_memory_bytes(self, rows, cols, rank, bits=3, group_size=64, comp_bits=3) -> int:
        return int(self._mmb(rows, cols, rank, bits, group_size, comp_bits))

    # ---- gemm.hpp -----------------------------------------------------------
    def pipeline_tail_check(self, k: int, cfg: GemmCfg):
        stages = np.zeros(4096, np.int32)
        n = np.zeros(1, np.int32)
        if self.which == "oracle":
            c = _or_cfg(cfg)
            st = self._ptc(k, C.byref(c), _p(stages, i32p), 4096, _p(n, i32p))
        else:
            st = self._ptc(k, cfg.tile_k, cfg.tile_n, cfg.pipeline_depth, _p(stages, i32p), 4096,
                           _p(n, i32p))
        self._check(st)
        return [int(x) for x in stages[: int(n[0])]]

    def gemm_w3a16(self, A: np.ndarray, P: Packed, comp: Optional[Comp] = None,
                   cfg: Optional[GemmCfg] = None) -> np.ndarray:
        cfg = cfg or GemmCfg(mode=P.mode)
        A = np.ascontiguousarray(A, dtype=np.float32)
        m, acols = A.shape
        out = np.zeros((m, P.cols), np.float32)
        if self.which == "oracle":
            pk = _or_packed(P)
            cc = _or_comp(comp) if comp is not None else None
            gc = _or_cfg(cfg)
            st = self._gemm(_p(A, f32p), m, acols, C.byref(pk),
                            C.byref(cc) if cc is not None else None, C.byref(gc), _p(out, f32p))
        else:
            w, a, b, s, z = P.arrays()
            has = comp is not None
            c = comp or Comp(0, 0, 0)
            st = self._gemm(_p(A, f32p), m, P.rows, P.cols, P.layout, int(P.split), P.mode,
                            P.group_size, w, a, b, s, z, int(has), c.rows, c.cols, c.rank,
                            c.storage, _p(c.U, f32p), _p(c.V, f32p), _p(c.qu_codes, u8p),
                            _p(c.qu_scales, f32p), _p(c.qvt_codes, u8p), _p(c.qvt_scales, f32p),
                            c.group_size, cfg.tile_k, cfg.tile_n, cfg.group_size, cfg.mode,
                            cfg.pipeline_depth, int(cfg.materialize_compensator), acols,
                            _p(out, f32p))
        self._check(st)
        return out

    # ---- reference-only generators -------------------------------------------
    def random_packed(self, k, n, mode, seed) -> Packed:
        """pipeline.cpp:408-426 (linear layout)."""
        assert self.which == "ref"
        words = np.zeros(k * n // 32 * 3, np.uint32)
        sh = np.zeros(k * n // 64, np.uint16)
        zh = np.zeros(k * n // 64, np.uint16) if mode == 1 else None
        self._check(self._rp(k, n, mode, seed, _p(words, u32p), _p(sh, u16p), _p(zh, u16p)))
        return Packed(k, n, 0, False, mode, 64, words, None, None, sh, zh)

    def save_packed(self, P: Packed, name: str, path: str):
        """milo::save_packed (pack.cpp:306-343): the reference's packed-i3 MILO1 writer."""
        assert self.which == "ref"
        self._check(self._save_packed(P.rows, P.cols, P.layout, int(P.split), P.mode, P.group_size,
                                      _p(P.words, u32p), _p(P.plane_a, u32p), _p(P.plane_b, u32p),
                                      _p(P.scales, u16p), _p(P.zeros, u16p), name.encode(), str(path).encode()))

    def load_packed(self, path: str) -> Packed:
        """milo::load_packed (pack.cpp:345-400)."""
        assert self.which == "ref"
        info = (C.c_uint64 * 6)()
        self._check(self._load_info(str(path).encode(), info))
        rows, cols, layout, split, mode, gs = (int(v) for v in info)
        groups = rows * cols // 32
        qg = rows * cols // gs
        words = None if split else np.zeros(groups * 3, np.uint32)
        pa = np.zeros(groups * 2, np.uint32) if split else None
        pb = np.zeros(groups, np.uint32) if split else None
        sh = np.zeros(qg, np.uint16)
        zh = np.zeros(qg, np.uint16) if mode == 1 else None
        self._check(self._load_packed(str(path).encode(), _p(words, u32p), _p(pa, u32p), _p(pb, u32p),
                                      _p(sh, u16p), _p(zh, u16p)))
        return Packed(rows, cols, layout, bool(split), mode, gs, words, pa, pb, sh, zh)

    def fill_normal(self, seed, count, mean=0.0, sigma=1.0) -> np.ndarray:
        assert self.which == "ref"
        out = np.zeros(count, np.float32)
        self._fill_normal(seed, count, mean, sigma, _p(out, f32p))
        return out

    def fnv1a64(self, s: str) -> int:
        assert self.which == "ref"
        return int(self._fnv(s.encode()))

    # ---- MoE (new layer, defined in milo_oracle.h) ----------------------------
    def router_gemm(self, x: np.ndarray, gate_bits: np.ndarray) -> np.ndarray:
        """The MoE gate in the device's exact fp32 order (or_router_gemm)."""
        assert self.which == "oracle"
        x = np.ascontiguousarray(x, dtype=np.float32)
        g = np.ascontiguousarray(gate_bits, dtype=np.uint16)
        m, d = x.shape
        E = g.shape[0]
        out = np.zeros((m, E), np.float32)
        self._rgemm(_p(x, f32p), m, d, _p(g, u16p), E, _p(out, f32p))
        return out

    def router_topk(self, logits: np.ndarray, K: int, score_mode: int = 0):
        assert self.which == "oracle"
        logits = np.ascontiguousarray(logits, dtype=np.float32)
        m, E = logits.shape
        ids = np.zeros((m, K), np.int32)
        w = np.zeros((m, K), np.float32)
        self._router(_p(logits, f32p), m, E, K, score_mode, _p(ids, i32p), _p(w, f32p))
        return ids, w

    def moe_forward(self, experts, shared, x, topk_ids, topk_w, n_threads=1):
        """experts/shared: lists of dicts {"w": [P1,P3,P2], "c": [C1,C3,C2] (None ok)}."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        topk_ids = np.ascontiguousarray(topk_ids, dtype=np.int32)
        topk_w = np.ascontiguousarray(topk_w, dtype=np.float32)
        m, d = x.shape
        K = topk_ids.shape[1]
        out = np.zeros((m, d), np.float32)
        if self.which == "oracle":
            def mk(ex):
                s = _ORExpert()
                for j in range(3):
                    s.w[j] = _or_packed(ex["w"][j])
                    c = ex["c"][j]
                    if c is not None and c.rank > 0:
                        s.c[j] = _or_comp(c)
                        s.has_comp[j] = 1
                return s
            arr = (_ORExpert * max(1, len(experts)))(*[mk(e) for e in experts])
            sarr = (_ORExpert * max(1, len(shared)))(*[mk(e) for e in shared])
            st = self._moe(arr, len(experts), sarr, len(shared), _p(x, f32p), m, d, K,
                           _p(topk_ids, i32p), _p(topk_w, f32p), n_threads, _p(out, f32p))
            self._check(st)
            return out
        h = RefMoE(self, experts, shared, n_threads)
        try:
            return h.forward(x, topk_ids, topk_w)
        finally:
            h.close()


class RefMoE:
    """A persistent MoE composition over the compiled reference (oracle/_ref):
    experts copied in once and cut into column slices for `workers` threads
    (ref_moe_prepare), so that forward() times only the reference's own
    gemm_w3a16 calls (oracle/ref/ref_capi.cpp ref_moe_forward)."""

    def __init__(self, o: "Oracle", experts, shared, workers: int = 1):
        assert o.which == "ref"
        self.o, self.lib = o, o.lib
        self.n_routed, self.n_shared = len(experts), len(shared)
        self.workers = workers
        allx = list(experts) + list(shared)
        self.h = self.lib.ref_moe_create(len(allx))
        for e, ex in enumerate(allx):
            for j in range(3):
                P = ex["w"][j]
                c = ex["c"][j]
                r = 0 if c is None else c.rank
                o._check(self.lib.ref_moe_set_linear(
                    self.h, e, j, P.rows, P.cols, _p(P.words, u32p), _p(P.scales, u16p),
                    _p(P.zeros, u16p), r, _p(c.qu_codes if r else None, u8p),
                    _p(c.qu_scales if r else None, f32p), _p(c.qvt_codes if r else None, u8p),
                    _p(c.qvt_scales if r else None, f32p)))
        o._check(self.lib.ref_moe_prepare(self.h, workers))

    def forward(self, x, topk_ids, topk_w):
        x = np.ascontiguousarray(x, dtype=np.float32)
        topk_ids = np.ascontiguousarray(topk_ids, dtype=np.int32)
        topk_w = np.ascontiguousarray(topk_w, dtype=np.float32)
        m, d = x.shape
        out = np.zeros((m, d), np.float32)
        if self.n_shared:
            # shared experts appended to the top-k lists with weight 1
            sid = np.tile(np.arange(self.n_routed, self.n_routed + self.n_shared, dtype=np.int32), (m, 1))
            ids2 = np.ascontiguousarray(np.concatenate([topk_ids, sid], 1))
            w2 = np.ascontiguousarray(np.concatenate([topk_w, np.ones((m, self.n_shared), np.float32)], 1))
        else:
            ids2, w2 = topk_ids, topk_w
        self.o._check(self.lib.ref_moe_forward(self.h, _p(x, f32p), m, d, ids2.shape[1],
                                               _p(ids2, i32p), _p(w2, f32p), self.workers,
                                               _p(out, f32p)))
        return out

    def close(self):
        if self.h:
            self.lib.ref_moe_destroy(self.h)
            self.h = None

    __del__ = close
