"""B200-native MiLo INT3 + LoRC hot path — Python mirror of the reference API.

Thin ctypes binding over the C ABI in include/milo_b200.h (libmilo_b200.so,
built in-tree by paper_2504_02658_b200/build.py).  Names and argument meaning
follow the reference's C++ operator API:

    milo::gemm_w3a16(A, PackedInt3Matrix, optional<Compensator>, GemmConfig)
        (proj/include/milo/gemm.hpp:43-48)

and the top-k routed grouped-expert call the reference lacks.  Errors raise
MiloError subclasses named after milo::ErrorCode (errors.hpp:9-48).

There is no CPU fallback: if the CUDA library is missing or no sm_100 device
is present, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libmilo_b200.so")

# ---------------------------------------------------------------- errors
_STATUS = {1: "Format", 2: "Data", 3: "Io", 4: "Shape", 5: "Rank", 6: "Numeric", 7: "Stat",
           8: "Plan", 9: "Range", 10: "Config", 100: "Cuda", 101: "Argument"}


class MiloError(RuntimeError):
    status = 0

    def __init__(self, msg: str = ""):
        super().__init__(msg)


def _mk(name, status):
    return type(name, (MiloError,), {"status": status})


FormatError = _mk("FormatError", 1)
DataError = _mk("DataError", 2)
IoError = _mk("IoError", 3)
ShapeError = _mk("ShapeError", 4)
RankError = _mk("RankError", 5)
NumericError = _mk("NumericError", 6)
StatError = _mk("StatError", 7)
PlanError = _mk("PlanError", 8)
RangeError = _mk("RangeError", 9)
ConfigError = _mk("ConfigError", 10)
CudaError = _mk("CudaError", 100)
ArgumentError = _mk("ArgumentError", 101)
_ERRORS = {c.status: c for c in (FormatError, DataError, IoError, ShapeError, RankError,
                                   NumericError, StatError, PlanError, RangeError, ConfigError,
                                   CudaError, ArgumentError)}

# ---------------------------------------------------------------- enums
LINEAR, TILED16X64 = 0, 1
SYMMETRIC, ASYMMETRIC = 0, 1
F32, F16 = 0, 1
COMP_REAL, COMP_SYMM_INT3 = 0, 1
SCORE_SOFTMAX_TOPK, SCORE_SOFTMAX_ALL = 0, 1

u8p = C.POINTER(C.c_uint8)
u16p = C.POINTER(C.c_uint16)
u32p = C.POINTER(C.c_uint32)
f32p = C.POINTER(C.c_float)
vp = C.c_void_p


class _PackedDesc(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("layout", C.c_int32),
                ("split", C.c_int32), ("mode", C.c_int32), ("group_size", C.c_uint64),
                ("words", u32p), ("n_words", C.c_uint64), ("plane_a", u32p),
                ("n_plane_a", C.c_uint64), ("plane_b", u32p), ("n_plane_b", C.c_uint64),
                ("scales", u16p), ("n_scales", C.c_uint64), ("zeros", u16p),
                ("n_zeros", C.c_uint64)]


class _CompDesc(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("rank", C.c_uint64),
                ("storage", C.c_int32), ("U", f32p), ("V", f32p), ("qu_codes", u8p),
                ("qu_scales", f32p), ("qvt_codes", u8p), ("qvt_scales", f32p),
                ("group_size", C.c_uint64)]


class _GemmCfg(C.Structure):
    _fields_ = [("tile_k", C.c_int32), ("tile_n", C.c_int32), ("group_size", C.c_uint64),
                ("mode", C.c_int32), ("pipeline_depth", C.c_int32),
                ("materialize_compensator", C.c_int32)]


class _ExpertDesc(C.Structure):
    _fields_ = [("w1", vp), ("w3", vp), ("w2", vp), ("c1", vp), ("c3", vp), ("c2", vp)]


_lib = None


def lib() -> C.CDLL:
    """Loads libmilo_b200.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("MILO_B200_LIB_VARIANT")  # tools/: an experimental build of the same library
    path = os.path.join(os.path.dirname(LIB_PATH), "variants", f"libmilo_b200_{path}.so") if path else LIB_PATH
    if not os.path.exists(path):
        raise CudaError(f"{LIB_PATH} missing: run paper_2504_02658_b200/build.py "
                        "(there is no CPU fallback)")
    L = C.CDLL(path)
    i32, i64, u64 = C.c_int32, C.c_int64, C.c_uint64
    L.milo_last_error.restype = C.c_char_p
    L.milo_status_name.restype = C.c_char_p
    L.milo_launch_count.restype = u64
    L.milo_profile_enable.argtypes = [i32]
    L.milo_profile_enable.restype = None
    L.milo_profile_read.argtypes = [i32, C.POINTER(C.c_double)]
    L.milo_profile_read.restype = i64
    sig = {
        "milo_device_check": [],
        "milo_weight_create": [C.POINTER(_PackedDesc), C.POINTER(vp)],
        "milo_weight_destroy": [vp],
        "milo_weight_info": [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(i32), C.POINTER(u64)],
        "milo_comp_info": [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64), C.POINTER(i32)],
        "milo_unpack_codes": [vp, vp, vp],
        "milo_dequant_half": [vp, i32, vp, vp],
        "milo_comp_create": [C.POINTER(_CompDesc), C.POINTER(vp)],
        "milo_comp_destroy": [vp],
        "milo_gemm_w3a16": [vp, vp, C.POINTER(_GemmCfg), vp, i64, i64, i32, vp, i32, vp],
        "milo_gemm_w3a16_host": [vp, vp, C.POINTER(_GemmCfg), f32p, i64, i64, f32p],
        "milo_moe_create": [C.POINTER(_ExpertDesc), i32, C.POINTER(_ExpertDesc), i32, i32, i32,
                            C.POINTER(vp)],
        "milo_moe_destroy": [vp],
        "milo_router_topk": [vp, i64, i32, i32, i32, vp, vp, vp],
        "milo_moe_forward": [vp, vp, i64, i32, vp, vp, i32, vp, vp, vp],
        "milo_moe_forward_routed": [vp, vp, i64, i32, vp, vp, vp, i32, vp],
        "milo_moe_forward_host": [vp, f32p, i64, i64, f32p, i64, f32p],
        "milo_stream_release": [vp],
        "milo_ep_unique_id": [vp, i64],
        "milo_ep_comm_create": [vp, i32, i32, C.POINTER(vp)],
        "milo_ep_comm_destroy": [vp],
        "milo_ep_layer_create": [vp, vp, i32, i32, i32, vp, C.POINTER(vp)],
        "milo_ep_layer_destroy": [vp],
        "milo_ep_forward": [vp, vp, i64, i32, vp, vp, i32, vp],
        "milo_router_gemm": [vp, i64, i64, i32, vp, i32, vp, vp],
        "milo_moe_set_gate": [vp, u16p, i64, i64],
        "milo_moe_forward_x": [vp, vp, i64, i32, vp, i32, vp, vp, vp],
        "milo_packed_load_host": [C.c_char_p, C.POINTER(_PackedDesc), C.POINTER(vp)],
        "milo_weight_load": [C.c_char_p, C.POINTER(vp)],
        "milo_comp_load": [C.c_char_p, C.c_char_p, C.POINTER(vp)],
        "milo_ep_dispatch": [vp, i64, i32, i32, i32, i32, vp, i32, i64, vp, i64, vp, vp, vp],
        "milo_ep_combine": [vp, vp, vp, i64, i32, i64, vp, vp],
    }
    for name, args in sig.items():
        if hasattr(L, name):
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
    _lib = L
    return L


def _check(status: int):
    if status:
        msg = lib().milo_last_error().decode(errors="replace")
        raise _ERRORS.get(status, MiloError)(msg)


def stream_release(stream=None):
    """Frees the scratch regions the library keeps for (current device, stream)."""
    _check(lib().milo_stream_release(_stream_ptr(stream)))


def launch_count() -> int:
    return int(lib().milo_launch_count())


def profile_enable(on: bool = True):
    lib().milo_profile_enable(int(on))


def profile_read(kind: int):
    """(launches, total_ms) of kernel kind 0 gemm phase 1, 1 phase 2, 2 lorc, 3 other."""
    t = C.c_double()
    n = lib().milo_profile_read(kind, C.byref(t))
    return int(n), float(t.value)


def device_check():
    _check(lib().milo_device_check())


def _np_ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _stream_ptr(stream=None):
    import torch
    if stream is not None:
        return C.c_void_p(stream.cuda_stream)
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)  # no Stream object per call
    if raw is not None:
        return C.c_void_p(raw(torch.cuda.current_device()))
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dptr(t):
    return C.c_void_p(t.data_ptr())


# ---------------------------------------------------------------- host mirrors
@dataclass
class PackedInt3Matrix:
    """milo::PackedInt3Matrix (pack.hpp:45-66): rows = k, cols = n."""
    rows: int
    cols: int
    layout: int = LINEAR
    split: bool = False
    mode: int = ASYMMETRIC
    group_size: int = 64
    words: Optional[np.ndarray] = None
    plane_a: Optional[np.ndarray] = None
    plane_b: Optional[np.ndarray] = None
    scales: Optional[np.ndarray] = None  # uint16 binary16
    zeros: Optional[np.ndarray] = None   # uint16 binary16 or None


@dataclass
class Compensator:
    """milo::Compensator (lowrank.hpp:31-50)."""
    rows: int
    cols: int
    rank: int
    storage: int = COMP_SYMM_INT3
    U: Optional[np.ndarray] = None
    V: Optional[np.ndarray] = None
    qu_codes: Optional[np.ndarray] = None
    qu_scales: Optional[np.ndarray] = None
    qvt_codes: Optional[np.ndarray] = None
    qvt_scales: Optional[np.ndarray] = None
    group_size: int = 64


@dataclass
class GemmConfig:
    """milo::GemmConfig (gemm.hpp:17-25)."""
    tile_shape: tuple = (128, 128)
    group_size: int = 64
    mode: int = ASYMMETRIC
    pipeline_depth: int = 4
    materialize_compensator: bool = False

    def _c(self) -> _GemmCfg:
        return _GemmCfg(int(self.tile_shape[0]), int(self.tile_shape[1]), self.group_size,
                        self.mode, self.pipeline_depth, int(self.materialize_compensator))


def _c32(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt).ravel()


def load_packed_host(path: str) -> PackedInt3Matrix:
    """Reads a packed-i3 MILO1 container (milo::load_packed, pack.cpp:345-400) on
    the host: the library's C++ reader, no device needed."""
    d = _PackedDesc()
    h = vp()
    _check(lib().milo_packed_load_host(str(path).encode(), C.byref(d), C.byref(h)))
    try:
        def arr(ptr, n, dt):
            return None if not ptr or n == 0 else np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True)
        return PackedInt3Matrix(int(d.rows), int(d.cols), int(d.layout), bool(d.split), int(d.mode),
                                int(d.group_size), arr(d.words, d.n_words, np.uint32),
                                arr(d.plane_a, d.n_plane_a, np.uint32), arr(d.plane_b, d.n_plane_b, np.uint32),
                                arr(d.scales, d.n_scales, np.uint16), arr(d.zeros, d.n_zeros, np.uint16))
    finally:
        lib().milo_packed_host_free(h)


class Weight:
    """Device-resident packed INT3 weight (milo_weight handle), repacked once."""

    @classmethod
    def load(cls, path: str) -> "Weight":
        """From a packed-i3 MILO1 container written by the reference's save_packed."""
        self = cls.__new__(cls)
        h = vp()
        _check(lib().milo_weight_load(str(path).encode(), C.byref(h)))
        self._h = h
        self._keep = None
        rows, cols, mode = C.c_uint64(), C.c_uint64(), C.c_int32()
        _check(lib().milo_weight_info(h, C.byref(rows), C.byref(cols), C.byref(mode), None))
        self.rows, self.cols, self.mode = rows.value, cols.value, mode.value
        return self

    def __init__(self, p):
        self._keep = [_c32(p.words, np.uint32), _c32(p.plane_a, np.uint32),
                      _c32(p.plane_b, np.uint32), _c32(p.scales, np.uint16),
                      _c32(p.zeros, np.uint16)]
        w, a, b, s, z = self._keep
        d = _PackedDesc(p.rows, p.cols, p.layout, int(bool(p.split)), p.mode, p.group_size,
                        _np_ptr(w, u32p), 0 if w is None else w.size, _np_ptr(a, u32p),
                        0 if a is None else a.size, _np_ptr(b, u32p), 0 if b is None else b.size,
                        _np_ptr(s, u16p), 0 if s is None else s.size, _np_ptr(z, u16p),
                        0 if z is None else z.size)
        h = vp()
        _check(lib().milo_weight_create(C.byref(d), C.byref(h)))
        self._h = h
        self._keep = None
        self.rows, self.cols, self.mode = p.rows, p.cols, p.mode

    @property
    def handle(self):
        return self._h

    @property
    def device_bytes(self) -> int:
        b = C.c_uint64()
        _check(lib().milo_weight_info(self._h, None, None, None, C.byref(b)))
        return b.value

    def unpack_codes(self, stream=None):
        import torch
        out = torch.empty((self.rows, self.cols), dtype=torch.uint8, device="cuda")
        _check(lib().milo_unpack_codes(self._h, _dptr(out), _stream_ptr(stream)))
        return out

    def dequant_half(self, mode: Optional[int] = None, stream=None):
        """binary16 bit patterns (torch.int16 view of uint16) in logical order."""
        import torch
        out = torch.empty((self.rows, self.cols), dtype=torch.float16, device="cuda")
        _check(lib().milo_dequant_half(self._h, self.mode if mode is None else mode, _dptr(out),
                                       _stream_ptr(stream)))
        return out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.milo_weight_destroy(h)
            self._h = None


class Comp:
    """Device-resident compensator (milo_comp handle)."""

    @classmethod
    def load(cls, u_path: str, v_path: str) -> "Comp":
        """From the factor pair the reference's quantize writes (<name>.u.milo / .v.milo)."""
        self = cls.__new__(cls)
        h = vp()
        _check(lib().milo_comp_load(str(u_path).encode(), str(v_path).encode(), C.byref(h)))
        self._h = h
        rows, cols, rank, storage = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int32()
        _check(lib().milo_comp_info(h, C.byref(rows), C.byref(cols), C.byref(rank), C.byref(storage)))
        self.rows, self.cols, self.rank, self.storage = rows.value, cols.value, rank.value, storage.value
        return self

    def __init__(self, c):
        keep = dict(U=_c32(c.U, np.float32), V=_c32(c.V, np.float32),
                    qu=_c32(c.qu_codes, np.uint8), qus=_c32(c.qu_scales, np.float32),
                    qvt=_c32(c.qvt_codes, np.uint8), qvts=_c32(c.qvt_scales, np.float32))
        d = _CompDesc(c.rows, c.cols, c.rank, c.storage, _np_ptr(keep["U"], f32p),
                      _np_ptr(keep["V"], f32p), _np_ptr(keep["qu"], u8p),
                      _np_ptr(keep["qus"], f32p), _np_ptr(keep["qvt"], u8p),
                      _np_ptr(keep["qvts"], f32p), c.group_size)
        h = vp()
        _check(lib().milo_comp_create(C.byref(d), C.byref(h)))
        self._h = h
        self.rows, self.cols, self.rank = c.rows, c.cols, c.rank

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.milo_comp_destroy(h)
            self._h = None


def gemm_w3a16(A, W: Weight, comp: Optional[Comp] = None, cfg: Optional[GemmConfig] = None,
               out_dtype=None, out=None, stream=None):
    """C = A_f16 (dequant(W) + U V) on the device (torch CUDA tensors in/out).

    A: (m, k) float32 or float16 CUDA tensor.  Returns (m, n) float32 (default)
    or float16.  Mirrors milo::gemm_w3a16 (gemm.cpp:117-199)."""
    import torch
    cfg = cfg or GemmConfig(mode=W.mode)
    if A.dim() != 2:
        raise ShapeError("A must be 2-D")
    A = A.contiguous()
    a_dt = F32 if A.dtype == torch.float32 else F16 if A.dtype == torch.float16 else None
    if a_dt is None:
        raise ArgumentError("A must be float32 or float16")
    m = A.shape[0]
    if out is not None:
        # the output buffer defines the output type
        if out_dtype is not None and out_dtype != out.dtype:
            raise ArgumentError("out_dtype does not match out.dtype")
        out_dtype = out.dtype
        if (out.dtype not in (torch.float32, torch.float16) or tuple(out.shape) != (m, W.cols)
                or not out.is_contiguous() or out.device != A.device):
            raise ArgumentError("out must be a contiguous (m, n) float32/float16 tensor on A's device")
    out_dtype = out_dtype or torch.float32
    if out_dtype not in (torch.float32, torch.float16):
        raise ArgumentError("out_dtype must be float32 or float16")
    c_dt = F32 if out_dtype == torch.float32 else F16
    if out is None:
        out = torch.empty((m, W.cols), dtype=out_dtype, device=A.device)
    c = cfg._c()
    _check(lib().milo_gemm_w3a16(W.handle, comp.handle if comp is not None else None,
                                 C.byref(c), _dptr(A), m, A.shape[1], a_dt, _dptr(out), c_dt,
                                 _stream_ptr(stream)))
    return out


def gemm_w3a16_host(A: np.ndarray, W: Weight, comp: Optional[Comp] = None,
                    cfg: Optional[GemmConfig] = None) -> np.ndarray:
    """Host-buffer variant (the reference's by-value semantics); blocking."""
    cfg = cfg or GemmConfig(mode=W.mode)
    A = np.ascontiguousarray(A, dtype=np.float32)
    m, acols = A.shape
    out = np.empty((m, W.cols), np.float32)
    c = cfg._c()
    _check(lib().milo_gemm_w3a16_host(W.handle, comp.handle if comp is not None else None,
                                      C.byref(c), _np_ptr(A, f32p), m, acols, _np_ptr(out, f32p)))
    return out


# ---------------------------------------------------------------- MoE layer
@dataclass
class Expert:
    """One expert FFN: w1 (d x f), w3 (d x f), w2 (f x d) + optional compensators."""
    w1: Weight
    w3: Weight
    w2: Weight
    c1: Optional[Comp] = None
    c3: Optional[Comp] = None
    c2: Optional[Comp] = None

    def _desc(self) -> _ExpertDesc:
        def h(x):
            return None if x is None else x.handle
        return _ExpertDesc(h(self.w1), h(self.w3), h(self.w2), h(self.c1), h(self.c3), h(self.c2))


def router_gemm(x, gate, stream=None):
    """The MoE gate on the device: logits (m, E) fp32 = half(x) gate^T, gate a
    (E, d) float16 CUDA tensor (fixed fp32 order, oracle/milo_oracle.c or_router_gemm)."""
    import torch
    x = x.contiguous()
    gate = gate.contiguous().half()
    m, d = x.shape
    E = gate.shape[0]
    if gate.shape[1] != d:
        raise ShapeError(f"gate {tuple(gate.shape)} vs x {tuple(x.shape)}")
    logits = torch.empty((m, E), dtype=torch.float32, device=x.device)
    _check(lib().milo_router_gemm(_dptr(x), m, d, F32 if x.dtype == torch.float32 else F16, _dptr(gate), E,
                                  _dptr(logits), _stream_ptr(stream)))
    return logits


def router_topk(logits, top_k: int, score_mode: int = SCORE_SOFTMAX_TOPK, stream=None):
    import torch
    logits = logits.contiguous().float()
    m, E = logits.shape
    ids = torch.empty((m, top_k), dtype=torch.int32, device=logits.device)
    w = torch.empty((m, top_k), dtype=torch.float32, device=logits.device)
    _check(lib().milo_router_topk(_dptr(logits), m, E, top_k, score_mode, _dptr(ids), _dptr(w),
                                  _stream_ptr(stream)))
    return ids, w


class MoELayer:
    """Top-k routed grouped-expert layer over device-resident experts."""

    def __init__(self, experts: Sequence[Expert], shared: Sequence[Expert] = (), top_k: int = 2,
                 score_mode: int = SCORE_SOFTMAX_TOPK):
        self.experts = list(experts)
        self.shared = list(shared)
        self.top_k = top_k
        self.score_mode = score_mode
        ed = (_ExpertDesc * max(1, len(self.experts)))(*[e._desc() for e in self.experts])
        sd = (_ExpertDesc * max(1, len(self.shared)))(*[e._desc() for e in self.shared])
        h = vp()
        _check(lib().milo_moe_create(ed, len(self.experts), sd, len(self.shared), top_k,
                                     score_mode, C.byref(h)))
        self._h = h
        self.d = self.experts[0].w1.rows if self.experts else self.shared[0].w1.rows

    def forward(self, x, router_logits, out_dtype=None, return_routing=False, stream=None):
        import torch
        x = x.contiguous()
        m = x.shape[0]
        x_dt = F32 if x.dtype == torch.float32 else F16
        out_dtype = out_dtype or torch.float32
        out = torch.empty((m, self.d), dtype=out_dtype, device=x.device)
        ids = w = None
        if return_routing:
            ids = torch.empty((m, self.top_k), dtype=torch.int32, device=x.device)
            w = torch.empty((m, self.top_k), dtype=torch.float32, device=x.device)
        lg = None if router_logits is None else router_logits.contiguous().float()
        _check(lib().milo_moe_forward(self._h, _dptr(x), m, x_dt,
                                      _dptr(lg) if lg is not None else None, _dptr(out),
                                      F32 if out_dtype == torch.float32 else F16,
                                      _dptr(ids) if ids is not None else None,
                                      _dptr(w) if w is not None else None, _stream_ptr(stream)))
        return (out, ids, w) if return_routing else out

    def set_gate(self, gate):
        """Attaches the router gate: (E, d) float16 values (numpy or torch, host or device)."""
        g = gate.detach().cpu().numpy() if hasattr(gate, "detach") else np.asarray(gate)
        g = np.ascontiguousarray(g.astype(np.float16)).view(np.uint16)
        if g.ndim != 2:
            raise ShapeError("gate must be (E, d)")
        _check(lib().milo_moe_set_gate(self._h, _np_ptr(g, u16p), g.shape[0], g.shape[1]))

    def forward_x(self, x, out_dtype=None, return_routing=False, stream=None):
        """The whole MoE block from x: router GEMM (set_gate) -> top-k -> experts -> combine."""
        import torch
        x = x.contiguous()
        m = x.shape[0]
        out_dtype = out_dtype or torch.float32
        out = torch.empty((m, self.d), dtype=out_dtype, device=x.device)
        ids = w = None
        if return_routing:
            ids = torch.empty((m, self.top_k), dtype=torch.int32, device=x.device)
            w = torch.empty((m, self.top_k), dtype=torch.float32, device=x.device)
        _check(lib().milo_moe_forward_x(self._h, _dptr(x), m, F32 if x.dtype == torch.float32 else F16, _dptr(out),
                                        F32 if out_dtype == torch.float32 else F16,
                                        _dptr(ids) if ids is not None else None,
                                        _dptr(w) if w is not None else None, _stream_ptr(stream)))
        return (out, ids, w) if return_routing else out

    def forward_routed(self, x, topk_ids, topk_w, out_dtype=None, stream=None):
        import torch
        x = x.contiguous()
        m = x.shape[0]
        out_dtype = out_dtype or torch.float32
        out = torch.empty((m, self.d), dtype=out_dtype, device=x.device)
        _check(lib().milo_moe_forward_routed(self._h, _dptr(x), m,
                                             F32 if x.dtype == torch.float32 else F16,
                                             _dptr(topk_ids.contiguous().int()),
                                             _dptr(topk_w.contiguous().float()), _dptr(out),
                                             F32 if out_dtype == torch.float32 else F16,
                                             _stream_ptr(stream)))
        return out

    def forward_host(self, x: np.ndarray, router_logits: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float32)
        lg = np.ascontiguousarray(router_logits, dtype=np.float32)
        if x.ndim != 2 or lg.ndim != 2 or lg.shape[0] != x.shape[0]:
            raise ShapeError(f"x {x.shape} / router logits {lg.shape}: need (m, d) / (m, E)")
        out = np.empty((x.shape[0], self.d), np.float32)
        _check(lib().milo_moe_forward_host(self._h, _np_ptr(x, f32p), x.shape[0], x.shape[1],
                                           _np_ptr(lg, f32p), lg.shape[1], _np_ptr(out, f32p)))
        return out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.milo_moe_destroy(h)
            self._h = None


# ---------------------------------------------------------------- expert-parallel helpers
def ep_dispatch(ids, x, world: int, per: int, capacity: int, stream=None, packed: bool = False):
    """Fixed-capacity EP dispatch on the device.  Returns (send_x f16 [world*C, d],
    send_meta int32 [world*C], slot int32 [m*K]); packed=True: (send f16
    [world*C, d + 8] with the local expert id as int32 at column d, None, slot)."""
    import torch
    m, K = ids.shape
    d = x.shape[1]
    ld = d + 8 if packed else d
    send_x = torch.empty((world * capacity, ld), dtype=torch.float16, device=x.device)
    send_m = None if packed else torch.empty((world * capacity,), dtype=torch.int32, device=x.device)
    slot = torch.empty((m * K,), dtype=torch.int32, device=x.device)
    ids = ids.contiguous().int()
    x = x.contiguous()
    _check(lib().milo_ep_dispatch(_dptr(ids), m, K, world, per, capacity, _dptr(x),
                                  F32 if x.dtype == torch.float32 else F16, d, _dptr(send_x), ld,
                                  _dptr(send_m) if send_m is not None else None, _dptr(slot),
                                  _stream_ptr(stream)))
    return send_x, send_m, slot


def ep_combine(y, slot, wts, stream=None):
    import torch
    m, K = wts.shape
    d = y.shape[1]
    out = torch.empty((m, d), dtype=torch.float32, device=y.device)
    _check(lib().milo_ep_combine(_dptr(y.contiguous()), _dptr(slot), _dptr(wts.contiguous().float()), m, K,
                                 d, _dptr(out), _stream_ptr(stream)))
    return out
