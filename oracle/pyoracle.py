"""pyoracle -- TEST INFRASTRUCTURE ONLY.

numpy/ctypes front-end over the two CPU checkers in this directory:

* ``liboracle.so``            -- the plain-C restatement (bitgnn_oracle.c);
* ``_ref/libbitgnn_ref.so``   -- the unmodified reference library compiled
                                 from /root/reference/proj/src (ref_capi.cpp).

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs import this module.  The product package
(paper_2305_02522_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbitgnn_ref.so")

F, B = 0, 1
BMM, BSPMM, ADD, CONCAT = 0, 1, 2, 3
ROW, COL = 0, 1
GCN, SAGE, GRAPHCONV, FC, SOFTMAX = 0, 1, 2, 3, 7


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and _ref when the reference sources exist)."""
    out = subprocess.run(["make", "-C", HERE, "-j8", "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def spw(cols: int, word_bits: int) -> int:
    """Storage u32 words per packed row (bitdense.hpp:72-73)."""
    return (cols + word_bits - 1) // word_bits * (word_bits // 32)


# --------------------------------------------------------------------------- #
# ctypes plumbing for liboracle.so
# --------------------------------------------------------------------------- #
class _Rng(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]


class _Frdc(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.POINTER(C.c_uint64)), ("col_ind", C.POINTER(C.c_uint32)),
                ("tiles", C.POINTER(C.c_uint16))]


class _Variant(C.Structure):
    _fields_ = [("op", C.c_int), ("in1", C.c_int), ("in2", C.c_int), ("out", C.c_int)]


class _Mat(C.Structure):
    _fields_ = [("prec", C.c_int), ("rows", C.c_int64), ("cols", C.c_int64),
                ("word_bits", C.c_int), ("f", C.POINTER(C.c_float)),
                ("bits", C.POINTER(C.c_uint32)), ("scale", C.POINTER(C.c_float))]


class _Graph(C.Structure):
    _fields_ = [("n", C.c_int64), ("structure", _Frdc), ("raw", _Frdc),
                ("norm", C.POINTER(C.c_float)), ("mean_row", C.POINTER(C.c_float)),
                ("ones", C.POINTER(C.c_float)), ("neighbor_count", C.POINTER(C.c_int64))]


class _Layer(C.Structure):
    _fields_ = [("kind", C.c_int), ("nplan", C.c_int), ("plan", _Variant * 4),
                ("w1", C.POINTER(C.c_float)), ("w1_rows", C.c_int64), ("w1_cols", C.c_int64),
                ("w2", C.POINTER(C.c_float)), ("w2_rows", C.c_int64), ("w2_cols", C.c_int64),
                ("relu", C.c_int)]


_TRACE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_char_p, C.POINTER(C.c_uint32), C.c_int64,
                        C.c_int64, C.c_int)

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.og_rng_seed.argtypes = [C.POINTER(_Rng), C.c_uint64]
        L.og_rng_next.restype = C.c_uint64
        L.og_rng_next.argtypes = [C.POINTER(_Rng)]
        L.og_rng_uniform.restype = C.c_double
        L.og_rng_uniform.argtypes = [C.POINTER(_Rng)]
        L.og_rng_index.restype = C.c_int64
        L.og_rng_index.argtypes = [C.POINTER(_Rng), C.c_int64]
        L.og_random_dense.argtypes = [C.POINTER(_Rng), C.c_int64, C.c_int64, C.c_void_p]
        L.og_random_edges.restype = C.c_int64
        L.og_random_edges.argtypes = [C.POINTER(_Rng), C.c_int64, C.c_int64, C.c_int,
                                      C.c_void_p, C.c_void_p]
        L.og_spw.restype = C.c_int64
        L.og_binarize.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p]
        L.og_l1_scales.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p]
        L.og_transpose_bits.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p]
        L.og_frdc_from_edges.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_int,
                                         C.POINTER(_Frdc), C.POINTER(C.c_int64)]
        L.og_frdc_free.argtypes = [C.POINTER(_Frdc)]
        L.og_row_popcounts.argtypes = [C.POINTER(_Frdc), C.c_void_p]
        L.og_mat_free.argtypes = [C.POINTER(_Mat)]
        L.og_bmm.argtypes = [_Variant, C.POINTER(_Mat), C.POINTER(_Mat), C.c_int, C.POINTER(_Mat)]
        L.og_bspmm.argtypes = [_Variant, C.POINTER(_Frdc), C.c_void_p, C.c_void_p,
                               C.POINTER(_Mat), C.c_int, C.POINTER(_Mat)]
        L.og_add.argtypes = [_Variant, C.POINTER(_Mat), C.POINTER(_Mat), C.POINTER(_Mat)]
        L.og_relu.argtypes = [C.POINTER(_Mat)]
        L.og_softmax_rows.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]
        L.og_error.restype = C.c_char_p
        L.og_prepare_graph.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
                                       C.POINTER(_Graph)]
        L.og_graph_free.argtypes = [C.POINTER(_Graph)]
        L.og_run_model.argtypes = [C.POINTER(_Layer), C.c_int, C.c_int, C.POINTER(_Graph),
                                   C.c_void_p, C.c_int64, C.c_int64,
                                   C.POINTER(C.POINTER(C.c_float)), C.POINTER(C.POINTER(C.c_float)),
                                   C.POINTER(C.c_int64), _TRACE_FN, C.c_void_p]
        L.og_free.argtypes = [C.c_void_p]
        L.og_tileset_count.restype = C.c_int64
        L.og_tileset_count.argtypes = [C.POINTER(_Frdc), C.c_int64, C.c_int]
        L.og_gather_tileset.argtypes = [C.POINTER(_Frdc), C.c_int64, C.c_int64, C.c_int,
                                        C.POINTER(TileSetC)]
        L.og_frdc_to_dense.argtypes = [C.POINTER(_Frdc), C.c_int, C.c_void_p]
        _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _err() -> str:
    return lib().og_error().decode()


# --------------------------------------------------------------------------- #
# rng.hpp
# --------------------------------------------------------------------------- #
class Rng:
    """std::mt19937_64 + the reference's mappings (rng.hpp:16-80)."""

    def __init__(self, seed: int):
        self._s = _Rng()
        lib().og_rng_seed(C.byref(self._s), C.c_uint64(seed))

    def next(self) -> int:
        return lib().og_rng_next(C.byref(self._s))

    def uniform(self) -> float:
        return lib().og_rng_uniform(C.byref(self._s))

    def index(self, n: int) -> int:
        return lib().og_rng_index(C.byref(self._s), n)

    def range(self, lo: int, hi: int) -> int:
        return lo + self.index(hi - lo + 1)

    def random_dense(self, rows: int, cols: int) -> np.ndarray:
        out = np.empty((rows, cols), dtype=np.float32)
        lib().og_random_dense(C.byref(self._s), rows, cols, _ptr(out))
        return out

    def random_edges(self, nodes: int, m: int, allow_self: bool = False) -> Tuple[np.ndarray, np.ndarray]:
        src = np.empty(max(m, 1), dtype=np.int64)
        dst = np.empty(max(m, 1), dtype=np.int64)
        k = lib().og_random_edges(C.byref(self._s), nodes, m, int(allow_self), _ptr(src), _ptr(dst))
        return src[:k].copy(), dst[:k].copy()


# --------------------------------------------------------------------------- #
# bitdense / bitsparse
# --------------------------------------------------------------------------- #
def binarize(x: np.ndarray, word_bits: int = 32) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    rows, cols = x.shape
    out = np.empty((rows, spw(cols, word_bits)), dtype=np.uint32)
    lib().og_binarize(_ptr(x), rows, cols, word_bits, _ptr(out))
    return out


def l1_scales(x: np.ndarray, axis: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    rows, cols = x.shape
    out = np.empty(rows if axis == ROW else cols, dtype=np.float32)
    lib().og_l1_scales(_ptr(x), rows, cols, axis, _ptr(out))
    return out


def transpose_bits(bits: np.ndarray, rows: int, cols: int, word_bits: int = 32) -> np.ndarray:
    bits = np.ascontiguousarray(bits, dtype=np.uint32)
    out = np.empty((cols, spw(rows, word_bits)), dtype=np.uint32)
    lib().og_transpose_bits(_ptr(bits), rows, cols, word_bits, _ptr(out))
    return out


@dataclass
class Frdc:
    rows: int
    cols: int
    row_ptr: np.ndarray
    col_ind: np.ndarray
    tiles: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.tiles.shape[0])

    def nnz_bits(self) -> int:
        return int(np.unpackbits(self.tiles.view(np.uint8)).sum())

    def _c(self) -> _Frdc:
        s = _Frdc()
        s.rows, s.cols, s.nnz = self.rows, self.cols, self.nnz
        s.row_ptr = self.row_ptr.ctypes.data_as(C.POINTER(C.c_uint64))
        s.col_ind = self.col_ind.ctypes.data_as(C.POINTER(C.c_uint32))
        s.tiles = self.tiles.ctypes.data_as(C.POINTER(C.c_uint16))
        return s

    def row_popcounts(self) -> np.ndarray:
        deg = np.empty(self.rows, dtype=np.int64)
        s = self._c()
        lib().og_row_popcounts(C.byref(s), _ptr(deg))
        return deg


class TileSetC(C.Structure):
    """ref: TileSet (bitsparse.hpp:62-71); the layout of og_tileset / bg_tileset."""
    _fields_ = [("ts", C.c_int32), ("reserved", C.c_int32), ("rows", C.c_uint64 * 4),
                ("cols", C.c_uint32 * 16)]


PAD_COL = 0xFFFFFFFF


def tileset_count(m: Frdc, tile_row: int, word_bits: int = 32) -> int:
    s = m._c()
    return int(lib().og_tileset_count(C.byref(s), tile_row, word_bits))


def gather_tileset(m: Frdc, tile_row: int, set_index: int, word_bits: int = 32):
    """(ts, rows[4], cols[16]) of one tile set (bitsparse.cpp:136-160)."""
    s, t = m._c(), TileSetC()
    if lib().og_gather_tileset(C.byref(s), tile_row, set_index, word_bits, C.byref(t)):
        raise ValueError(_err())
    return t.ts, [int(v) for v in t.rows], [int(v) for v in t.cols]


def frdc_to_dense(m: Frdc, word_bits: int = 32) -> np.ndarray:
    """ZeroOne bits rows x spw(cols) (bitsparse.cpp:114-127)."""
    out = np.zeros((m.rows, spw(m.cols, word_bits)), np.uint32)
    s = m._c()
    lib().og_frdc_to_dense(C.byref(s), word_bits, _ptr(out))
    return out


def _frdc_copy(s: _Frdc) -> Frdc:
    tr = (s.rows + 3) // 4
    rp = np.ctypeslib.as_array(s.row_ptr, shape=(tr + 1,)).copy()
    if s.nnz:
        ci = np.ctypeslib.as_array(s.col_ind, shape=(s.nnz,)).copy()
        ti = np.ctypeslib.as_array(s.tiles, shape=(s.nnz,)).copy()
    else:
        ci = np.zeros(0, dtype=np.uint32)
        ti = np.zeros(0, dtype=np.uint16)
    return Frdc(s.rows, s.cols, rp, ci, ti)


def frdc_from_edges(n: int, src: np.ndarray, dst: np.ndarray, self_loops: bool) -> Frdc:
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    s = _Frdc()
    bad = C.c_int64(-1)
    rc = lib().og_frdc_from_edges(n, _ptr(src), _ptr(dst), src.shape[0], int(self_loops),
                                  C.byref(s), C.byref(bad))
    if rc:
        raise ValueError(f"edge {bad.value} out of range for {n} nodes")
    out = _frdc_copy(s)
    lib().og_frdc_free(C.byref(s))
    return out


# --------------------------------------------------------------------------- #
# kernels.cpp
# --------------------------------------------------------------------------- #
_OPS = {"BMM": BMM, "MM": BMM, "BSPMM": BSPMM, "ADD": ADD, "CONCAT": CONCAT}


def parse_variant(text: str) -> Tuple[int, int, int, int]:
    op, tags = text.split(".")
    p = [F if c in "Ff" else B for c in tags]
    return (_OPS[op.upper()], p[0], p[1], p[2])


def _variant(v) -> _Variant:
    if isinstance(v, str):
        v = parse_variant(v)
    return _Variant(*v)


@dataclass
class Mat:
    """F operand (f: float32 rows x cols) or B operand (bits: u32 rows x spw)."""
    prec: int
    rows: int
    cols: int
    word_bits: int = 32
    f: Optional[np.ndarray] = None
    bits: Optional[np.ndarray] = None
    scale: Optional[np.ndarray] = None

    @staticmethod
    def dense(x: np.ndarray) -> "Mat":
        x = np.ascontiguousarray(x, dtype=np.float32)
        return Mat(F, x.shape[0], x.shape[1], 32, f=x)

    @staticmethod
    def binary(bits: np.ndarray, rows: int, cols: int, word_bits: int = 32,
               scale: Optional[np.ndarray] = None) -> "Mat":
        return Mat(B, rows, cols, word_bits, bits=np.ascontiguousarray(bits, dtype=np.uint32),
                   scale=None if scale is None else np.ascontiguousarray(scale, dtype=np.float32))

    def _c(self) -> _Mat:
        m = _Mat()
        m.prec, m.rows, m.cols, m.word_bits = self.prec, self.rows, self.cols, self.word_bits
        if self.f is not None:
            m.f = self.f.ctypes.data_as(C.POINTER(C.c_float))
        if self.bits is not None:
            m.bits = self.bits.ctypes.data_as(C.POINTER(C.c_uint32))
        if self.scale is not None:
            m.scale = self.scale.ctypes.data_as(C.POINTER(C.c_float))
        return m


def _take(m: _Mat) -> Mat:
    if m.prec == F:
        f = np.ctypeslib.as_array(m.f, shape=(m.rows * m.cols,)).reshape(m.rows, m.cols).copy() \
            if m.rows * m.cols else np.zeros((m.rows, m.cols), np.float32)
        out = Mat(F, m.rows, m.cols, m.word_bits, f=f)
    else:
        n = m.rows * spw(m.cols, m.word_bits)
        bits = np.ctypeslib.as_array(m.bits, shape=(n,)).reshape(m.rows, -1).copy() \
            if n else np.zeros((m.rows, spw(m.cols, m.word_bits)), np.uint32)
        out = Mat(B, m.rows, m.cols, m.word_bits, bits=bits)
    lib().og_mat_free(C.byref(m))
    return out


def bmm(v, a: Mat, w: Mat, word_bits: int = 32) -> Mat:
    ca, cw, out = a._c(), w._c(), _Mat()
    if lib().og_bmm(_variant(v), C.byref(ca), C.byref(cw), word_bits, C.byref(out)):
        raise ValueError(_err())
    return _take(out)


def bspmm(v, adj: Frdc, x: Mat, row_scale: Optional[np.ndarray] = None,
          col_scale: Optional[np.ndarray] = None, word_bits: int = 32) -> Mat:
    cadj, cx, out = adj._c(), x._c(), _Mat()
    if lib().og_bspmm(_variant(v), C.byref(cadj), _ptr(row_scale), _ptr(col_scale), C.byref(cx),
                      word_bits, C.byref(out)):
        raise ValueError(_err())
    return _take(out)


def add(v, a: Mat, b: Mat) -> Mat:
    ca, cb, out = a._c(), b._c(), _Mat()
    if lib().og_add(_variant(v), C.byref(ca), C.byref(cb), C.byref(out)):
        raise ValueError(_err())
    return _take(out)


def softmax_rows(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(x)
    lib().og_softmax_rows(_ptr(x), x.shape[0], x.shape[1], _ptr(out))
    return out


# --------------------------------------------------------------------------- #
# graphops.cpp / modelconfig.cpp
# --------------------------------------------------------------------------- #
class Graph:
    """prepare_graph (graphops.cpp:146-170)."""

    def __init__(self, n: int, src: np.ndarray, dst: np.ndarray):
        self.n = n
        self._src = np.ascontiguousarray(src, dtype=np.int64)
        self._dst = np.ascontiguousarray(dst, dtype=np.int64)
        self._g = _Graph()
        if lib().og_prepare_graph(n, _ptr(self._src), _ptr(self._dst), self._src.shape[0],
                                  C.byref(self._g)):
            raise ValueError(_err())
        self.structure = _frdc_copy(self._g.structure)
        self.raw = _frdc_copy(self._g.raw)
        self.norm = np.ctypeslib.as_array(self._g.norm, shape=(n,)).copy() if n else np.zeros(0, np.float32)
        self.mean_row = np.ctypeslib.as_array(self._g.mean_row, shape=(n,)).copy() if n else np.zeros(0, np.float32)
        self.neighbor_count = np.ctypeslib.as_array(self._g.neighbor_count, shape=(n,)).copy() if n else np.zeros(0, np.int64)

    def __del__(self):
        try:
            lib().og_graph_free(C.byref(self._g))
        except Exception:
            pass


@dataclass
class Layer:
    kind: int
    plan: List[str] = field(default_factory=list)
    w1: Optional[np.ndarray] = None
    w2: Optional[np.ndarray] = None
    relu: bool = False


DEFAULT_PLANS = {  # modelconfig.cpp:49-60
    "gcn": ["MM.FBB+BSpMM.BBB", "MM.BBF+BSpMM.FBF"],
    "sage": ["MM.FBB+MM.FBB+BSpMM.BBB+ADD.BBF", "MM.FBF+MM.FBF+BSpMM.FFF+ADD.FFF"],
    "saint": ["MM.FBB+MM.FBB+BSpMM.BBB+ADD.BBF", "MM.FBB+MM.FBB+BSpMM.BBB+ADD.BBF", "MM.FBF"],
}


def build_model(model: str, features: int, hidden: int, classes: int, seed: int, nodes: int,
                plan: Optional[Sequence[str]] = None) -> Tuple[List[Layer], np.ndarray]:
    """build_model (modelconfig.cpp:99-173): X first, then W1 (and W2) per
    layer from one mt19937_64 stream; softmax appended."""
    plan = list(plan) if plan else DEFAULT_PLANS[model]
    rng = Rng(seed)
    X = rng.random_dense(nodes, features)

    def dims(n):
        d, fin = [], features
        for i in range(n):
            fout = classes if i + 1 == n else hidden
            d.append((fin, fout))
            fin = fout
        return d

    layers: List[Layer] = []
    if model == "gcn":
        dd = dims(len(plan))
        for i, chain in enumerate(plan):
            w1 = rng.random_dense(*dd[i])
            layers.append(Layer(GCN, chain.split("+"), w1, None, i + 1 < len(plan)))
    else:
        conv = len(plan) - 1 if model == "saint" else len(plan)
        dd = dims(conv + (1 if model == "saint" else 0))
        for i in range(conv):
            w1 = rng.random_dense(*dd[i])
            w2 = rng.random_dense(*dd[i])
            layers.append(Layer(SAGE if model == "sage" else GRAPHCONV, plan[i].split("+"), w1, w2, True))
        if model == "saint":
            layers.append(Layer(FC, plan[-1].split("+"), rng.random_dense(*dd[-1]), None, False))
        else:
            layers[-1].relu = False
    layers.append(Layer(SOFTMAX))
    return layers, X


@dataclass
class TracePoint:
    label: str
    bits: np.ndarray
    rows: int
    cols: int
    word_bits: int


def run_model(layers: Sequence[Layer], graph: Optional[Graph], x0: np.ndarray, word_bits: int = 32,
              trace: bool = True):
    """run_model (graphops.cpp:390-484).  Returns (out, logits, trace points)."""
    x0 = np.ascontiguousarray(x0, dtype=np.float32)
    cl = (_Layer * len(layers))()
    keep = []
    for i, l in enumerate(layers):
        cl[i].kind = l.kind
        cl[i].nplan = len(l.plan)
        for k, p in enumerate(l.plan):
            cl[i].plan[k] = _variant(p)
        for name in ("w1", "w2"):
            w = getattr(l, name)
            if w is not None:
                w = np.ascontiguousarray(w, dtype=np.float32)
                keep.append(w)
                setattr(cl[i], name, w.ctypes.data_as(C.POINTER(C.c_float)))
                setattr(cl[i], name + "_rows", w.shape[0])
                setattr(cl[i], name + "_cols", w.shape[1])
        cl[i].relu = int(l.relu)
    points: List[TracePoint] = []

    def sink(_ctx, label, bits, rows, cols, wb):
        n = rows * spw(cols, wb)
        arr = np.ctypeslib.as_array(bits, shape=(n,)).reshape(rows, -1).copy() if n else \
            np.zeros((rows, spw(cols, wb)), np.uint32)
        points.append(TracePoint(label.decode(), arr, rows, cols, wb))

    cb = _TRACE_FN(sink) if trace else _TRACE_FN()
    out_p, log_p = C.POINTER(C.c_float)(), C.POINTER(C.c_float)()
    oc = C.c_int64(0)
    gp = C.byref(graph._g) if graph is not None else None
    rc = lib().og_run_model(cl, len(layers), word_bits, gp, _ptr(x0), x0.shape[0], x0.shape[1],
                            C.byref(out_p), C.byref(log_p), C.byref(oc), cb, None)
    if rc:
        raise ValueError(_err())
    rows = x0.shape[0]
    out = np.ctypeslib.as_array(out_p, shape=(rows * oc.value,)).reshape(rows, -1).copy()
    logits = np.ctypeslib.as_array(log_p, shape=(rows * oc.value,)).reshape(rows, -1).copy()
    lib().og_free(C.cast(out_p, C.c_void_p))
    lib().og_free(C.cast(log_p, C.c_void_p))
    return out, logits, points


# --------------------------------------------------------------------------- #
# The real reference (oracle/_ref) -- present when built in the dev container.
# --------------------------------------------------------------------------- #
_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        L.ref_error.restype = C.c_char_p
        if hasattr(L, "ref_enumerate_plans"):
            L.ref_enumerate_plans.restype = C.c_int64
            L.ref_enumerate_plans.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_int64]
        L.ref_max_threads.restype = C.c_int
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_random_edges.restype = C.c_int64
        L.ref_random_edges.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
        L.ref_random_dense.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_void_p]
        L.ref_graph_create.restype = C.c_void_p
        L.ref_graph_create.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int64]
        L.ref_graph_free.argtypes = [C.c_void_p]
        L.ref_graph_from_frdc.restype = C.c_void_p
        L.ref_graph_from_frdc.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
        L.ref_graph_frdc.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int64),
                                     C.POINTER(C.POINTER(C.c_uint64)), C.POINTER(C.POINTER(C.c_uint32)),
                                     C.POINTER(C.POINTER(C.c_uint16))]
        L.ref_graph_scales.argtypes = [C.c_void_p, C.POINTER(C.POINTER(C.c_float)),
                                       C.POINTER(C.POINTER(C.c_float)), C.POINTER(C.POINTER(C.c_int64))]
        L.ref_model_build.restype = C.c_void_p
        L.ref_model_build.argtypes = [C.c_void_p, C.c_char_p, C.c_int64, C.c_int64, C.c_int64,
                                      C.c_uint64, C.c_int, C.c_char_p, C.c_int64]
        L.ref_model_free.argtypes = [C.c_void_p]
        L.ref_model_features.restype = C.POINTER(C.c_float)
        L.ref_model_features.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.ref_model_layers.argtypes = [C.c_void_p]
        L.ref_model_weight.restype = C.POINTER(C.c_float)
        L.ref_model_weight.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.ref_model_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                    C.c_void_p, _TRACE_FN, C.c_void_p]
        L.ref_model_time_forward.restype = C.c_double
        L.ref_model_time_forward.argtypes = [C.c_void_p]
        L.ref_model_kernel_times.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_int, C.c_void_p]
        L.ref_binarize.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p]
        _ref = L
    return _ref


def ref_random_edges(seed: int, nodes: int, m: int, allow_self: bool = False):
    src = np.empty(max(m, 1), np.int64)
    dst = np.empty(max(m, 1), np.int64)
    k = ref().ref_random_edges(seed, nodes, m, int(allow_self), _ptr(src), _ptr(dst))
    return src[:k].copy(), dst[:k].copy()


class _RefLayer(C.Structure):
    _fields_ = [("kind", C.c_int), ("plan", C.c_char_p),
                ("w1", C.c_void_p), ("w1_rows", C.c_int64), ("w1_cols", C.c_int64),
                ("w2", C.c_void_p), ("w2_rows", C.c_int64), ("w2_cols", C.c_int64),
                ("relu", C.c_int),
                ("bn_gamma", C.c_void_p), ("bn_beta", C.c_void_p), ("bn_mean", C.c_void_p),
                ("bn_sigma", C.c_void_p), ("bn_len", C.c_int64),
                ("scale_row", C.c_void_p), ("scale_row_len", C.c_int64),
                ("scale_col", C.c_void_p), ("scale_col_len", C.c_int64)]


def ref_spec_run(layers, graph: Optional["RefGraph"], x: np.ndarray, word_bits: int = 32):
    """Any layer list through the real reference's run_model (graphops.cpp:
    390-484).  `layers`: objects with kind (LayerKind order), plan (variant
    names), w1, w2, relu, bn (gamma, beta, mean, sigma), scale_row, scale_col.
    Returns (out, logits, trace points)."""
    arr = (_RefLayer * max(len(layers), 1))()
    keep = []

    def host(a):
        a = np.ascontiguousarray(a, dtype=np.float32)
        keep.append(a)
        return a

    for i, l in enumerate(layers):
        d = arr[i]
        d.kind = int(l.kind)
        plan = "+".join(str(p) if isinstance(p, str) else p.name() for p in (l.plan or []))
        keep.append(plan.encode())
        d.plan = keep[-1]
        for name in ("w1", "w2"):
            w = getattr(l, name, None)
            if w is not None:
                w = host(w)
                setattr(d, name, w.ctypes.data)
                setattr(d, name + "_rows", w.shape[0])
                setattr(d, name + "_cols", w.shape[1])
        d.relu = int(bool(getattr(l, "relu", False)))
        bn = getattr(l, "bn", None)
        if bn is not None:
            g, b, m, sg = (host(v) for v in bn)
            d.bn_gamma, d.bn_beta, d.bn_mean, d.bn_sigma = g.ctypes.data, b.ctypes.data, m.ctypes.data, sg.ctypes.data
            d.bn_len = g.shape[0]
        for name in ("scale_row", "scale_col"):
            v = getattr(l, name, None)
            if v is not None:
                v = host(v)
                setattr(d, name, v.ctypes.data)
                setattr(d, name + "_len", v.shape[0])
    x = np.ascontiguousarray(x, dtype=np.float32)
    points: List[TracePoint] = []

    def sink(_ctx, label, bits, r, c, wb):
        n = r * spw(c, wb)
        a = np.ctypeslib.as_array(bits, shape=(n,)).reshape(r, -1).copy() if n else \
            np.zeros((r, spw(c, wb)), np.uint32)
        points.append(TracePoint(label.decode(), a, r, c, wb))

    cb = _TRACE_FN(sink)
    out_p, log_p, oc = C.POINTER(C.c_float)(), C.POINTER(C.c_float)(), C.c_int64(0)
    L = ref()
    L.ref_spec_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_int64,
                               C.c_void_p, C.c_void_p, C.c_void_p, _TRACE_FN, C.c_void_p]
    L.ref_free.argtypes = [C.c_void_p]
    rc = L.ref_spec_run(graph.h if graph is not None else None, arr, len(layers), word_bits, _ptr(x),
                        x.shape[0], x.shape[1], C.byref(out_p), C.byref(log_p), C.byref(oc), cb, None)
    if rc:
        raise ValueError(L.ref_error().decode())
    rows = x.shape[0]
    out = np.ctypeslib.as_array(out_p, shape=(max(rows * oc.value, 1),))[:rows * oc.value].reshape(rows, -1).copy()
    lg = np.ctypeslib.as_array(log_p, shape=(max(rows * oc.value, 1),))[:rows * oc.value].reshape(rows, -1).copy()
    L.ref_free(C.cast(out_p, C.c_void_p))
    L.ref_free(C.cast(log_p, C.c_void_p))
    return out, lg, points


def ref_layer_run(graph: "RefGraph", layer, x, word_bits: int = 32, prefix: str = "", x_word_bits: int = 32):
    """One layer through the real reference's gcn_layer / sage_layer /
    graphconv_layer (graphops.cpp:270-335) by layer.kind (0 / 1 / 2).  x: a
    float32 matrix, or (bits u32 [rows, spw], rows, cols) for a binary input.
    Returns (result, trace points): result is float32 rows x cols for an F
    output, else (bits, rows, cols, word_bits)."""
    arr = (_RefLayer * 1)()
    d = arr[0]
    keep = []
    d.kind = int(layer.kind)
    plan = "+".join(str(p) if isinstance(p, str) else p.name() for p in (layer.plan or []))
    keep.append(plan.encode())
    d.plan = keep[-1]
    for name in ("w1", "w2"):
        w = getattr(layer, name, None)
        if w is not None:
            w = np.ascontiguousarray(w, dtype=np.float32)
            keep.append(w)
            setattr(d, name, w.ctypes.data)
            setattr(d, name + "_rows", w.shape[0])
            setattr(d, name + "_cols", w.shape[1])
    d.relu = int(bool(getattr(layer, "relu", False)))
    if isinstance(x, tuple):
        bits, rows, cols = x
        xa, prec = np.ascontiguousarray(bits, dtype=np.uint32), 1
    else:
        xa, prec = np.ascontiguousarray(x, dtype=np.float32), 0
        rows, cols = xa.shape
    points: List[TracePoint] = []

    def sink(_ctx, label, bits, r, c, wb):
        n = r * spw(c, wb)
        a = np.ctypeslib.as_array(bits, shape=(n,)).reshape(r, -1).copy() if n else \
            np.zeros((r, spw(c, wb)), np.uint32)
        points.append(TracePoint(label.decode(), a, r, c, wb))

    cb = _TRACE_FN(sink)
    L = ref()
    L.ref_layer_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_int64,
                                C.c_int, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_void_p),
                                C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int), _TRACE_FN,
                                C.c_void_p]
    L.ref_free.argtypes = [C.c_void_p]
    op, outp, r, c, wb = C.c_int(), C.c_void_p(), C.c_int64(), C.c_int64(), C.c_int()
    if L.ref_layer_run(graph.h, arr, word_bits, prec, _ptr(xa), rows, cols, x_word_bits, prefix.encode(),
                       C.byref(op), C.byref(outp), C.byref(r), C.byref(c), C.byref(wb), cb, None):
        raise ValueError(L.ref_error().decode())
    try:
        if op.value == 0:
            n = r.value * c.value
            res = np.ctypeslib.as_array(C.cast(outp, C.POINTER(C.c_float)), shape=(max(n, 1),))[:n] \
                .reshape(r.value, c.value).copy()
        else:
            n = r.value * spw(c.value, wb.value)
            bits = np.ctypeslib.as_array(C.cast(outp, C.POINTER(C.c_uint32)), shape=(max(n, 1),))[:n] \
                .reshape(r.value, -1).copy()
            res = (bits, r.value, c.value, wb.value)
    finally:
        L.ref_free(outp)
    return res, points


def ref_oracle_run(graph: "RefGraph", model: "RefModel", full_precision: bool = False, word_bits: int = 32):
    """The reference's dense oracle::run_model (oracle.cpp:194-317): (trace
    points as packed sign bits, logits float64).  O(N^2) memory: small graphs."""
    L = ref()
    L.ref_oracle_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, _TRACE_FN, C.c_void_p,
                                 C.POINTER(C.POINTER(C.c_double)), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.ref_free.argtypes = [C.c_void_p]
    points: List[TracePoint] = []

    def sink(_ctx, label, bits, r, c, wb):
        n = r * spw(c, wb)
        a = np.ctypeslib.as_array(bits, shape=(n,)).reshape(r, -1).copy() if n else \
            np.zeros((r, spw(c, wb)), np.uint32)
        points.append(TracePoint(label.decode(), a, r, c, wb))

    cb = _TRACE_FN(sink)
    lp, r, c = C.POINTER(C.c_double)(), C.c_int64(), C.c_int64()
    if L.ref_oracle_run(graph.h, model.h, int(full_precision), word_bits, cb, None, C.byref(lp), C.byref(r),
                        C.byref(c)):
        raise ValueError(L.ref_error().decode())
    n = r.value * c.value
    lg = np.ctypeslib.as_array(lp, shape=(max(n, 1),))[:n].reshape(r.value, c.value).copy()
    L.ref_free(C.cast(lp, C.c_void_p))
    return points, lg


def ref_verify_model(graph: "RefGraph", model: "RefModel", full_precision: bool = False,
                     tolerance: float = 1e-6, corrupt_tile: int = -1) -> dict:
    """The reference's own verify_model (runreport.cpp:51-135) report."""
    L = ref()
    L.ref_verify_model.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_int64,
                                   C.POINTER(C.c_double), C.c_void_p, C.c_char_p, C.c_int,
                                   C.POINTER(C.c_double), C.POINTER(C.c_int)]
    mr, ag, ok = C.c_double(), C.c_double(), C.c_int()
    counts = np.zeros(5, np.int64)
    lab = C.create_string_buffer(128)
    if L.ref_verify_model(graph.h, model.h, int(full_precision), tolerance, corrupt_tile, C.byref(mr),
                          _ptr(counts), lab, 128, C.byref(ag), C.byref(ok)):
        raise ValueError(L.ref_error().decode())
    return {"max_rel_logit_error": mr.value, "bin_points": int(counts[0]), "bin_values": int(counts[1]),
            "bin_mismatches": int(counts[2]), "first_mismatch_row": int(counts[3]),
            "first_mismatch_col": int(counts[4]), "first_mismatch_label": lab.value.decode(),
            "argmax_agreement": ag.value, "pass": bool(ok.value)}


def ref_read_graph(kind: int, text, name: str = "<stream>", forced_nodes: int = -1, undirected: bool = False):
    """The reference's graphio readers (kind 0 read_edge_list, 1
    read_matrix_market, 2 load_graph(path=text)).  Returns (node_count, src,
    dst, weights) or raises ValueError with the reference's message."""
    b = text.encode() if isinstance(text, str) else bytes(text)
    L = ref()
    L.ref_read_graph.argtypes = [C.c_int, C.c_char_p, C.c_size_t, C.c_char_p, C.c_int64, C.c_int,
                                 C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.POINTER(C.c_int64)),
                                 C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.c_int64),
                                 C.POINTER(C.POINTER(C.c_double))]
    L.ref_free.argtypes = [C.c_void_p]
    n, m, nw = C.c_int64(), C.c_int64(), C.c_int64()
    sp, dp, wp = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)(), C.POINTER(C.c_double)()
    rc = L.ref_read_graph(kind, b, len(b), name.encode(), forced_nodes, int(undirected), C.byref(n), C.byref(m),
                          C.byref(sp), C.byref(dp), C.byref(nw), C.byref(wp))
    if rc:
        raise ValueError(L.ref_error().decode())
    try:
        src = np.ctypeslib.as_array(sp, shape=(max(m.value, 1),))[:m.value].copy()
        dst = np.ctypeslib.as_array(dp, shape=(max(m.value, 1),))[:m.value].copy()
        w = np.ctypeslib.as_array(wp, shape=(max(nw.value, 1),))[:nw.value].copy()
    finally:
        for p in (sp, dp, wp):
            L.ref_free(C.cast(p, C.c_void_p))
    return n.value, src, dst, w


class RefGraph:
    @staticmethod
    def from_frdc(n: int, loops: "Frdc", raw: "Frdc") -> "RefGraph":
        g = RefGraph.__new__(RefGraph)
        g.n = n
        a = [np.ascontiguousarray(x) for x in (loops.row_ptr, loops.col_ind, loops.tiles,
                                               raw.row_ptr, raw.col_ind, raw.tiles)]
        g.h = ref().ref_graph_from_frdc(n, _ptr(a[0]), _ptr(a[1]), _ptr(a[2]), loops.nnz,
                                        _ptr(a[3]), _ptr(a[4]), _ptr(a[5]), raw.nnz)
        if not g.h:
            raise ValueError(ref().ref_error().decode())
        return g

    def __init__(self, n: int, src: np.ndarray, dst: np.ndarray):
        src = np.ascontiguousarray(src, dtype=np.int64)
        dst = np.ascontiguousarray(dst, dtype=np.int64)
        self.n = n
        self.h = ref().ref_graph_create(n, _ptr(src), _ptr(dst), src.shape[0])
        if not self.h:
            raise ValueError(ref().ref_error().decode())

    def frdc(self, which: int) -> Frdc:
        nnz = C.c_int64()
        rp, ci, ti = C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint16)()
        ref().ref_graph_frdc(self.h, which, C.byref(nnz), C.byref(rp), C.byref(ci), C.byref(ti))
        tr = (self.n + 3) // 4
        s = _Frdc(self.n, self.n, nnz.value, rp, ci, ti)
        return _frdc_copy(s)

    def scales(self):
        a, b, c = C.POINTER(C.c_float)(), C.POINTER(C.c_float)(), C.POINTER(C.c_int64)()
        ref().ref_graph_scales(self.h, C.byref(a), C.byref(b), C.byref(c))
        n = self.n
        return (np.ctypeslib.as_array(a, shape=(n,)).copy(), np.ctypeslib.as_array(b, shape=(n,)).copy(),
                np.ctypeslib.as_array(c, shape=(n,)).copy())

    def __del__(self):
        try:
            if self.h:
                ref().ref_graph_free(self.h)
        except Exception:
            pass


class RefModel:
    def __init__(self, graph: Optional[RefGraph], model: str, features: int, hidden: int,
                 classes: int, seed: int, nodes: int, word_bits: int = 32,
                 plan: Optional[Sequence[str]] = None):
        p = "|".join(plan) if plan else ""
        self.h = ref().ref_model_build(graph.h if graph else None, model.encode(), features, hidden,
                                       classes, seed, word_bits, p.encode(), nodes)
        if not self.h:
            raise ValueError(ref().ref_error().decode())
        self.graph = graph

    def features(self) -> np.ndarray:
        r, c = C.c_int64(), C.c_int64()
        p = ref().ref_model_features(self.h, C.byref(r), C.byref(c))
        return np.ctypeslib.as_array(p, shape=(r.value * c.value,)).reshape(r.value, c.value).copy()

    def weights(self):
        out = []
        for i in range(ref().ref_model_layers(self.h)):
            ws = []
            for which in (1, 2):
                r, c = C.c_int64(), C.c_int64()
                p = ref().ref_model_weight(self.h, i, which, C.byref(r), C.byref(c))
                ws.append(None if not p else
                          np.ctypeslib.as_array(p, shape=(r.value * c.value,)).reshape(r.value, c.value).copy())
            out.append(tuple(ws))
        return out

    def run(self, out_cols: int, x: Optional[np.ndarray] = None, trace: bool = True):
        rows = self.features().shape[0] if x is None else x.shape[0]
        logits = np.empty((rows, out_cols), np.float32)
        out = np.empty((rows, out_cols), np.float32)
        points: List[TracePoint] = []

        def sink(_ctx, label, bits, r, c, wb):
            n = r * spw(c, wb)
            arr = np.ctypeslib.as_array(bits, shape=(n,)).reshape(r, -1).copy() if n else \
                np.zeros((r, spw(c, wb)), np.uint32)
            points.append(TracePoint(label.decode(), arr, r, c, wb))

        cb = _TRACE_FN(sink) if trace else _TRACE_FN()
        xp = None
        if x is not None:
            x = np.ascontiguousarray(x, dtype=np.float32)
            xp = _ptr(x)
        rc = ref().ref_model_run(self.h, xp, rows, 0 if x is None else x.shape[1],
                                 _ptr(logits), _ptr(out), cb, None)
        if rc:
            raise ValueError(ref().ref_error().decode())
        return out, logits, points

    def time_forward(self) -> float:
        return ref().ref_model_time_forward(self.h)

    def kernel_times(self):
        cap, ll = 64, 96
        labels = C.create_string_buffer(cap * ll)
        ms = np.zeros(cap, np.float64)
        n = ref().ref_model_kernel_times(self.h, cap, labels, ll, _ptr(ms))
        raw = labels.raw
        return [(raw[i * ll:(i + 1) * ll].split(b"\0")[0].decode(), float(ms[i])) for i in range(max(n, 0))]

    def __del__(self):
        try:
            if self.h:
                ref().ref_model_free(self.h)
        except Exception:
            pass


def ref_bench_bspmm_bbb(nodes: int = 65536, density: float = 0.001, cols: int = 128, seed: int = 7,
                        word_bits: int = 32) -> dict:
    """The reference's own single-thread kernelbench (kernelbench.cpp:110-186):
    BSpMM.BBB vs a naive CSR SpMM.  GTEPS = adjacency bits / engine time."""
    L = ref()
    em, bm = C.c_double(), C.c_double()
    edges, match = C.c_int64(), C.c_int()
    L.ref_bench_bspmm_bbb.argtypes = [C.c_int64, C.c_double, C.c_int64, C.c_uint64, C.c_int,
                                      C.POINTER(C.c_double), C.POINTER(C.c_double),
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int)]
    if L.ref_bench_bspmm_bbb(nodes, density, cols, seed, word_bits, C.byref(em), C.byref(bm),
                             C.byref(edges), C.byref(match)):
        raise RuntimeError(L.ref_error().decode())
    return {"nodes": nodes, "density": density, "features": cols, "edges": edges.value,
            "engine_ms": em.value, "naive_csr_ms": bm.value, "values_match": bool(match.value),
            "gteps": edges.value / (em.value * 1e-3) / 1e9 if em.value > 0 else None,
            "threads": 1}


def ref_gather_tileset(m: Frdc, tile_row: int, set_index: int, word_bits: int = 32):
    """The real reference's gather_tileset (bitsparse.cpp:136-160)."""
    L = ref()
    ts = C.c_int32()
    rows = (C.c_uint64 * 4)()
    cols = (C.c_uint32 * 16)()
    if L.ref_gather_tileset(C.c_int64(m.rows), C.c_int64(m.cols), _ptr(m.row_ptr), _ptr(m.col_ind),
                            _ptr(m.tiles), C.c_int64(m.nnz), C.c_int64(tile_row), C.c_int64(set_index),
                            C.c_int(word_bits), C.byref(ts), rows, cols):
        raise ValueError(L.ref_error().decode())
    return ts.value, [int(v) for v in rows], [int(v) for v in cols]


def ref_frdc_to_dense(m: Frdc, word_bits: int = 32) -> np.ndarray:
    L = ref()
    out = np.zeros((m.rows, spw(m.cols, word_bits)), np.uint32)
    if L.ref_frdc_to_dense(C.c_int64(m.rows), C.c_int64(m.cols), _ptr(m.row_ptr), _ptr(m.col_ind),
                           _ptr(m.tiles), C.c_int64(m.nnz), C.c_int(word_bits), _ptr(out)):
        raise ValueError(L.ref_error().decode())
    return out


def ref_enumerate_plans(model: str, layers: int):
    """The real reference's enumerate_plans for a model skeleton (tune.cpp)."""
    L = ref()
    buf = C.create_string_buffer(1 << 22)
    n = L.ref_enumerate_plans(model.encode(), layers, buf, len(buf))
    if n < 0:
        raise RuntimeError(L.ref_error().decode())
    return [line.split("|") for line in buf.value.decode().splitlines()]
