"""Python host mirror of the reference operator API (proj/include/bitgnn).

Same names, argument meaning and error behaviour as the C++ reference, over
the B200 C ABI (include/bitgnn_b200.h).  Dense operands are CUDA fp32
``torch.Tensor``s, binary operands are :class:`BitOperand` (packed u32 words
held in an int32 CUDA tensor with the reference layout).  Errors raise
:class:`InvalidArgument` (std::invalid_argument), :class:`RuntimeFailure`
(std::runtime_error) or :class:`LogicError` (std::logic_error).

Reference map:
  binarize / binarize_with_scale / unpack / transpose  -> bitdense.hpp:110-141
  frdc_from_edges / FrdcMatrix                        -> bitsparse.hpp:26-81
  KernelVariant / bmm / bspmm / add / concat / ...     -> kernels.hpp:19-97
  prepare_graph / LayerSpec / ModelSpec / run_model    -> graphops.hpp:40-133
  Rng / random_dense / random_edges                    -> rng.hpp:16-80
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple, Union

import numpy as np
import torch

from . import _lib as L
from ._lib import (AND_ANDNOT, B, F, IF_ELSE, PLUS_MINUS, TWO_AND_MINUS_POPC, ZERO_ONE,
                   CudaError, InvalidArgument, LogicError, RuntimeFailure, check, lib)

Precision = int
ROW, COL = L.AXIS_ROW, L.AXIS_COL


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def set_aggregation(mode: int, window_nodes: int = 0) -> None:
    """Process-wide aggregation layout (L.AGG_AUTO / AGG_SLIVERS / AGG_TILES /
    AGG_WINDOW).  Every layout gives identical results; window_nodes > 0 sets
    the shared-memory window size of the windowed BBB kernel (tests)."""
    L.check(L.lib().bg_set_aggregation(int(mode), int(window_nodes)))


def set_persistent(enable: bool) -> None:
    """Whole-forward persistent kernel for small binary GCN chains (opt-in;
    identical results, see bg_set_persistent)."""
    L.check(L.lib().bg_set_persistent(int(enable)))


def get_aggregation() -> Tuple[int, int]:
    m, w = C.c_int(), C.c_int()
    L.check(L.lib().bg_get_aggregation(C.byref(m), C.byref(w)))
    return m.value, w.value


def storage_words_per_row(cols: int, word_bits: int) -> int:
    return (cols + word_bits - 1) // word_bits * (word_bits // 32)


class _CAI:
    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


def device_view(ptr: int, shape, typestr: str) -> torch.Tensor:
    """Zero-copy torch view of library-owned device memory."""
    if int(np.prod(shape)) == 0:
        dt = {"<f4": torch.float32, "<i4": torch.int32, "<i8": torch.int64, "<i2": torch.int16}[typestr]
        return torch.empty(tuple(shape), dtype=dt, device="cuda")
    return torch.as_tensor(_CAI(ptr, shape, typestr), device="cuda")


# --------------------------------------------------------------------------- #
# KernelVariant (kernels.hpp:23-33)
# --------------------------------------------------------------------------- #
@dataclass(frozen=True)
class KernelVariant:
    op: int = L.BMM
    in1: int = B
    in2: int = B
    out: int = B

    @staticmethod
    def parse(text: str) -> "KernelVariant":
        v = L.Variant()
        check(lib().bg_variant_parse(text.encode(), C.byref(v)))
        return KernelVariant(v.op, v.in1, v.in2, v.out)

    def valid(self) -> bool:
        return bool(lib().bg_variant_valid(self._c()))

    def name(self) -> str:
        buf = C.create_string_buffer(32)
        check(lib().bg_variant_name(self._c(), buf, 32))
        return buf.value.decode()

    def _c(self) -> L.Variant:
        return L.Variant(self.op, self.in1, self.in2, self.out)

    def __str__(self) -> str:
        return self.name()


def _v(v) -> KernelVariant:
    return KernelVariant.parse(v) if isinstance(v, str) else v


# --------------------------------------------------------------------------- #
# Bit matrices (bitdense.hpp)
# --------------------------------------------------------------------------- #
@dataclass
class BitDenseMatrix:
    """Packed rows on the device: ``words`` is int32 [rows, spw] holding the
    reference's MSB-first u32 words."""
    words: torch.Tensor
    rows: int
    cols: int
    word_bits: int = 32
    semantics: int = PLUS_MINUS

    @staticmethod
    def empty(rows: int, cols: int, word_bits: int = 32, semantics: int = PLUS_MINUS):
        if word_bits not in (32, 64):
            raise InvalidArgument("BitDenseMatrix: word_bits must be 32 or 64")
        w = torch.zeros((rows, storage_words_per_row(cols, word_bits)), dtype=torch.int32, device="cuda")
        return BitDenseMatrix(w, rows, cols, word_bits, semantics)

    @staticmethod
    def from_numpy(words: np.ndarray, rows: int, cols: int, word_bits: int = 32,
                   semantics: int = PLUS_MINUS) -> "BitDenseMatrix":
        w = torch.from_numpy(np.ascontiguousarray(words, dtype=np.uint32).view(np.int32)).cuda()
        return BitDenseMatrix(w.reshape(rows, storage_words_per_row(cols, word_bits)), rows, cols,
                              word_bits, semantics)

    @property
    def storage_words_per_row(self) -> int:
        return storage_words_per_row(self.cols, self.word_bits)

    def numpy(self) -> np.ndarray:
        return self.words.cpu().numpy().view(np.uint32).reshape(self.rows, self.storage_words_per_row)

    def bit(self, i: int, j: int) -> bool:
        return bool((int(self.numpy()[i, j // 32]) >> (31 - (j & 31))) & 1)

    def payload_bytes(self) -> int:
        return self.rows * self.storage_words_per_row * 4

    def __eq__(self, o) -> bool:
        return (isinstance(o, BitDenseMatrix) and self.rows == o.rows and self.cols == o.cols and
                self.word_bits == o.word_bits and self.semantics == o.semantics and
                torch.equal(self.words, o.words))


@dataclass
class BitOperand:
    """kernels.hpp:37-40 -- packed bits plus an optional reconstruction scale."""
    bits: BitDenseMatrix
    scale: Optional[torch.Tensor] = None
    scale_axis: int = ROW


MatOperand = Union[torch.Tensor, BitOperand]


def _mat(m: MatOperand, scale_axis: int = ROW) -> L.Mat:
    c = L.Mat()
    if isinstance(m, BitOperand):
        c.precision = B
        c.word_bits = m.bits.word_bits
        c.semantics = m.bits.semantics
        c.rows, c.cols = m.bits.rows, m.bits.cols
        words = m.bits.words.contiguous()
        sc = _vec(m.scale)
        c.data = words.data_ptr()
        c.scale = sc.data_ptr() if sc is not None else None
        c.scale_axis = m.scale_axis
        c._keep = (words, sc)  # alive as long as the descriptor (the C call reads them)
    elif isinstance(m, BitDenseMatrix):
        return _mat(BitOperand(m))
    else:
        t = _dense(m)
        c.precision = F
        c.word_bits = 32
        c.rows, c.cols = t.shape
        c.data = t.data_ptr()
        c._keep = (t,)  # a non-contiguous input's contiguous copy must outlive the call
    return c


def _vec(t: Optional[torch.Tensor]) -> Optional[torch.Tensor]:
    """A scale vector as the C ABI reads it: contiguous float32 on the device."""
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or not t.is_cuda:
        raise InvalidArgument("scale vectors are float32 CUDA tensors")
    return t.contiguous()


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _dense(t: torch.Tensor) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or not t.is_cuda or t.dim() != 2:
        raise InvalidArgument("dense operands are 2-D float32 CUDA tensors")
    return t.contiguous()


def _alloc(desc: L.Mat) -> Tuple[MatOperand, L.Mat]:
    if desc.precision == F:
        t = torch.empty((desc.rows, desc.cols), dtype=torch.float32, device="cuda")
        desc.data = t.data_ptr()
        return t, desc
    bm = BitDenseMatrix.empty(desc.rows, desc.cols, desc.word_bits)
    desc.data = bm.words.data_ptr()
    return BitOperand(bm), desc


def binarize(x: torch.Tensor, word_bits: int = 32) -> BitDenseMatrix:
    """bitdense.cpp:71-88 -- sign(x) with sign(0) = +1, PlusMinus bits."""
    x = _dense(x)
    out = BitDenseMatrix.empty(x.shape[0], x.shape[1], word_bits)
    check(lib().bg_binarize(x.data_ptr(), x.shape[0], x.shape[1], word_bits, out.words.data_ptr(), _stream()))
    return out


def binarize_with_scale(x: torch.Tensor, axis: int, word_bits: int = 32):
    """bitdense.cpp:90-104 -- bits plus mean-|x| row or column scale."""
    x = _dense(x)
    out = BitDenseMatrix.empty(x.shape[0], x.shape[1], word_bits)
    sc = torch.empty(x.shape[0] if axis == ROW else x.shape[1], dtype=torch.float32, device="cuda")
    check(lib().bg_binarize_with_scale(x.data_ptr(), x.shape[0], x.shape[1], axis, word_bits,
                                       out.words.data_ptr(), sc.data_ptr(), _stream()))
    return out, sc


def unpack(m: BitDenseMatrix) -> torch.Tensor:
    out = torch.empty((m.rows, m.cols), dtype=torch.float32, device="cuda")
    check(lib().bg_unpack(m.words.data_ptr(), m.rows, m.cols, m.word_bits, m.semantics, out.data_ptr(), _stream()))
    return out


def transpose(m: BitDenseMatrix) -> BitDenseMatrix:
    out = BitDenseMatrix.empty(m.cols, m.rows, m.word_bits, m.semantics)
    check(lib().bg_transpose(m.words.data_ptr(), m.rows, m.cols, m.word_bits, out.words.data_ptr(), _stream()))
    return out


# --------------------------------------------------------------------------- #
# FRDC (bitsparse.hpp)
# --------------------------------------------------------------------------- #
class FrdcMatrix:
    """Device-resident FRDC bit-tile matrix (owning handle)."""

    def __init__(self, handle: int, owner=None):
        self._h = C.c_void_p(handle)
        self._owner = owner  # graph bundle that owns a borrowed structure

    @staticmethod
    def from_host(node_rows: int, node_cols: int, row_ptr, col_ind, tiles) -> "FrdcMatrix":
        rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
        ci = np.ascontiguousarray(col_ind, dtype=np.uint32)
        ti = np.ascontiguousarray(tiles, dtype=np.uint16)
        if rp.shape[0] != (node_rows + 3) // 4 + 1:
            raise InvalidArgument("FRDC: row_ptr length mismatch")
        if ci.shape[0] != ti.shape[0]:
            raise InvalidArgument("FRDC: offsets do not match payload")
        h = C.c_void_p()
        check(lib().bg_frdc_from_host(node_rows, node_cols, rp.ctypes.data, ci.ctypes.data,
                                      ti.ctypes.data, ti.shape[0], C.byref(h), _stream()))
        return FrdcMatrix(h.value)

    def info(self) -> L.FrdcInfo:
        i = L.FrdcInfo()
        check(lib().bg_frdc_info_get(self._h, C.byref(i)))
        return i

    @property
    def node_rows(self) -> int:
        return self.info().node_rows

    @property
    def node_cols(self) -> int:
        return self.info().node_cols

    @property
    def tile_rows(self) -> int:
        return self.info().tile_rows

    @property
    def nnz_tiles(self) -> int:
        return self.info().nnz_tiles

    @property
    def nnz_bits(self) -> int:
        return self.info().nnz_bits

    def payload_bytes(self) -> int:
        i = self.info()
        return (i.tile_rows + 1) * 8 + i.nnz_tiles * 6

    def download(self):
        """(row_ptr u64, col_ind u32, tiles u16) as host numpy arrays."""
        i = self.info()
        rp = np.empty(i.tile_rows + 1, np.uint64)
        ci = np.empty(max(i.nnz_tiles, 1), np.uint32)
        ti = np.empty(max(i.nnz_tiles, 1), np.uint16)
        check(lib().bg_frdc_download(self._h, rp.ctypes.data, ci.ctypes.data, ti.ctypes.data))
        return rp, ci[:i.nnz_tiles], ti[:i.nnz_tiles]

    def degree(self) -> torch.Tensor:
        i = self.info()
        return device_view(i.degree, (i.node_rows,), "<i4")

    # -- container I/O (ref: write_frdc / read_frdc, bitsparse.cpp:171-222) --
    def to_bytes(self, word_bits: int = 32) -> bytes:
        n = C.c_size_t()
        check(lib().bg_frdc_serialized_size(self._h, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        check(lib().bg_frdc_serialize(self._h, word_bits, buf, n.value))
        return bytes(buf)

    @staticmethod
    def from_bytes(data: bytes) -> Tuple["FrdcMatrix", int]:
        h, wb = C.c_void_p(), C.c_int()
        check(lib().bg_frdc_deserialize(data, len(data), C.byref(h), C.byref(wb), _stream()))
        return FrdcMatrix(h.value), wb.value

    def write(self, path: str, word_bits: int = 32) -> None:
        check(lib().bg_frdc_write_file(self._h, word_bits, str(path).encode()))

    @staticmethod
    def read(path: str) -> Tuple["FrdcMatrix", int]:
        h, wb = C.c_void_p(), C.c_int()
        check(lib().bg_frdc_read_file(str(path).encode(), C.byref(h), C.byref(wb), _stream()))
        return FrdcMatrix(h.value), wb.value

    def corrupt_tile(self, k: int) -> None:
        check(lib().bg_frdc_corrupt_tile(self._h, k))

    def __del__(self):
        try:
            if self._owner is None and self._h:
                lib().bg_frdc_destroy(self._h)
        except Exception:
            pass


@dataclass
class EdgeList:
    """ref: EdgeList (bitsparse.hpp) -- node count, (src, dst) pairs and the
    optional weight column (possibly shorter than the edges, as in the
    reference: it is padded with 1.0 only up to the last weighted line)."""
    node_count: int
    src: np.ndarray
    dst: np.ndarray
    weights: np.ndarray


def _take_edges(h: C.c_void_p) -> EdgeList:
    try:
        n, m, nw = C.c_int64(), C.c_int64(), C.c_int64()
        sp, dp, wp = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib().bg_edges_info(h, C.byref(n), C.byref(m), C.byref(sp), C.byref(dp), C.byref(wp), C.byref(nw)))

        def arr(p, k, t):
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(t)), shape=(k,)).copy() if k else \
                np.zeros(0, np.int64 if t is C.c_int64 else np.float64)
        return EdgeList(n.value, arr(sp.value, m.value, C.c_int64), arr(dp.value, m.value, C.c_int64),
                        arr(wp.value, nw.value, C.c_double))
    finally:
        lib().bg_edges_destroy(h)


def _text(t) -> bytes:
    return t.encode() if isinstance(t, str) else bytes(t)


def read_edge_list(text, name: str = "<stream>", forced_nodes: int = -1, undirected: bool = False) -> EdgeList:
    """graphio.cpp:72-99: whitespace 'src dst [weight]' lines, 0-based."""
    b = _text(text)
    h = C.c_void_p()
    check(lib().bg_read_edge_list(b, len(b), name.encode(), forced_nodes, int(undirected), C.byref(h)))
    return _take_edges(h)


def read_matrix_market(text, name: str = "<stream>", undirected: bool = False) -> EdgeList:
    """graphio.cpp:101-155: MatrixMarket coordinate, weights dropped."""
    b = _text(text)
    h = C.c_void_p()
    check(lib().bg_read_matrix_market(b, len(b), name.encode(), int(undirected), C.byref(h)))
    return _take_edges(h)


def load_graph(path: str, forced_nodes: int = -1, undirected: bool = False) -> EdgeList:
    """graphio.cpp:157-176: FRDC container, MatrixMarket or edge list by sniffing."""
    h = C.c_void_p()
    check(lib().bg_load_graph(str(path).encode(), forced_nodes, int(undirected), C.byref(h)))
    return _take_edges(h)


def _edges(src, dst) -> Tuple[torch.Tensor, torch.Tensor]:
    s = torch.as_tensor(np.asarray(src, dtype=np.int64) if not isinstance(src, torch.Tensor) else src)
    d = torch.as_tensor(np.asarray(dst, dtype=np.int64) if not isinstance(dst, torch.Tensor) else dst)
    return s.to(device="cuda", dtype=torch.int64).contiguous(), d.to(device="cuda", dtype=torch.int64).contiguous()


def frdc_from_edges(node_count: int, src, dst, add_self_loops: bool) -> FrdcMatrix:
    """bitsparse.cpp:72-112, built on the device."""
    s, d = _edges(src, dst)
    h = C.c_void_p()
    check(lib().bg_frdc_from_edges(s.data_ptr(), d.data_ptr(), s.shape[0], node_count,
                                   int(add_self_loops), C.byref(h), _stream()))
    return FrdcMatrix(h.value)


# --------------------------------------------------------------------------- #
# Tile sets, dense expansion, statistics (bitsparse.hpp:62-90)
# --------------------------------------------------------------------------- #
PAD_COL = 0xFFFFFFFF  # TileSet::kPadCol


@dataclass
class TileSet:
    """bitsparse.hpp:66-71 -- ts tiles' nibble rows concatenated into 4 words."""
    ts: int = 8
    rows: Tuple[int, int, int, int] = (0, 0, 0, 0)
    cols: Tuple[int, ...] = (PAD_COL,) * 16


@dataclass
class FrdcStats:
    """bitsparse.hpp:83-88"""
    nnz_tiles: int = 0
    nnz_bits: int = 0
    bytes: int = 0
    fill_ratio: float = 0.0


def tileset_count(m: FrdcMatrix, tile_row: int, word_bits: int = 32) -> int:
    """bitsparse.cpp:129-134"""
    n = C.c_int64()
    check(lib().bg_tileset_count(m._h, tile_row, word_bits, C.byref(n)))
    return n.value


def gather_tileset(m: FrdcMatrix, tile_row: int, set_index: int, word_bits: int = 32) -> TileSet:
    """bitsparse.cpp:136-160 (the reference's checks and messages)."""
    t = L.TileSetC()
    check(lib().bg_gather_tileset(m._h, tile_row, set_index, word_bits, C.byref(t)))
    return TileSet(t.ts, tuple(int(v) for v in t.rows), tuple(int(v) for v in t.cols))


def gather_tilesets(m: FrdcMatrix, word_bits: int = 32) -> Tuple[torch.Tensor, torch.Tensor]:
    """Every tile set of the matrix, assembled on the device (Algorithm 1
    lines 1-5 for all tile rows): (set_ptr int64 [tile_rows+1] with set_ptr[r]
    the first set of tile row r, sets uint8 [total, 96] of bg_tileset records:
    ts i32, pad i32, rows u64[4], cols u32[16])."""
    tr = m.tile_rows
    set_ptr = torch.empty(tr + 1, dtype=torch.int64, device="cuda")
    total = C.c_int64()
    check(lib().bg_tileset_ptr(m._h, word_bits, set_ptr.data_ptr(), C.byref(total), _stream()))
    sets = torch.empty((max(total.value, 0), C.sizeof(L.TileSetC)), dtype=torch.uint8, device="cuda")
    check(lib().bg_gather_tilesets(m._h, word_bits, set_ptr.data_ptr(), total.value,
                                   sets.data_ptr() if total.value else None, _stream()))
    return set_ptr, sets


def frdc_to_dense(m: FrdcMatrix, word_bits: int = 32) -> BitDenseMatrix:
    """bitsparse.cpp:114-127 -- ZeroOne bits, node_rows x node_cols."""
    out = BitDenseMatrix.empty(m.node_rows, m.node_cols, word_bits, ZERO_ONE)
    check(lib().bg_frdc_to_dense(m._h, word_bits, out.words.data_ptr(), _stream()))
    return out


def frdc_stats(m: FrdcMatrix) -> FrdcStats:
    """bitsparse.cpp:162-169"""
    st = L.FrdcStatsC()
    check(lib().bg_frdc_stats_get(m._h, C.byref(st)))
    return FrdcStats(st.nnz_tiles, st.nnz_bits, st.bytes, st.fill_ratio)


@dataclass
class AdjacencyOperand:
    """kernels.hpp:52-57 -- raw structure, or diag(row)*A*diag(col) when factorized."""
    structure: FrdcMatrix
    row_scale: Optional[torch.Tensor] = None
    col_scale: Optional[torch.Tensor] = None

    def factorized(self) -> bool:
        return self.row_scale is not None


class GraphBundle:
    """graphops.hpp:28-38 -- A+I, loop-free A and their scales, on the device."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        i = L.GraphInfo()
        check(lib().bg_graph_info_get(self._h, C.byref(i)))
        self.n = i.n
        self.structure = FrdcMatrix(i.structure, owner=self)
        self.raw = FrdcMatrix(i.raw, owner=self)
        n = max(i.n, 0)
        self.norm_row = device_view(i.norm, (n,), "<f4")
        self.norm_col = self.norm_row
        self.mean_row = device_view(i.mean_row, (n,), "<f4")
        self.ones_row = device_view(i.ones, (n,), "<f4")
        self.ones_col = self.ones_row
        self.neighbor_count = device_view(i.neighbor_count, (n,), "<i8")

    def corrupt_tile(self, k: int) -> None:
        check(lib().bg_graph_corrupt_tile(self._h, k))

    def shard(self, row_begin: int, row_end: int) -> "GraphBundle":
        """This rank's share: both structures cut to node rows [row_begin,
        row_end) (whole tile rows), the scale vectors whole (bg_graph_shard)."""
        h = C.c_void_p()
        check(lib().bg_graph_shard(self._h, row_begin, row_end, C.byref(h), _stream()))
        g = GraphBundle(h.value)
        g.row0 = row_begin
        return g

    def partition_rows(self, world_size: int, rank: int) -> Tuple[int, int]:
        a, b = C.c_int64(), C.c_int64()
        check(lib().bg_partition_rows(self._h, world_size, rank, C.byref(a), C.byref(b)))
        return a.value, b.value

    def __del__(self):
        try:
            if self._h:
                lib().bg_graph_destroy(self._h)
        except Exception:
            pass


def prepare_graph(node_count: int, src, dst) -> GraphBundle:
    """graphops.cpp:146-170, on the device."""
    s, d = _edges(src, dst)
    h = C.c_void_p()
    check(lib().bg_prepare_graph(s.data_ptr(), d.data_ptr(), s.shape[0], node_count, C.byref(h), _stream()))
    return GraphBundle(h.value)


# --------------------------------------------------------------------------- #
# Kernel families (kernels.hpp:63-97)
# --------------------------------------------------------------------------- #
def bmm(v, a: MatOperand, w: MatOperand, word_bits: int = 32) -> MatOperand:
    v = _v(v)
    ca, cw = _mat(a, ROW), _mat(w, COL)
    if isinstance(w, BitOperand):
        cw.scale_axis = w.scale_axis if w.scale is not None else COL
    desc = L.Mat()
    check(lib().bg_bmm_out_desc(v._c(), C.byref(ca), C.byref(cw), word_bits, C.byref(desc)))
    out, desc = _alloc(desc)
    check(lib().bg_bmm(v._c(), C.byref(ca), C.byref(cw), word_bits, C.byref(desc), _stream()))
    return out


def bspmm(v, adj: AdjacencyOperand, x: MatOperand, strategy: Optional[int] = None,
          word_bits: int = 32) -> MatOperand:
    v = _v(v)
    if adj is None or adj.structure is None:
        raise InvalidArgument("bspmm: missing adjacency structure")
    cx = _mat(x)
    desc = L.Mat()
    check(lib().bg_bspmm_out_desc(v._c(), adj.structure._h, C.byref(cx), word_bits, C.byref(desc)))
    out, desc = _alloc(desc)
    st = -1 if strategy is None else int(strategy)
    rs, cs = _vec(adj.row_scale), _vec(adj.col_scale)  # kept alive until the call returns
    check(lib().bg_bspmm(v._c(), adj.structure._h, _ptr(rs), _ptr(cs),
                         C.byref(cx), st, word_bits, C.byref(desc), _stream()))
    return out


def _shape_of(m: MatOperand) -> Tuple[int, int]:
    if isinstance(m, BitOperand):
        return m.bits.rows, m.bits.cols
    return tuple(m.shape)


def add(v, a: MatOperand, b: MatOperand) -> MatOperand:
    v = _v(v)
    ca, cb = _mat(a), _mat(b)
    desc = L.Mat()
    desc.precision, (desc.rows, desc.cols) = v.out, _shape_of(a)
    desc.word_bits = a.bits.word_bits if isinstance(a, BitOperand) else 32
    out, desc = _alloc(desc)
    check(lib().bg_add(v._c(), C.byref(ca), C.byref(cb), C.byref(desc), _stream()))
    return out


def concat(v, a: MatOperand, b: MatOperand) -> MatOperand:
    v = _v(v)
    ca, cb = _mat(a), _mat(b)
    (ra, ka), (_, kb) = _shape_of(a), _shape_of(b)
    desc = L.Mat()
    desc.precision, desc.rows, desc.cols = v.out, ra, ka + kb
    desc.word_bits = a.bits.word_bits if isinstance(a, BitOperand) else 32
    out, desc = _alloc(desc)
    check(lib().bg_concat(v._c(), C.byref(ca), C.byref(cb), C.byref(desc), _stream()))
    return out


def fused_mm_spmm(mm, spmm, x: MatOperand, w: MatOperand, adj: AdjacencyOperand,
                  strategy: Optional[int] = None) -> MatOperand:
    mm, spmm = _v(mm), _v(spmm)
    if mm.out != spmm.in1:
        raise InvalidArgument(f"fused_mm_spmm: precision chain mismatch ({mm.name()} -> {spmm.name()})")
    cx, cw = _mat(x), _mat(w, COL)
    hdesc = L.Mat()
    check(lib().bg_bmm_out_desc(mm._c(), C.byref(cx), C.byref(cw), 32, C.byref(hdesc)))
    desc = L.Mat()
    check(lib().bg_bspmm_out_desc(spmm._c(), adj.structure._h, C.byref(hdesc), 32, C.byref(desc)))
    out, desc = _alloc(desc)
    st = -1 if strategy is None else int(strategy)
    rs, cs = _vec(adj.row_scale), _vec(adj.col_scale)
    check(lib().bg_fused_mm_spmm(mm._c(), spmm._c(), C.byref(cx), C.byref(cw), adj.structure._h,
                                 _ptr(rs), _ptr(cs), st,
                                 C.byref(desc), _stream()))
    return out


def dense_mm(a: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    a, w = _dense(a), _dense(w)
    if a.shape[1] != w.shape[0]:
        raise InvalidArgument("dense_mm: inner dimensions disagree")
    out = torch.empty((a.shape[0], w.shape[1]), dtype=torch.float32, device="cuda")
    check(lib().bg_dense_mm(a.data_ptr(), w.data_ptr(), a.shape[0], a.shape[1], w.shape[1], out.data_ptr(), _stream()))
    return out


def scl(x: torch.Tensor, row: torch.Tensor, col: torch.Tensor) -> torch.Tensor:
    x = _dense(x)
    if row.numel() != x.shape[0] or col.numel() != x.shape[1]:
        raise InvalidArgument("scl: scale length mismatch")
    row, col = _vec(row), _vec(col)
    out = torch.empty_like(x)
    check(lib().bg_scl(x.data_ptr(), x.shape[0], x.shape[1], row.data_ptr(),
                       col.data_ptr(), out.data_ptr(), _stream()))
    return out


def softmax_rows(x: torch.Tensor) -> torch.Tensor:
    x = _dense(x)
    out = torch.empty_like(x)
    check(lib().bg_softmax_rows(x.data_ptr(), x.shape[0], x.shape[1], out.data_ptr(), _stream()))
    return out


def batchnorm_infer(x: torch.Tensor, gamma, beta, mean, sigma) -> torch.Tensor:
    x = _dense(x)
    ps = [torch.as_tensor(p, dtype=torch.float32).cuda().contiguous() for p in (gamma, beta, mean, sigma)]
    if any(p.numel() != x.shape[1] for p in ps):
        raise InvalidArgument(f"batchnorm: parameter lengths do not match {x.shape[1]} columns")
    out = torch.empty_like(x)
    check(lib().bg_batchnorm_infer(x.data_ptr(), x.shape[0], x.shape[1], *[p.data_ptr() for p in ps],
                                   out.data_ptr(), _stream()))
    return out


# --------------------------------------------------------------------------- #
# Models (graphops.hpp:57-133, modelconfig.cpp:49-173)
# --------------------------------------------------------------------------- #
KIND = {"gcn_conv": L.LAYER_GCN, "sage_conv": L.LAYER_SAGE, "graph_conv": L.LAYER_GRAPHCONV,
        "fc": L.LAYER_FC, "aggregate": L.LAYER_AGGREGATE, "relu": L.LAYER_RELU,
        "batchnorm": L.LAYER_BATCHNORM, "softmax": L.LAYER_SOFTMAX, "binarize": L.LAYER_BINARIZE,
        "scale": L.LAYER_SCALE}


@dataclass
class LayerSpec:
    kind: int
    plan: List[Union[str, KernelVariant]] = field(default_factory=list)
    w1: Optional[np.ndarray] = None
    w2: Optional[np.ndarray] = None
    relu: bool = False
    bn: Optional[Tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]] = None  # gamma, beta, mean, sigma
    scale_row: Optional[np.ndarray] = None
    scale_col: Optional[np.ndarray] = None


def _descs(layers: Sequence[LayerSpec]):
    arr = (L.LayerDesc * max(len(layers), 1))()
    keep = []

    def host(a):
        a = np.ascontiguousarray(a, dtype=np.float32)
        keep.append(a)
        return a

    for i, l in enumerate(layers):
        d = arr[i]
        d.kind = l.kind
        d.n_plan = len(l.plan)
        for k, p in enumerate(l.plan[:4]):
            d.plan[k] = _v(p)._c()
        if l.w1 is not None:
            w = host(l.w1)
            d.w1, d.w1_rows, d.w1_cols = w.ctypes.data, w.shape[0], w.shape[1]
        if l.w2 is not None:
            w = host(l.w2)
            d.w2, d.w2_rows, d.w2_cols = w.ctypes.data, w.shape[0], w.shape[1]
        d.relu = int(l.relu)
        if l.bn is not None:
            g, b, m, s = (host(p) for p in l.bn)
            d.bn_gamma, d.bn_beta, d.bn_mean, d.bn_sigma = g.ctypes.data, b.ctypes.data, m.ctypes.data, s.ctypes.data
            d.bn_len = g.shape[0]
        if l.scale_row is not None and l.scale_col is not None:
            r, c = host(l.scale_row), host(l.scale_col)
            d.scale_row, d.scale_row_len = r.ctypes.data, r.shape[0]
            d.scale_col, d.scale_col_len = c.ctypes.data, c.shape[0]
    return arr, keep


def validate_model(layers: Sequence[LayerSpec], has_graph: bool = True,
                   input_precision: int = F) -> List[str]:
    """graphops.cpp:245-268 -- human-readable problems, empty when well formed."""
    arr, keep = _descs(layers)
    buf = C.create_string_buffer(1 << 16)
    n = lib().bg_validate_model(int(has_graph), input_precision, arr, len(layers), buf, len(buf))
    return buf.value.decode().split("\n") if n else []


def rewrite_eliminate_scl(layers: Sequence[LayerSpec]) -> List[LayerSpec]:
    """graphops.cpp:357-368 -- drop every Scale layer directly ahead of a
    Binarize (positive factors move no value across the sign threshold)."""
    return [l for i, l in enumerate(layers)
            if not (l.kind == L.LAYER_SCALE and i + 1 < len(layers) and layers[i + 1].kind == L.LAYER_BINARIZE)]


@dataclass
class TracePoint:
    label: str
    bits: BitDenseMatrix


@dataclass
class KernelTiming:
    label: str
    ms: float


class Model:
    """A ModelSpec compiled onto the device (graphops.hpp:75-81)."""

    def __init__(self, layers: Sequence[LayerSpec], graph: Optional[GraphBundle] = None,
                 input_precision: int = F, word_bits: int = 32, strategy: Optional[int] = None):
        arr, keep = _descs(layers)
        h = C.c_void_p()
        check(lib().bg_model_create(graph._h if graph is not None else None, input_precision,
                                    -1 if strategy is None else strategy, word_bits, arr,
                                    len(layers), C.byref(h), _stream()))
        self._h = h
        self.graph = graph
        self.word_bits = word_bits
        self.layers = list(layers)

    def output_cols(self) -> int:
        c = C.c_int64()
        check(lib().bg_model_output_cols(self._h, C.byref(c)))
        return c.value

    def set_graph_capture(self, enable: bool) -> None:
        check(lib().bg_model_set_graph_capture(self._h, int(enable)))

    def _out(self, rows: int):
        return torch.empty((rows, self.output_cols()), dtype=torch.float32, device="cuda")

    def forward(self, x0: MatOperand, out: Optional[torch.Tensor] = None,
                logits: Optional[torch.Tensor] = None) -> torch.Tensor:
        cx = _mat(x0)
        out = self._out(cx.rows) if out is None else out
        check(lib().bg_model_forward(self._h, C.byref(cx), out.data_ptr(),
                                     logits.data_ptr() if logits is not None else None, _stream()))
        return out

    def forward_traced(self, x0: MatOperand):
        """run_model with a RunTrace: (out, logits, [TracePoint])."""
        cx = _mat(x0)
        out, logits = self._out(cx.rows), self._out(cx.rows)
        t = C.c_void_p()
        check(lib().bg_trace_create(C.byref(t)))
        try:
            check(lib().bg_model_forward_traced(self._h, C.byref(cx), out.data_ptr(), logits.data_ptr(), t, _stream()))
            pts = _trace_points(t)
        finally:
            lib().bg_trace_destroy(t)
        return out, logits, pts

    def forward_timed(self, x0: MatOperand) -> Tuple[torch.Tensor, List[KernelTiming]]:
        cx = _mat(x0)
        out = self._out(cx.rows)
        cap = 256
        arr = (L.KernelTiming * cap)()
        n = C.c_int()
        check(lib().bg_model_forward_timed(self._h, C.byref(cx), out.data_ptr(), None, arr, cap, C.byref(n), _stream()))
        return out, [KernelTiming(arr[i].label.decode(), arr[i].ms) for i in range(n.value)]

    def forward_host(self, x: np.ndarray, logits: bool = False, stream: Optional[torch.cuda.Stream] = None):
        """End-to-end call with host buffers (H2D + forward + D2H).  The
        returned host tensors are the model's pinned result buffers: they stay
        valid until the next forward_host call (clone to keep them)."""
        if isinstance(x, torch.Tensor):
            xh = x.contiguous()
            rows, cols, xp = xh.shape[0], xh.shape[1], xh.data_ptr()
        else:
            xh = np.ascontiguousarray(x, dtype=np.float32)
            rows, cols, xp = xh.shape[0], xh.shape[1], xh.ctypes.data
        oc = self.output_cols()
        # pinned result buffers are reused across calls with the same shape
        # (page-locking 10s of MB per call would cost more than the copy)
        cache = getattr(self, "_host_out", None)
        if cache is None or cache[0].shape != (rows, oc) or (logits and cache[1] is None):
            cache = (torch.empty((rows, oc), dtype=torch.float32, pin_memory=True),
                     torch.empty((rows, oc), dtype=torch.float32, pin_memory=True) if logits else None)
            self._host_out = cache
        out, lg = cache[0], (cache[1] if logits else None)
        s = (stream or torch.cuda.current_stream()).cuda_stream
        check(lib().bg_model_forward_host(self._h, xp, rows, cols, out.data_ptr(),
                                          lg.data_ptr() if lg is not None else None, s))
        return (out, lg) if logits else out

    def __del__(self):
        try:
            if self._h:
                lib().bg_model_destroy(self._h)
        except Exception:
            pass


def _trace_points(t) -> List["TracePoint"]:
    pts = []
    for i in range(lib().bg_trace_size(t)):
        lab, r, c, wb, bits = C.c_char_p(), C.c_int64(), C.c_int64(), C.c_int(), C.c_void_p()
        check(lib().bg_trace_point(t, i, C.byref(lab), C.byref(r), C.byref(c), C.byref(wb), C.byref(bits)))
        view = device_view(bits.value, (r.value, storage_words_per_row(c.value, wb.value)), "<i4")
        pts.append(TracePoint(lab.value.decode(), BitDenseMatrix(view.clone(), r.value, c.value, wb.value)))
    return pts


def _layer(kind: int, fn, x: MatOperand, l: LayerSpec, g: GraphBundle, strategy: Optional[int],
           trace: Optional[list], prefix: str, word_bits: int) -> MatOperand:
    arr, keep = _descs([l])
    cx = _mat(x)
    desc = L.Mat()
    check(lib().bg_layer_out_desc(kind, arr, C.byref(cx), word_bits, C.byref(desc)))
    out, desc = _alloc(desc)
    t = C.c_void_p()
    if trace is not None:
        check(lib().bg_trace_create(C.byref(t)))
    try:
        check(fn(C.byref(cx), arr, g._h, -1 if strategy is None else int(strategy), t if trace is not None else None,
                 prefix.encode(), word_bits, C.byref(desc), _stream()))
        if trace is not None:
            trace.extend(_trace_points(t))
    finally:
        if trace is not None:
            lib().bg_trace_destroy(t)
    return out


def gcn_layer(x: MatOperand, l: LayerSpec, g: GraphBundle, strategy: Optional[int] = None,
              trace: Optional[list] = None, prefix: str = "", word_bits: int = 32) -> MatOperand:
    """graphops.cpp:270-285 -- {mm, spmm} over A+I (norm scales when in2 = F);
    BIN points are appended to `trace` (a list of TracePoint) under `prefix`."""
    return _layer(L.LAYER_GCN, lib().bg_gcn_layer, x, l, g, strategy, trace, prefix, word_bits)


def sage_layer(x: MatOperand, l: LayerSpec, g: GraphBundle, strategy: Optional[int] = None,
               trace: Optional[list] = None, prefix: str = "", word_bits: int = 32) -> MatOperand:
    """graphops.cpp:325-329 -- neighborhood layer over loop-free A, mean aggregation."""
    return _layer(L.LAYER_SAGE, lib().bg_sage_layer, x, l, g, strategy, trace, prefix, word_bits)


def graphconv_layer(x: MatOperand, l: LayerSpec, g: GraphBundle, strategy: Optional[int] = None,
                    trace: Optional[list] = None, prefix: str = "", word_bits: int = 32) -> MatOperand:
    """graphops.cpp:331-335 -- neighborhood layer over loop-free A, sum aggregation."""
    return _layer(L.LAYER_GRAPHCONV, lib().bg_graphconv_layer, x, l, g, strategy, trace, prefix, word_bits)


@dataclass
class VerifyReport:
    """runreport.hpp:13-25"""
    max_rel_logit_error: float = 0.0
    bin_points: int = 0
    bin_values: int = 0
    bin_mismatches: int = 0
    first_mismatch_label: str = ""
    first_mismatch_row: int = -1
    first_mismatch_col: int = -1
    argmax_agreement: float = 0.0
    tolerance: float = 1e-6
    passed: bool = False

    def to_dict(self) -> dict:
        """The fields of VerifyReport::to_json (runreport.cpp:137-152)."""
        d = {"max_rel_logit_error": self.max_rel_logit_error, "tolerance": self.tolerance,
             "bin_points": self.bin_points, "bin_values": self.bin_values,
             "bin_mismatches": self.bin_mismatches}
        if self.bin_mismatches > 0:
            d["first_mismatch"] = {"label": self.first_mismatch_label, "row": self.first_mismatch_row,
                                   "col": self.first_mismatch_col}
        d.update(argmax_agreement=self.argmax_agreement, **{"pass": self.passed})
        return d


def verify_model(model: Model, x0: MatOperand, ref_points: Sequence, ref_logits: np.ndarray,
                 tolerance: float = 1e-6, compare_bits: bool = True) -> VerifyReport:
    """runreport.cpp:51-135 on the device: a traced forward of `model`
    compared with a reference run -- ref_points (objects with label, bits
    [rows, spw] u32, rows, cols, word_bits, in trace order) and ref_logits
    (rows x cols, compared in double).  compare_bits=False is the
    reference's full-precision mode.  Misaligned traces raise LogicError."""
    cx = _mat(x0)
    keep = []
    arr = (L.RefPointC * max(len(ref_points), 1))()
    for i, p in enumerate(ref_points):
        b = np.ascontiguousarray(p.bits, dtype=np.uint32)
        lab = p.label.encode()
        keep += [b, lab]
        arr[i] = L.RefPointC(lab, p.rows, p.cols, p.word_bits, b.ctypes.data)
    lg = np.ascontiguousarray(ref_logits, dtype=np.float64)
    r = L.VerifyReportC()
    check(lib().bg_model_verify(model._h, C.byref(cx), arr, len(ref_points), lg.ctypes.data, lg.shape[0],
                                lg.shape[1], int(compare_bits), tolerance, C.byref(r), _stream()))
    return VerifyReport(r.max_rel_logit_error, r.bin_points, r.bin_values, r.bin_mismatches,
                        r.first_mismatch_label.decode(), r.first_mismatch_row, r.first_mismatch_col,
                        r.argmax_agreement, r.tolerance, bool(r.pass_))


def run_model(model: Model, x0: MatOperand, trace: bool = False):
    """graphops.cpp:390-484 -- returns the final output (and the trace)."""
    if trace:
        return model.forward_traced(x0)
    return model.forward(x0)


# --------------------------------------------------------------------------- #
# rng.hpp -- the product's own synthetic-input generator (std::mt19937_64)
# --------------------------------------------------------------------------- #
class Rng:
    def __init__(self, seed: int):
        h = C.c_void_p()
        check(lib().bg_rng_create(C.c_uint64(seed), C.byref(h)))
        self._h = h

    def random_dense(self, rows: int, cols: int) -> np.ndarray:
        out = np.empty((rows, cols), np.float32)
        check(lib().bg_rng_dense(self._h, rows, cols, out.ctypes.data))
        return out

    def random_edges(self, nodes: int, m: int, allow_self: bool = False):
        src = np.empty(max(m, 1), np.int64)
        dst = np.empty(max(m, 1), np.int64)
        k = C.c_int64()
        check(lib().bg_rng_edges(self._h, nodes, m, int(allow_self), src.ctypes.data, dst.ctypes.data, C.byref(k)))
        return src[:k.value], dst[:k.value]

    def __del__(self):
        try:
            if self._h:
                lib().bg_rng_destroy(self._h)
        except Exception:
            pass


DEFAULT_PLANS = {  # modelconfig.cpp:49-60
    "gcn": ["MM.FBB+BSpMM.BBB", "MM.BBF+BSpMM.FBF"],
    "sage": ["MM.FBB+MM.FBB+BSpMM.BBB+ADD.BBF", "MM.FBF+MM.FBF+BSpMM.FFF+ADD.FFF"],
    "saint": ["MM.FBB+MM.FBB+BSpMM.BBB+ADD.BBF", "MM.FBB+MM.FBB+BSpMM.BBB+ADD.BBF", "MM.FBF"],
}


def build_model_spec(model: str, features: int, hidden: int, classes: int, seed: int, nodes: int,
                     plan: Optional[Sequence[str]] = None):
    """build_model (modelconfig.cpp:99-173): X first, then W1 (and W2) per
    layer from one stream.  Returns (layer specs, X as host float32)."""
    plan = list(plan) if plan else DEFAULT_PLANS[model]
    rng = Rng(seed)
    X = rng.random_dense(nodes, features)

    def dims(n):
        out, fin = [], features
        for i in range(n):
            fo = classes if i + 1 == n else hidden
            out.append((fin, fo))
            fin = fo
        return out

    layers: List[LayerSpec] = []
    if model == "gcn":
        dd = dims(len(plan))
        for i, chain in enumerate(plan):
            layers.append(LayerSpec(L.LAYER_GCN, chain.split("+"), rng.random_dense(*dd[i]), None, i + 1 < len(plan)))
    elif model in ("sage", "saint"):
        conv = len(plan) - 1 if model == "saint" else len(plan)
        dd = dims(conv + (1 if model == "saint" else 0))
        for i in range(conv):
            w1 = rng.random_dense(*dd[i])
            w2 = rng.random_dense(*dd[i])
            layers.append(LayerSpec(L.LAYER_SAGE if model == "sage" else L.LAYER_GRAPHCONV,
                                    plan[i].split("+"), w1, w2, True))
        if model == "saint":
            layers.append(LayerSpec(L.LAYER_FC, plan[-1].split("+"), rng.random_dense(*dd[-1]), None, False))
        else:
            layers[-1].relu = False
    else:
        raise RuntimeFailure(f'config: unknown model "{model}"')
    layers.append(LayerSpec(L.LAYER_SOFTMAX))
    return layers, X
