"""ctypes binding of the C ABI in include/bitgnn_b200.h.

The shared library is built in-tree (``make lib`` or ``__graft_entry__.build()``)
as ``paper_2305_02522_b200/libbitgnn_b200.so``.  There is deliberately no
fallback: if the library is missing or cannot be loaded, importing the package
fails with the loader's error.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbitgnn_b200.so")

BG_OK, BG_INVALID_ARGUMENT, BG_RUNTIME_ERROR, BG_LOGIC_ERROR, BG_CUDA_ERROR = range(5)
F, B = 0, 1
BMM, BSPMM, ADD, CONCAT = 0, 1, 2, 3
AXIS_ROW, AXIS_COL = 0, 1
ZERO_ONE, PLUS_MINUS = 0, 1
STRATEGY_DEFAULT, IF_ELSE, AND_ANDNOT, TWO_AND_MINUS_POPC = -1, 0, 1, 2
(LAYER_GCN, LAYER_SAGE, LAYER_GRAPHCONV, LAYER_FC, LAYER_AGGREGATE, LAYER_RELU,
 LAYER_BATCHNORM, LAYER_SOFTMAX, LAYER_BINARIZE, LAYER_SCALE) = range(10)


class Variant(C.Structure):
    _fields_ = [("op", C.c_int32), ("in1", C.c_int32), ("in2", C.c_int32), ("out", C.c_int32)]


class Mat(C.Structure):
    _fields_ = [("precision", C.c_int32), ("word_bits", C.c_int32), ("semantics", C.c_int32),
                ("scale_axis", C.c_int32), ("rows", C.c_int64), ("cols", C.c_int64),
                ("data", C.c_void_p), ("scale", C.c_void_p)]


class FrdcInfo(C.Structure):
    _fields_ = [("node_rows", C.c_int64), ("node_cols", C.c_int64), ("tile_rows", C.c_int64),
                ("tile_cols", C.c_int64), ("nnz_tiles", C.c_int64), ("nnz_bits", C.c_int64),
                ("max_row_degree", C.c_int64), ("row_ptr", C.c_void_p), ("col_ind", C.c_void_p),
                ("tiles", C.c_void_p), ("degree", C.c_void_p)]


class GraphInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("structure", C.c_void_p), ("raw", C.c_void_p),
                ("norm", C.c_void_p), ("mean_row", C.c_void_p), ("ones", C.c_void_p),
                ("neighbor_count", C.c_void_p)]


class LayerDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_plan", C.c_int32), ("plan", Variant * 4),
                ("w1", C.c_void_p), ("w1_rows", C.c_int64), ("w1_cols", C.c_int64),
                ("w2", C.c_void_p), ("w2_rows", C.c_int64), ("w2_cols", C.c_int64),
                ("relu", C.c_int32),
                ("bn_gamma", C.c_void_p), ("bn_beta", C.c_void_p), ("bn_mean", C.c_void_p),
                ("bn_sigma", C.c_void_p), ("bn_len", C.c_int64),
                ("scale_row", C.c_void_p), ("scale_row_len", C.c_int64),
                ("scale_col", C.c_void_p), ("scale_col_len", C.c_int64)]


class TileSetC(C.Structure):
    _fields_ = [("ts", C.c_int32), ("reserved", C.c_int32), ("rows", C.c_uint64 * 4),
                ("cols", C.c_uint32 * 16)]


class FrdcStatsC(C.Structure):
    _fields_ = [("nnz_tiles", C.c_uint64), ("nnz_bits", C.c_uint64), ("bytes", C.c_uint64),
                ("fill_ratio", C.c_double)]


class VerifyReportC(C.Structure):
    _fields_ = [("max_rel_logit_error", C.c_double), ("bin_points", C.c_int64), ("bin_values", C.c_int64),
                ("bin_mismatches", C.c_int64), ("first_mismatch_label", C.c_char * 64),
                ("first_mismatch_row", C.c_int64), ("first_mismatch_col", C.c_int64),
                ("argmax_agreement", C.c_double), ("tolerance", C.c_double), ("pass_", C.c_int32)]


class RefPointC(C.Structure):
    _fields_ = [("label", C.c_char_p), ("rows", C.c_int64), ("cols", C.c_int64), ("word_bits", C.c_int32),
                ("bits", C.c_void_p)]


class KernelTiming(C.Structure):
    _fields_ = [("label", C.c_char * 64), ("ms", C.c_double)]


AGG_AUTO, AGG_SLIVERS, AGG_TILES, AGG_WINDOW = 0, 1, 2, 3

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int
PI64 = C.POINTER(C.c_int64)

# name -> (restype, argtypes); every bg_* symbol declared in include/bitgnn_b200.h.
PROTOTYPES = {
    "bg_last_error": (C.c_char_p, []),
    "bg_version": (I32, []),
    "bg_set_aggregation": (I32, [I32, I32]),
    "bg_get_aggregation": (I32, [C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "bg_set_persistent": (I32, [I32]),
    "bg_device_count": (I32, [C.POINTER(C.c_int)]),
    "bg_device_alloc": (I32, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "bg_device_free": (I32, [P]),
    "bg_memcpy": (I32, [P, P, C.c_size_t, I32, P]),
    "bg_memset": (I32, [P, I32, C.c_size_t, P]),
    "bg_stream_synchronize": (I32, [P]),
    "bg_variant_parse": (I32, [C.c_char_p, C.POINTER(Variant)]),
    "bg_variant_valid": (I32, [Variant]),
    "bg_variant_name": (I32, [Variant, C.c_char_p, C.c_size_t]),
    "bg_storage_words_per_row": (I64, [I64, I32]),
    "bg_binarize": (I32, [P, I64, I64, I32, P, P]),
    "bg_binarize_with_scale": (I32, [P, I64, I64, I32, I32, P, P, P]),
    "bg_unpack": (I32, [P, I64, I64, I32, I32, P, P]),
    "bg_transpose": (I32, [P, I64, I64, I32, P, P]),
    "bg_frdc_from_edges": (I32, [P, P, I64, I64, I32, C.POINTER(P), P]),
    "bg_frdc_from_host": (I32, [I64, I64, P, P, P, I64, C.POINTER(P), P]),
    "bg_frdc_info_get": (I32, [P, C.POINTER(FrdcInfo)]),
    "bg_frdc_download": (I32, [P, P, P, P]),
    "bg_frdc_corrupt_tile": (I32, [P, I64]),
    "bg_tileset_count": (I32, [P, I64, I32, PI64]),
    "bg_gather_tileset": (I32, [P, I64, I64, I32, C.POINTER(TileSetC)]),
    "bg_tileset_ptr": (I32, [P, I32, P, PI64, P]),
    "bg_gather_tilesets": (I32, [P, I32, P, I64, P, P]),
    "bg_frdc_to_dense": (I32, [P, I32, P, P]),
    "bg_frdc_stats_get": (I32, [P, C.POINTER(FrdcStatsC)]),
    "bg_frdc_serialized_size": (I32, [P, C.POINTER(C.c_size_t)]),
    "bg_frdc_serialize": (I32, [P, I32, P, C.c_size_t]),
    "bg_frdc_deserialize": (I32, [P, C.c_size_t, C.POINTER(C.c_void_p), C.POINTER(C.c_int), P]),
    "bg_frdc_write_file": (I32, [P, I32, C.c_char_p]),
    "bg_frdc_read_file": (I32, [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int), P]),
    "bg_frdc_destroy": (None, [P]),
    "bg_read_edge_list": (I32, [C.c_char_p, C.c_size_t, C.c_char_p, I64, I32, C.POINTER(P)]),
    "bg_read_matrix_market": (I32, [C.c_char_p, C.c_size_t, C.c_char_p, I32, C.POINTER(P)]),
    "bg_load_graph": (I32, [C.c_char_p, I64, I32, C.POINTER(P)]),
    "bg_edges_info": (I32, [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(P), C.POINTER(P), C.POINTER(P),
                            C.POINTER(I64)]),
    "bg_edges_destroy": (None, [P]),
    "bg_prepare_graph": (I32, [P, P, I64, I64, C.POINTER(P), P]),
    "bg_graph_info_get": (I32, [P, C.POINTER(GraphInfo)]),
    "bg_graph_corrupt_tile": (I32, [P, I64]),
    "bg_graph_destroy": (None, [P]),
    "bg_bmm_out_desc": (I32, [Variant, C.POINTER(Mat), C.POINTER(Mat), I32, C.POINTER(Mat)]),
    "bg_bspmm_out_desc": (I32, [Variant, P, C.POINTER(Mat), I32, C.POINTER(Mat)]),
    "bg_bmm": (I32, [Variant, C.POINTER(Mat), C.POINTER(Mat), I32, C.POINTER(Mat), P]),
    "bg_bspmm": (I32, [Variant, P, P, P, C.POINTER(Mat), I32, I32, C.POINTER(Mat), P]),
    "bg_add": (I32, [Variant, C.POINTER(Mat), C.POINTER(Mat), C.POINTER(Mat), P]),
    "bg_concat": (I32, [Variant, C.POINTER(Mat), C.POINTER(Mat), C.POINTER(Mat), P]),
    "bg_scl": (I32, [P, I64, I64, P, P, P, P]),
    "bg_dense_mm": (I32, [P, P, I64, I64, I64, P, P]),
    "bg_relu_inplace": (I32, [C.POINTER(Mat), P]),
    "bg_softmax_rows": (I32, [P, I64, I64, P, P]),
    "bg_batchnorm_infer": (I32, [P, I64, I64, P, P, P, P, P, P]),
    "bg_fused_mm_spmm": (I32, [Variant, Variant, C.POINTER(Mat), C.POINTER(Mat), P, P, P, I32,
                               C.POINTER(Mat), P]),
    "bg_layer_out_desc": (I32, [I32, C.POINTER(LayerDesc), C.POINTER(Mat), I32, C.POINTER(Mat)]),
    "bg_gcn_layer": (I32, [C.POINTER(Mat), C.POINTER(LayerDesc), P, I32, P, C.c_char_p, I32, C.POINTER(Mat), P]),
    "bg_sage_layer": (I32, [C.POINTER(Mat), C.POINTER(LayerDesc), P, I32, P, C.c_char_p, I32, C.POINTER(Mat), P]),
    "bg_graphconv_layer": (I32, [C.POINTER(Mat), C.POINTER(LayerDesc), P, I32, P, C.c_char_p, I32,
                                 C.POINTER(Mat), P]),
    "bg_validate_model": (I32, [I32, I32, C.POINTER(LayerDesc), I32, C.c_char_p, C.c_size_t]),
    "bg_model_create": (I32, [P, I32, I32, I32, C.POINTER(LayerDesc), I32, C.POINTER(P), P]),
    "bg_model_destroy": (None, [P]),
    "bg_model_output_cols": (I32, [P, PI64]),
    "bg_model_set_graph_capture": (I32, [P, I32]),
    "bg_model_forward": (I32, [P, C.POINTER(Mat), P, P, P]),
    "bg_model_forward_host": (I32, [P, P, I64, I64, P, P, P]),
    "bg_trace_create": (I32, [C.POINTER(P)]),
    "bg_trace_destroy": (None, [P]),
    "bg_model_forward_traced": (I32, [P, C.POINTER(Mat), P, P, P, P]),
    "bg_trace_size": (I32, [P]),
    "bg_trace_point": (I32, [P, I32, C.POINTER(C.c_char_p), PI64, PI64, C.POINTER(C.c_int),
                             C.POINTER(P)]),
    "bg_verify_trace": (I32, [P, P, I64, I64, C.POINTER(RefPointC), I32, P, I32, C.c_double,
                              C.POINTER(VerifyReportC), P]),
    "bg_model_verify": (I32, [P, C.POINTER(Mat), C.POINTER(RefPointC), I32, P, I64, I64, I32, C.c_double,
                              C.POINTER(VerifyReportC), P]),
    "bg_model_forward_timed": (I32, [P, C.POINTER(Mat), P, P, C.POINTER(KernelTiming), I32,
                                     C.POINTER(C.c_int), P]),
    "bg_partition_rows": (I32, [P, I32, I32, PI64, PI64]),
    "bg_partition_bounds": (I32, [P, I64, I64, I32, P]),
    "bg_comm_unique_id": (I32, [P, C.c_size_t]),
    "bg_comm_create": (I32, [I32, I32, P, C.c_size_t, C.POINTER(P)]),
    "bg_comm_destroy": (None, [P]),
    "bg_comm_create_external": (I32, [I32, I32, P, P, C.POINTER(P)]),
    "bg_graph_shard": (I32, [P, I64, I64, C.POINTER(P), P]),
    "bg_model_forward_sharded": (I32, [P, P, C.POINTER(Mat), P, I32, I32, P, P, P]),
    "bg_model_forward_sharded_timed": (I32, [P, P, C.POINTER(Mat), P, I32, I32, P, C.POINTER(KernelTiming), I32,
                                             C.POINTER(I32), P]),
    "bg_rng_create": (I32, [C.c_uint64, C.POINTER(P)]),
    "bg_rng_destroy": (None, [P]),
    "bg_rng_dense": (I32, [P, I64, I64, P]),
    "bg_rng_edges": (I32, [P, I64, I64, I32, P, P, PI64]),
}


class BitGNNError(RuntimeError):
    """Base class; the concrete type mirrors the reference's exception."""


class InvalidArgument(BitGNNError, ValueError):  # std::invalid_argument
    pass


class RuntimeFailure(BitGNNError):  # std::runtime_error
    pass


class LogicError(BitGNNError):  # std::logic_error
    pass


class CudaError(BitGNNError):
    pass


_EXC = {BG_INVALID_ARGUMENT: InvalidArgument, BG_RUNTIME_ERROR: RuntimeFailure,
        BG_LOGIC_ERROR: LogicError, BG_CUDA_ERROR: CudaError}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make lib` (or __graft_entry__.build()); "
                "there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != BG_OK:
        msg = lib().bg_last_error().decode()
        raise _EXC.get(rc, BitGNNError)(msg)
