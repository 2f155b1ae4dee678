"""B200-native binary-GNN inference hot path (BitGNN, arXiv 2305.02522).

The compute path is hand-written sm_100a CUDA behind the C ABI in
include/bitgnn_b200.h; this package is the Python host mirror of the
reference operator API (see bitgnn.py).  Importing it loads the in-tree
libbitgnn_b200.so and fails if it is missing -- there is no CPU fallback.
"""
from ._lib import lib as _load

_load()

from .bitgnn import *  # noqa: E402,F401,F403
from .bitgnn import (AdjacencyOperand, BitDenseMatrix, BitOperand, FrdcMatrix,  # noqa: E402,F401
                     GraphBundle, KernelVariant, LayerSpec, Model, Rng, add, binarize,
                     binarize_with_scale, bmm, bspmm, build_model_spec, concat, EdgeList, frdc_from_edges,
                     load_graph, read_edge_list, read_matrix_market,
                     prepare_graph, rewrite_eliminate_scl, run_model, transpose, unpack, validate_model,
                     TileSet, FrdcStats, gather_tileset, gather_tilesets, tileset_count, frdc_to_dense,
                     frdc_stats, gcn_layer, sage_layer, graphconv_layer,
                     VerifyReport, verify_model)
from ._lib import (B, F, CudaError, InvalidArgument, LogicError, RuntimeFailure)  # noqa: E402,F401
