"""Row-sharded multi-GPU forward: one process per GPU (torch.distributed for
the plumbing, NCCL inside the C++ engine for the exchange).

Each rank builds the same graph and model, owns a contiguous range of node
rows (tile-row aligned, balanced by FRDC tiles: ``partition_bounds``) and
computes those rows of every layer; before every neighbour aggregation the
C++ engine all-gathers the aggregated operand over NVLink (a grouped NCCL
broadcast per rank, include/bitgnn_b200.h ``bg_model_forward_sharded``).
Outputs are bit-identical to the single-GPU forward for every shard count.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib as L
from .bitgnn import KernelTiming, Model, _mat, _stream, storage_words_per_row
from ._lib import check, lib


def partition_bounds(row_ptr: np.ndarray, node_count: int, world_size: int) -> List[int]:
    """Host-side tile-row partition (C ABI bg_partition_bounds): bounds[0..world]."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
    out = np.zeros(world_size + 1, np.int64)
    check(lib().bg_partition_bounds(rp.ctypes.data, rp.shape[0] - 1, node_count, world_size,
                                    out.ctypes.data))
    return [int(v) for v in out]


class Comm:
    """NCCL communicator owned by the C++ engine; the unique id travels over
    the caller's torch.distributed process group."""

    ID_BYTES = 128

    def __init__(self, dist, world: int, rank: int):
        buf = torch.zeros(self.ID_BYTES, dtype=torch.uint8)
        if rank == 0:
            raw = (C.c_uint8 * self.ID_BYTES)()
            check(lib().bg_comm_unique_id(raw, self.ID_BYTES))
            buf = torch.tensor(list(bytes(raw)), dtype=torch.uint8)
        obj = [buf.numpy().tobytes()]
        dist.broadcast_object_list(obj, src=0)
        ident = (C.c_uint8 * self.ID_BYTES).from_buffer_copy(obj[0])
        h = C.c_void_p()
        check(lib().bg_comm_create(world, rank, ident, self.ID_BYTES, C.byref(h)))
        self._h = h
        self.world, self.rank = world, rank

    def __del__(self):
        try:
            if self._h:
                lib().bg_comm_destroy(self._h)
        except Exception:
            pass


class ShardedModel:
    """The model of ``layers`` on ``graph``, this rank computing its rows.

    forward(x, out): x holds this rank's rows (or the full matrix, in which
    case the rank's slice is taken); out receives this rank's output rows.
    """

    def __init__(self, layers: Sequence, graph, dist, world: int, rank: int, word_bits: int = 32):
        self.model = Model(layers, graph, word_bits=word_bits)
        rp, _, _ = graph.structure.download()
        self.bounds = partition_bounds(rp, graph.n, world)
        self.b = np.asarray(self.bounds, np.int64)
        self.world, self.rank = world, rank
        self.row0, self.row1 = self.bounds[rank], self.bounds[rank + 1]
        self.comm = Comm(dist, world, rank) if world > 1 else None
        self.n = graph.n

    def _local(self, x: torch.Tensor) -> torch.Tensor:
        return x[self.row0:self.row1] if x.shape[0] == self.n else x

    def forward(self, x: torch.Tensor, out: Optional[torch.Tensor] = None,
                logits: Optional[torch.Tensor] = None) -> torch.Tensor:
        xl = self._local(x).contiguous()
        rows = self.row1 - self.row0
        oc = self.model.output_cols()
        if out is None or out.shape[0] != rows:
            out = torch.empty((rows, oc), dtype=torch.float32, device="cuda")
        cx = _mat(xl)
        check(lib().bg_model_forward_sharded(
            self.model._h, self.comm._h if self.comm else None, C.byref(cx), self.b.ctypes.data,
            self.world, self.rank, out.data_ptr(), logits.data_ptr() if logits is not None else None,
            _stream()))
        return out

    def forward_timed(self, x):
        """The sharded forward with per-op CUDA-event times on this rank
        (same labels as Model.forward_timed, plus 'layerI.allgather')."""
        xl = self._local(x).contiguous()
        rows = self.row1 - self.row0
        out = torch.empty((rows, self.model.output_cols()), dtype=torch.float32, device="cuda")
        cx = _mat(xl)
        cap = 256
        arr = (L.KernelTiming * cap)()
        n = C.c_int()
        check(lib().bg_model_forward_sharded_timed(
            self.model._h, self.comm._h if self.comm else None, C.byref(cx), self.b.ctypes.data, self.world,
            self.rank, out.data_ptr(), arr, cap, C.byref(n), _stream()))
        return out, [KernelTiming(arr[i].label.decode(), arr[i].ms) for i in range(n.value)]

    def forward_host(self, xh):
        """End to end on this rank: its rows of the host X in (a pinned tensor's
        row slice stays pinned, so the copy is a DMA), the sharded forward,
        its output rows back to the host."""
        if isinstance(xh, torch.Tensor):
            xl = xh[self.row0:self.row1].to("cuda", non_blocking=True)
        else:
            xl = torch.from_numpy(np.ascontiguousarray(xh[self.row0:self.row1])).cuda()
        out = self.forward(xl)
        return out.cpu()


def forward_virtual_ranks(model: Model, x: torch.Tensor, bounds: Sequence[int],
                          logits: bool = False):
    """Run every rank's row range of the sharded forward in this process on
    this device (no communicator): the single-GPU check of the sharded path."""
    b = np.asarray(bounds, np.int64)
    cx = _mat(x)
    oc = model.output_cols()
    out = torch.empty((x.shape[0], oc), dtype=torch.float32, device="cuda")
    lg = torch.empty_like(out) if logits else None
    check(lib().bg_model_forward_sharded(model._h, None, C.byref(cx), b.ctypes.data, len(b) - 1, 0,
                                         out.data_ptr(), lg.data_ptr() if lg is not None else None,
                                         _stream()))
    return (out, lg) if logits else out
