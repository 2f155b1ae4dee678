"""Row-sharded multi-GPU forward: one process per GPU (torch.distributed for
the plumbing, NCCL inside the C++ engine for the exchange).

Each rank builds the graph, owns a contiguous range of node rows (tile-row
aligned, balanced by FRDC tiles: ``partition_bounds``), keeps only its slice
of the adjacency (``GraphBundle.shard``) and computes those rows of every
layer; before every neighbour aggregation the C++ engine all-gathers the
aggregated operand over NVLink (a grouped NCCL broadcast per rank,
include/bitgnn_b200.h ``bg_model_forward_sharded``; captured with the
kernels as one CUDA graph).  ``HostComm`` replaces NCCL by a host-staged
all-gather over any torch.distributed group (gloo): the same engine and
exchange points, used to run several ranks on one GPU in the tests.
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
        if world > 1:
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


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64), C.c_int,
                           C.c_int, C.c_void_p)


class HostComm:
    """An external exchange (bg_comm_create_external): the engine hands this
    rank's produced rows over on the host and the other ranks' rows come back
    through ``dist.all_gather`` of host tensors (gloo), padded to the largest
    range.  Slower than NVLink, but any process group works -- several ranks
    on one GPU included."""

    def __init__(self, dist, world: int, rank: int, group=None):
        self.dist, self.group = dist, group
        self.world, self.rank = world, rank
        self.calls = 0
        self._fn = ALLGATHER_FN(self._allgather)  # kept alive with the handle
        h = C.c_void_p()
        check(lib().bg_comm_create_external(world, rank, self._fn, None, C.byref(h)))
        self._h = h

    def _allgather(self, _ctx, buf, row_bytes, bounds_p, world, rank, _stream):
        try:
            b = [int(bounds_p[q]) for q in range(world + 1)]
            from .bitgnn import device_view
            full = device_view(buf, (b[-1], row_bytes), "|i1") if b[-1] and row_bytes else None
            mx = max(b[q + 1] - b[q] for q in range(world))
            mine = torch.zeros((mx, row_bytes), dtype=torch.int8)
            if b[rank + 1] > b[rank]:
                mine[: b[rank + 1] - b[rank]] = full[b[rank]:b[rank + 1]].cpu()
            parts = [torch.zeros_like(mine) for _ in range(world)]
            self.dist.all_gather(parts, mine, group=self.group)
            for q in range(world):
                if q != rank and b[q + 1] > b[q]:
                    full[b[q]:b[q + 1]].copy_(parts[q][: b[q + 1] - b[q]])
            torch.cuda.synchronize()
            self.calls += 1
            return 0
        except Exception as ex:  # reported as the forward's failure
            print("HostComm all-gather failed:", ex)
            return 1

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

    def __init__(self, layers: Sequence, graph, dist, world: int, rank: int, word_bits: int = 32,
                 transport: str = "nccl", shard_graph: bool = True, group=None, input_precision: int = L.F):
        rp, _, _ = graph.structure.download()
        self.bounds = partition_bounds(rp, graph.n, world)
        self.b = np.asarray(self.bounds, np.int64)
        self.world, self.rank = world, rank
        self.row0, self.row1 = self.bounds[rank], self.bounds[rank + 1]
        # this rank keeps its slice of the adjacency only (the caller may
        # drop the whole graph afterwards)
        self.graph = graph.shard(self.row0, self.row1) if shard_graph else graph
        self.model = Model(layers, self.graph, input_precision=input_precision, word_bits=word_bits)
        if transport == "host":
            self.comm = HostComm(dist, world, rank, group)
        elif world > 1 or transport == "nccl1":
            self.comm = Comm(dist, world, rank)  # "nccl1": NCCL even for one rank (tests)
        else:
            self.comm = None
        self.n = graph.n

    def _local(self, x):
        """This rank's rows of the model input (a dense tensor or a BitOperand)."""
        from .bitgnn import BitDenseMatrix, BitOperand
        if isinstance(x, BitOperand):
            b = x.bits
            if b.rows != self.n:
                return x
            words = b.words[self.row0:self.row1].contiguous()
            sc = x.scale[self.row0:self.row1] if (x.scale is not None and x.scale_axis == L.AXIS_ROW) else x.scale
            return BitOperand(BitDenseMatrix(words, self.row1 - self.row0, b.cols, b.word_bits, b.semantics),
                              sc, x.scale_axis)
        return (x[self.row0:self.row1] if x.shape[0] == self.n else x).contiguous()

    def forward(self, x, out: Optional[torch.Tensor] = None,
                logits: Optional[torch.Tensor] = None) -> torch.Tensor:
        xl = self._local(x)
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
        xl = self._local(x)
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
