"""Row-sharded multi-GPU forward (one process per GPU).  Filled in below."""
from __future__ import annotations


class ShardedModel:
    def __init__(self, layers, graph, dist, world, rank):
        raise NotImplementedError("row-sharded forward: not built yet")
