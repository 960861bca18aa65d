"""DLRM embedding stage across GPUs (config 4): table-sharded
buffers and pooling, one all-to-all of pooled embeddings per batch.

Rank g owns tables T_g (``shard.assign_tables``), their rows in pinned host
memory, its buffer shard and its slice of the access stream.  For a batch of
B samples, every sample has one bag of P ids per table (the synthetic trace
has no query boundaries, so the bag layout is builder-defined — SPEC.md:104):

1. the local accesses of the batch run through the hot path (models +
   buffer replay, ``HotPath``) and the changed buffer rows are gathered from
   host memory (K5, ``RowStore.refresh``);
2. K6 (``RowStore.pool``) sums each local bag, writing rows in
   (sample, local table) order — which is already peer-major: rank r needs
   samples [r*B/G, (r+1)*B/G), a contiguous block;
3. one ``all_to_all_single`` (NCCL over NVLink; no pack kernel) leaves rank
   r with [B/G, T, D]: every table's pooled row for its samples.

The pooling is injectable (``pool_fn``) so the multi-process host logic is
tested on CPU with gloo (tests/test_dist.py).
"""
from __future__ import annotations

import numpy as np

from .trace import table_offsets


def build_bags(trace, tables, batch: int, pooling: int, start: int = 0) -> np.ndarray:
    """[batch, len(tables), pooling] global ids: bag (b, t) = the
    (start+b)-th run of `pooling` consecutive accesses to table t in trace
    order (cyclic when a table's stream is shorter)."""
    off = table_offsets(trace.table_sizes)
    g = np.asarray(trace.gid_array)
    tid = np.searchsorted(off, g, side="right") - 1
    out = np.empty((batch, len(tables), pooling), dtype=np.int64)
    for j, t in enumerate(tables):
        stream = g[tid == t]
        if len(stream) == 0:
            stream = np.array([off[t]], dtype=np.int64)   # a never-accessed table: row 0
        idx = (np.arange(batch)[:, None] + start) * pooling + np.arange(pooling)[None, :]
        out[:, j, :] = stream[idx % len(stream)]
    return out


class DlrmEmbeddingStage:
    def __init__(self, table_sizes, assignment, rank: int, world: int, dim: int, pool_fn,
                 group=None):
        self.table_sizes = list(table_sizes)
        self.assignment = np.asarray(assignment)
        self.rank, self.world, self.dim = rank, world, dim
        self.pool_fn = pool_fn
        self.group = group
        self.local_tables = [t for t in range(len(self.table_sizes)) if self.assignment[t] == rank]
        self.tables_of = [[t for t in range(len(self.table_sizes)) if self.assignment[t] == r]
                          for r in range(world)]

    def forward(self, local_bags):
        """local_bags: [B, T_g, P] ids of this rank's tables (torch, on the
        pooling device).  Returns [B/G, T, D] pooled rows for this rank's
        samples, tables in global order."""
        import torch
        import torch.distributed as dist
        B, Tg, P = local_bags.shape
        G = self.world
        if B % G:
            raise ValueError("batch must split evenly across ranks")
        flat = local_bags.reshape(-1).to(torch.int32)
        offsets = torch.arange(0, B * Tg * P + 1, P, dtype=torch.int64, device=flat.device)
        pooled = self.pool_fn(flat, offsets)                        # [B*Tg, D], peer-major
        send = pooled.reshape(B * Tg * self.dim)
        splits_out = [B // G * len(ts) * self.dim for ts in self.tables_of]
        recv = torch.empty(sum(splits_out), dtype=pooled.dtype, device=pooled.device)
        if G > 1:
            dist.all_to_all_single(recv, send, output_split_sizes=splits_out,
                                   input_split_sizes=[B // G * Tg * self.dim] * G,
                                   group=self.group)
        else:
            recv.copy_(send)
        out = torch.empty((B // G, len(self.table_sizes), self.dim), dtype=pooled.dtype,
                          device=pooled.device)
        pos = 0
        for r, ts in enumerate(self.tables_of):
            n = B // G * len(ts) * self.dim
            if ts:
                out[:, ts, :] = recv[pos:pos + n].reshape(B // G, len(ts), self.dim)
            pos += n
        return out
