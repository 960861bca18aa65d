"""Table-wise sharding of the hot path across GPUs.

Every GPU owns a set of embedding tables, the order-preserving sub-trace of
accesses to them, its own buffer shard (capacity = 20% of the shard's unique
ids) and its slice of the model inference.  The replay needs no collective:
each shard equals the reference ``replay`` run on
``trace_from_gids(shard_gids, full_table_sizes)`` (full table sizes keep the
vocabulary check, runtime.py:213-217, and the global decode scale,
model.py:255, identical).  Counters are summed once at the end; the float64
coverage is a per-shard value (runtime.py:282) and is reported per shard.

Assignment is greedy by access count (largest table first onto the least
loaded rank), never in contiguous blocks: the hottest table carries up to
16.7x the mean load.
"""
from __future__ import annotations

import heapq

import numpy as np

from .errors import InvalidConfigError
from .trace import Trace, table_offsets

COUNTERS = ("cache_hits", "prefetch_hits", "on_demand", "prefetch_issued", "prefetch_useful",
            "evictions", "prefetch_inserts")


def table_access_counts(trace) -> np.ndarray:
    off = table_offsets(trace.table_sizes)
    tid = np.searchsorted(off, np.asarray(trace.gid_array), side="right") - 1
    return np.bincount(tid, minlength=len(trace.table_sizes)).astype(np.int64)


def assign_tables(counts, n_ranks: int) -> np.ndarray:
    """rank of every table: LPT greedy (heaviest first -> lightest rank),
    ties broken by table index and rank index so every rank computes the
    same assignment."""
    counts = np.asarray(counts, dtype=np.int64)
    order = sorted(range(len(counts)), key=lambda t: (-int(counts[t]), t))
    heap = [(0, r) for r in range(n_ranks)]
    out = np.empty(len(counts), dtype=np.int64)
    for t in order:
        load, r = heapq.heappop(heap)
        out[t] = r
        heapq.heappush(heap, (load + int(counts[t]), r))
    return out


def shard_trace(trace, assignment, rank: int) -> Trace:
    """Order-preserving sub-trace of the tables assigned to `rank`."""
    off = table_offsets(trace.table_sizes)
    g = np.asarray(trace.gid_array)
    tid = np.searchsorted(off, g, side="right") - 1
    mask = np.asarray(assignment)[tid] == rank
    return Trace(g[mask], trace.table_sizes)


def shard_capacity(shard: Trace, fraction: float = 0.2, ways: int | None = 32) -> int:
    c = int(np.floor(fraction * shard.unique_count))
    if ways:
        c -= c % ways
    return max(c, ways or 1)


def reduce_counters(local: dict, group=None) -> dict:
    """Sum integer counters over the process group (one all_reduce)."""
    import torch
    import torch.distributed as dist
    v = torch.tensor([int(local[k]) for k in COUNTERS], dtype=torch.int64)
    if dist.is_initialized():
        if dist.get_backend(group) == "nccl":
            v = v.cuda()
        dist.all_reduce(v, group=group)
    return dict(zip(COUNTERS, (int(x) for x in v.cpu().tolist())))


class TableShard:
    """One rank's tables of a table-sharded layout.

    The rank's models are packed over its LOCAL vocabulary (its tables in
    ascending global order, rows renumbered from 0), so a GPU holds only its
    own embed_id rows / folded tables; the replay keeps GLOBAL gids and the
    prefetch decode keeps the global scale (decode_ids = total_ids,
    model.py:255), so a shard predicts foreign gids exactly as the reference
    does on ``trace_from_gids(shard_gids, full_table_sizes)``.
    """

    def __init__(self, table_sizes, tables):
        self.table_sizes = [int(s) for s in table_sizes]
        self.tables = sorted({int(t) for t in tables})
        if not self.tables or self.tables[0] < 0 or self.tables[-1] >= len(self.table_sizes):
            raise InvalidConfigError("shard tables outside the table layout")
        self.local_sizes = [self.table_sizes[t] for t in self.tables]
        self.offsets = table_offsets(self.table_sizes)
        self.local_offsets = table_offsets(self.local_sizes)
        self.table_local = np.full(len(self.table_sizes), -1, dtype=np.int32)
        self.table_local[self.tables] = np.arange(len(self.tables), dtype=np.int32)
        self.total_ids = int(self.offsets[-1])
        self.local_ids = int(self.local_offsets[-1])

    def to_local(self, gids):
        """(local gid, local table) of global gids (host; -1 for foreign ids)."""
        g = np.asarray(gids, dtype=np.int64)
        t = np.searchsorted(self.offsets, g, side="right") - 1
        lt = self.table_local[t]
        lg = np.where(lt >= 0, g - self.offsets[t] + self.local_offsets[np.maximum(lt, 0)], -1)
        return lg, lt.astype(np.int64)


def init_params_shard(kind, table_sizes, tables, dim=32, stacks=None, l_in=15, l_out=5, seed=0,
                      init_scale=0.08, device=True, block_rows=1 << 20):
    """init_params (model.py:83-100) restricted to a table shard, bit-exact.

    init_params draws every array from one default_rng(seed) stream, one
    double per element, embed_id [V, d] first.  Here the PCG64 stream jumps
    (bit_generator.advance) over the embed_id rows of other shards' tables,
    so only the shard's rows are drawn; embed_table keeps the shard's rows,
    every dense array is drawn whole.  Returns (ModelParameters over the
    local vocabulary, without "embed_id"; the local embed_id rows as fp32,
    on the GPU when device else a numpy array).
    """
    from .model import CACHING, PREFETCH, ModelParameters, _shapes
    if kind not in (CACHING, PREFETCH):
        raise InvalidConfigError(f"unknown model kind {kind!r}")
    if stacks is None:
        stacks = 1 if kind == CACHING else 2
    sh = tables if isinstance(tables, TableShard) else TableShard(table_sizes, tables)
    d = int(dim)
    rng = np.random.default_rng(seed)
    bg = rng.bit_generator
    if device:
        from . import _native
        torch = _native.torch_cuda()
        emb = torch.empty((sh.local_ids, d), dtype=torch.float32, device="cuda")
    else:
        emb = np.empty((sh.local_ids, d), dtype=np.float32)
    pos = 0   # PCG64 outputs consumed so far
    for lt, t in enumerate(sh.tables):
        r0, rows = int(sh.offsets[t]), sh.table_sizes[t]
        bg.advance(r0 * d - pos)
        l0 = int(sh.local_offsets[lt])
        for b in range(0, rows, block_rows):
            nb = min(block_rows, rows - b)
            blk = rng.uniform(-init_scale, init_scale, size=(nb, d)).astype(np.float32)
            if device:
                emb[l0 + b:l0 + b + nb].copy_(torch.from_numpy(blk))
            else:
                emb[l0 + b:l0 + b + nb] = blk
        pos = (r0 + rows) * d
    bg.advance(sh.total_ids * d - pos)
    shapes = _shapes(kind, sh.total_ids, len(sh.table_sizes), d, stacks, l_out)
    arrays = {name: rng.uniform(-init_scale, init_scale, size=shape)
              for name, shape in shapes.items() if name != "embed_id"}
    arrays["embed_table"] = np.ascontiguousarray(arrays["embed_table"][sh.tables])
    return ModelParameters(kind, list(sh.local_sizes), d, stacks, l_in, l_out, arrays), emb
