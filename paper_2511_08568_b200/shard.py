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
