"""ORACLE — TEST INFRASTRUCTURE ONLY.

The reference's synthetic trace generator (generate_trace, trace.py:124-161,
/root/reference/pkg/src/embcache) restated over numpy + the C pool pass
(replay_oracle.c:oracle_pool_pass), with no dependency on the product
package, so bench.py's reference arm builds its workload from the oracle
alone.  Pinned: tests/test_oracle.py checks it against the sha256 of
reference-generated traces (tests/golden/traces.npz).
"""
from __future__ import annotations

import ctypes
import heapq
import os

import numpy as np

from . import lib as _lib


def _pool_pass(zipf, sticky, poolc, stickiness, pool_size, pool, plen):
    L = _lib()
    i64p = ctypes.POINTER(ctypes.c_int64)
    dp = ctypes.POINTER(ctypes.c_double)
    L.oracle_pool_pass.argtypes = [i64p, dp, dp, ctypes.c_int64, ctypes.c_double,
                                   ctypes.c_int32, i64p, ctypes.POINTER(ctypes.c_int32), i64p]
    out = np.empty(len(zipf), dtype=np.int64)
    rc = L.oracle_pool_pass(zipf.ctypes.data_as(i64p), sticky.ctypes.data_as(dp),
                            poolc.ctypes.data_as(dp), len(zipf), float(stickiness),
                            int(pool_size), pool.ctypes.data_as(i64p),
                            plen.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                            out.ctypes.data_as(i64p))
    if rc != 0:
        raise ValueError(f"oracle_pool_pass failed rc={rc}")
    return out


def generate_gids(table_sizes, total_accesses, zipf_exponent=1.1, markov_stickiness=0.0,
                  correlation_pool_size=32, rng_seed=0) -> np.ndarray:
    """trace.py:124-161: int64 [n] flat ids, the same default_rng(seed)
    stream (permutation, choice with p, two coin arrays) and the same
    sequential pool pass."""
    rng = np.random.default_rng(rng_seed)
    total = int(sum(table_sizes))
    n = int(total_accesses)
    ranks = np.arange(1, total + 1, dtype=np.float64)
    weights = ranks ** (-zipf_exponent)
    probs = weights / weights.sum()
    rank_to_gid = rng.permutation(total)
    zipf = rank_to_gid[rng.choice(total, size=n, p=probs)].astype(np.int64)
    sticky = rng.random(n)
    poolc = rng.random(n)
    pool = np.zeros(correlation_pool_size, dtype=np.int64)
    return _pool_pass(zipf, sticky, poolc, markov_stickiness, correlation_pool_size, pool,
                      np.zeros(1, dtype=np.int32))


def generate_gid_blocks(table_sizes, total_accesses, zipf_exponent=1.1, markov_stickiness=0.0,
                        correlation_pool_size=32, rng_seed=0, block=1 << 24,
                        threads=None):
    """generate_gids block by block (bounded memory for 5e8 accesses): the
    three random() streams of generate_trace start at outputs 0, n and 2n of
    the PCG64 state right after the permutation (choice with p draws one
    double per access: cdf.searchsorted(random(n), 'right')), reached with
    PCG64.advance; the pool carries across blocks.  Yields int64 blocks."""
    rng = np.random.default_rng(rng_seed)
    total = int(sum(table_sizes))
    n = int(total_accesses)
    ranks = np.arange(1, total + 1, dtype=np.float64)
    weights = ranks ** (-zipf_exponent)
    del ranks
    cdf = (weights / weights.sum()).cumsum()
    del weights
    cdf /= cdf[-1]
    rank_to_gid = rng.permutation(total)
    state = rng.bit_generator.state

    def stream(offset):
        b = np.random.PCG64()
        b.state = state
        b.advance(offset)
        return np.random.Generator(b)

    def draws(i0):
        c = min(block, n - i0)
        zipf = rank_to_gid[cdf.searchsorted(stream(i0).random(c), side="right")]
        return zipf.astype(np.int64), stream(n + i0).random(c), stream(2 * n + i0).random(c)

    # the draws of a wave of blocks run on the host cores (numpy releases the
    # GIL in random() and searchsorted()); the pool pass stays sequential
    from concurrent.futures import ThreadPoolExecutor
    workers = threads or max(1, min(32, len(os.sched_getaffinity(0))))
    pool = np.zeros(correlation_pool_size, dtype=np.int64)
    plen = np.zeros(1, dtype=np.int32)
    starts = list(range(0, n, block))
    with ThreadPoolExecutor(max_workers=workers) as ex:
        for w0 in range(0, len(starts), workers):
            for zipf, sticky, poolc in ex.map(draws, starts[w0:w0 + workers]):
                yield _pool_pass(zipf, sticky, poolc, markov_stickiness,
                                 correlation_pool_size, pool, plen)


def table_offsets(table_sizes) -> np.ndarray:
    return np.concatenate([[0], np.cumsum(np.asarray(table_sizes, dtype=np.int64))])


def table_ids(gids, table_sizes) -> np.ndarray:
    """trace.py:86 (searchsorted of the table offsets)."""
    return np.searchsorted(table_offsets(table_sizes), gids, side="right") - 1


def assign_tables(counts, n_ranks: int) -> np.ndarray:
    """The benchmark's table sharding: LPT greedy by access
    count, heaviest table first to the lightest rank, ties by table then
    rank index."""
    counts = np.asarray(counts, dtype=np.int64)
    order = sorted(range(len(counts)), key=lambda t: (-int(counts[t]), t))
    heap = [(0, r) for r in range(n_ranks)]
    out = np.empty(len(counts), dtype=np.int64)
    for t in order:
        load, r = heapq.heappop(heap)
        out[t] = r
        heapq.heappush(heap, (load + int(counts[t]), r))
    return out
