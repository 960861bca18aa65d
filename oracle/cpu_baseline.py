"""ORACLE — TEST INFRASTRUCTURE ONLY.

The reference algorithm timed on the host cores (the CPU baseline of
bench.py and its ``--impl reference`` arm), built from the oracle alone:

* weights: ``init_params`` (model.py:83-100) drawn row by row -- embed_id row
  g is PCG64 outputs [g*d, (g+1)*d) of default_rng(seed) (Generator.uniform
  takes one 64-bit output per double), the dense arrays start at output V*d
  in _shapes order -- so only the rows a sample touches are materialised;
* decisions: the float64 numpy forwards (model_oracle.py) in batches of 256
  chunks (runtime.py:181-210), bits = logit >= 0, ids = the fp64 decode;
* replay: the C restatement in the reference's dense per-id layout
  (runtime.py:41-112, 220-283) plus the 32-way LRU (cache_sim.py:92-106).

The product package is never imported here.
"""
from __future__ import annotations

import os
import time

import numpy as np

from . import lru as _lru
from . import num_chunks as _num_chunks
from . import replay as _replay
from . import model_oracle as mo
from .trace_oracle import table_ids


def shapes(kind, total_ids, table_count, dim, stacks, l_out=5):
    """_shapes (model.py:54-80): names and order of the parameter arrays."""
    d = dim
    out = {"embed_id": (total_ids, d), "embed_table": (table_count, d),
           "att_enc": (d, d), "att_dec": (d, d), "att_v": (d, 1),
           "comb_w": (2 * d, d), "comb_b": (d,), "head_w": (d, 1), "head_b": (1,)}
    for k in range(stacks):
        out[f"enc{k}_wx"] = (2 * d if k == 0 else d, 4 * d)
        out[f"enc{k}_wh"] = (d, 4 * d)
        out[f"enc{k}_b"] = (4 * d,)
        out[f"dec{k}_wx"] = (3 * d if k == 0 else d, 4 * d)
        out[f"dec{k}_wh"] = (d, 4 * d)
        out[f"dec{k}_b"] = (4 * d,)
    if kind == "prefetch":
        out["slot_embed"] = (l_out, 2 * d)
    return out


def draw_params(kind, table_sizes, dim, rows, seed, init_scale, l_out=5):
    """init_params(kind, table_sizes, dim, seed=seed, init_scale=s) with
    embed_id restricted to `rows` (int array): (arrays, stacks)."""
    stacks = 1 if kind == "caching" else 2
    V = int(sum(table_sizes))
    emb = np.empty((len(rows), dim))
    for i, g in enumerate(np.asarray(rows, dtype=np.int64)):
        b = np.random.PCG64(seed)
        b.advance(int(g) * dim)
        emb[i] = np.random.Generator(b).uniform(-init_scale, init_scale, dim)
    b = np.random.PCG64(seed)
    b.advance(V * dim)
    rng = np.random.Generator(b)
    arrays = {nm: rng.uniform(-init_scale, init_scale, size=s)
              for nm, s in shapes(kind, V, len(table_sizes), dim, stacks, l_out).items()
              if nm != "embed_id"}
    arrays["embed_id"] = emb
    return arrays, stacks


def run(gids, table_sizes, dim, init_scale, n_sample, capacity, ways, eviction_speed=4,
        cores=None, label="trace"):
    """Time the reference algorithm on the first n_sample accesses of `gids`
    (the workload's trace or a table shard's sub-trace, global ids):
    forwards on `cores` threads (one per core, BLAS single-threaded inside),
    then the sequential replay and the LRU.  Returns the baseline dict plus
    the decisions ("_bits", "_pf") for agreement checks."""
    from concurrent.futures import ThreadPoolExecutor
    from threadpoolctl import threadpool_limits
    g = np.asarray(gids[:n_sample], dtype=np.int64)
    V = int(sum(table_sizes))
    K = _num_chunks(len(g))
    uniq, inv = np.unique(g[:K * 15], return_inverse=True)
    lg = inv.reshape(K, 15)
    tid = table_ids(g[:K * 15], table_sizes).reshape(K, 15)
    ac, cs = draw_params("caching", table_sizes, dim, uniq, 0, init_scale)
    ap, ps = draw_params("prefetch", table_sizes, dim, uniq, 1, init_scale)
    cores = cores or len(os.sched_getaffinity(0))
    bits = np.empty((K, 15), dtype=np.uint8)
    pf = np.empty((K, 5), dtype=np.int64)

    def batches(b0, b1):
        for b in range(b0, b1, 256):          # runtime.py:181-210, batches of 256
            e = min(b + 256, b1)
            bits[b:e] = mo.caching_logits(ac, dim, cs, lg[b:e], tid[b:e]) >= 0
            lp = mo.prefetch_logits(ap, dim, ps, 5, lg[b:e], tid[b:e])
            pf[b:e] = mo.decode_gids(mo.sigmoid(lp), V)

    step = max(256, (K // cores + 255) // 256 * 256)
    with threadpool_limits(limits=1), ThreadPoolExecutor(max_workers=cores) as pool:
        # warm-up (thread pool, page faults) on the first batches, untimed
        list(pool.map(lambda b: batches(b, min(b + 256, K)), range(0, min(K, 256 * cores), 256)))
        t0 = time.perf_counter()
        list(pool.map(lambda b: batches(b, min(b + step, K)), range(0, K, step)))
        t1 = time.perf_counter()
    _replay(g, V, capacity, ways, eviction_speed, bits=bits, pf=pf, dense=True)
    _lru(g, V, capacity, ways)
    t2 = time.perf_counter()
    return {"value": len(g) / (t2 - t0), "unit": "accesses/s", "cores": cores, "kind": "port",
            "sample": f"first {len(g)} accesses of the {label} ({K} chunks): numpy float64 "
                      f"forwards on {cores} threads {t1 - t0:.2f}s + C replay (dense per-id "
                      f"layout, sequential as runtime.py) + 32-way LRU {t2 - t1:.2f}s",
            "model_s": t1 - t0, "replay_s": t2 - t1, "_bits": bits, "_pf": pf}
