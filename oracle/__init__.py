"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference (arxiv 2511.08568 ``embcache``) hot path:

* ``replay_oracle.c`` — the buffer replay, set-associative LRU and LRU+PF
  baselines (runtime.py / cache_sim.py), built into ``liboracle.so``;
* ``model_oracle.py`` — float64 numpy forwards of both models (model.py).

Pinned against the reference's own outputs: tests/golden/ (made by
tests/golden/make_golden.py, which imports /root/reference in the build
container).  Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU
baseline legs may import this package; the product path never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

COUNTER_NAMES = ("cache_hits", "prefetch_hits", "on_demand", "prefetch_issued",
                 "prefetch_useful", "evictions", "prefetch_inserts", "max_occupancy")


def build():
    """Compile replay_oracle.c (make -C oracle)."""
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "replay_oracle.c"))):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        dp = ctypes.POINTER(ctypes.c_double)
        L.oracle_replay.argtypes = [i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                    ctypes.c_int32, ctypes.c_int32, u8p, i64p,
                                    ctypes.c_int32, ctypes.c_int, i64p, dp, u8p]
        L.oracle_replay.restype = ctypes.c_int
        L.oracle_lru.argtypes = [i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                 ctypes.c_int64, u8p, i64p]
        L.oracle_lru.restype = ctypes.c_int
        L.oracle_lru_prefetch.argtypes = [i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                          i64p, ctypes.c_int32, i64p, dp]
        L.oracle_lru_prefetch.restype = ctypes.c_int
        L.oracle_num_chunks.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_int32]
        L.oracle_num_chunks.restype = ctypes.c_int64
        L.oracle_coverage_sum.argtypes = [u8p, u8p, ctypes.c_int64]
        L.oracle_coverage_sum.restype = ctypes.c_double
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct)) if a is not None else None


def pad_prefetches(prefetches, stride=None):
    """list of per-chunk gid lists -> int64 [K, stride] padded with -1."""
    if stride is None:
        stride = max((len(p) for p in prefetches), default=0)
    out = np.full((len(prefetches), max(stride, 1)), -1, dtype=np.int64)
    for k, p in enumerate(prefetches):
        out[k, :len(p)] = p
    return out


def replay(gids, total_ids, capacity, ways=0, eviction_speed=4, l_in=15, l_out=5,
           window_ratio=3, bits=None, pf=None, dense=False, access_class=False):
    """Returns (counters dict, coverage float[, access_class uint8[n]])."""
    gids = np.ascontiguousarray(gids, dtype=np.int64)
    n = len(gids)
    b = None if bits is None else np.ascontiguousarray(bits, dtype=np.uint8).reshape(-1)
    p = None if pf is None else np.ascontiguousarray(pf, dtype=np.int64)
    stride = 0 if p is None else p.shape[1]
    p = None if p is None else p.reshape(-1)
    ctr = np.zeros(8, dtype=np.int64)
    cov = ctypes.c_double(0.0)
    cls = np.zeros(n, dtype=np.uint8) if access_class else None
    rc = lib().oracle_replay(_p(gids, ctypes.c_int64), n, int(total_ids), int(capacity),
                             int(ways), int(eviction_speed), l_in, l_out, window_ratio,
                             _p(b, ctypes.c_uint8), _p(p, ctypes.c_int64), stride,
                             1 if dense else 0, _p(ctr, ctypes.c_int64), ctypes.byref(cov),
                             _p(cls, ctypes.c_uint8))
    if rc != 0:
        raise ValueError(f"oracle_replay failed rc={rc}")
    res = dict(zip(COUNTER_NAMES, (int(x) for x in ctr)))
    if access_class:
        return res, cov.value, cls
    return res, cov.value


def lru(gids, total_ids, capacity, ways=0, per_access=False):
    gids = np.ascontiguousarray(gids, dtype=np.int64)
    hits = ctypes.c_int64(0)
    pa = np.zeros(len(gids), dtype=np.uint8) if per_access else None
    rc = lib().oracle_lru(_p(gids, ctypes.c_int64), len(gids), int(total_ids), int(capacity),
                          int(ways), _p(pa, ctypes.c_uint8), ctypes.byref(hits))
    if rc != 0:
        raise ValueError(f"oracle_lru failed rc={rc}")
    return (hits.value, pa) if per_access else hits.value


def lru_prefetch(gids, total_ids, capacity, pf, l_in=15, l_out=5, window_ratio=3):
    gids = np.ascontiguousarray(gids, dtype=np.int64)
    p = np.ascontiguousarray(pf, dtype=np.int64)
    ctr = np.zeros(8, dtype=np.int64)
    cov = ctypes.c_double(0.0)
    rc = lib().oracle_lru_prefetch(_p(gids, ctypes.c_int64), len(gids), int(total_ids),
                                   int(capacity), l_in, l_out, window_ratio,
                                   _p(p.reshape(-1), ctypes.c_int64), p.shape[1],
                                   _p(ctr, ctypes.c_int64), ctypes.byref(cov))
    if rc != 0:
        raise ValueError(f"oracle_lru_prefetch failed rc={rc}")
    return dict(zip(COUNTER_NAMES, (int(x) for x in ctr))), cov.value


def num_chunks(n, l_in=15, l_out=5, window_ratio=3):
    return int(lib().oracle_num_chunks(n, l_in, l_out, window_ratio))
