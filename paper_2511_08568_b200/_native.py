"""ctypes binding of librecmg.so (the C ABI in include/recmg.h).

The product path has no CPU fallback: every compute entry point needs the
in-tree librecmg.so *and* a CUDA device, and raises otherwise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import (CheckpointError, EmbcacheError, InvalidConfigError, NumericalError,
                     OutOfVocabularyError, VocabularyMismatchError)

_HERE = os.path.dirname(os.path.abspath(__file__))
# RECMG_LIB: an alternative in-tree build of the same ABI (A/B timing of kernel variants)
LIB_PATH = os.path.join(_HERE, os.environ.get("RECMG_LIB", "librecmg.so"))

RECMG_OK = 0
RECMG_E_INVALID_CONFIG = -1
RECMG_E_VOCAB_MISMATCH = -2
RECMG_E_OUT_OF_VOCAB = -3
RECMG_E_BUFFER_STATE = -4
RECMG_E_NON_FINITE = -5
RECMG_E_CUDA = -6
RECMG_E_WORKSPACE = -7

POLICY_PRIORITY = 0
POLICY_LRU = 1
POLICY_LRU_PF = 2
POLICY_LFU = 3
POLICY_SRRIP = 4
POLICY_OPTGEN = 5
OP_ADD, OP_POPULATE, OP_REFERENCE, OP_SET_PRIORITY, OP_QUERY = range(5)
MODEL_CACHING, MODEL_PREFETCH = 0, 1
PREC_FP32 = 0
PREC_TC32 = 1
REPLAY_SKIP_STATS = 1   # recmg.h RECMG_REPLAY_SKIP_STATS
PREC_TC16 = 2

# every symbol include/recmg.h declares (tests check the export table)
EXPORTS = (
    "recmg_status_string", "recmg_status_category", "recmg_buffer_state_bytes",
    "recmg_buffer_reset", "recmg_num_chunks", "recmg_replay_workspace_bytes", "recmg_replay",
    "recmg_coverage_mean", "recmg_simulate_workspace_bytes", "recmg_simulate",
    "recmg_buffer_op", "recmg_model_dense_floats", "recmg_model_packed_bytes",
    "recmg_model_pack", "recmg_model_forward", "recmg_table_ids", "recmg_trace_pool_pass",
    "recmg_launch_count", "recmg_selftest_umma", "recmg_model_pack_tc",
    "recmg_model_workspace_bytes", "recmg_replay_chunks", "recmg_set_model_sm_budget",
    "recmg_model_forward_profile", "recmg_rows_refresh", "recmg_embedding_bag",
    "recmg_simulate_ex", "recmg_model_forward_ex", "recmg_pcg64_uniforms", "recmg_trace_guide",
    "recmg_trace_generate_block", "recmg_shard_local_ids", "recmg_trace_parse_text",
    "recmg_coverage_accumulate", "recmg_embedding_bag_a2a", "recmg_peer_alloc",
    "recmg_peer_free", "recmg_peer_handle", "recmg_peer_open", "recmg_peer_close",
    "recmg_replay_chunks_lru",
    "recmg_model_forward_signal", "recmg_wait_progress", "recmg_replay_chunks_ex",
    "recmg_prefetch_stats",
)


class BufferCfg(ctypes.Structure):
    _fields_ = [("capacity", ctypes.c_int64), ("ways", ctypes.c_int32),
                ("eviction_speed", ctypes.c_int32), ("policy", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("total_ids", ctypes.c_int64)]


class ModelShape(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("dim", ctypes.c_int32), ("stacks", ctypes.c_int32),
                ("l_in", ctypes.c_int32), ("l_out", ctypes.c_int32),
                ("n_tables", ctypes.c_int32), ("total_ids", ctypes.c_int64)]


COUNTER_FIELDS = ("cache_hits", "prefetch_hits", "on_demand", "prefetch_issued",
                  "prefetch_useful", "evictions", "prefetch_inserts", "occupancy")

_lib = None


def lib():
    """Load librecmg.so (loudly: no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (make -C paper_2511_08568_b200/csrc)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
    cfgp, shp = ctypes.POINTER(BufferCfg), ctypes.POINTER(ModelShape)
    sig = {
        "recmg_status_string": (ctypes.c_char_p, [ctypes.c_int]),
        "recmg_status_category": (ctypes.c_char_p, [ctypes.c_int]),
        "recmg_buffer_state_bytes": (sz, [cfgp]),
        "recmg_buffer_reset": (ctypes.c_int, [cfgp, vp, vp]),
        "recmg_num_chunks": (i64, [i64, i32, i32, i32]),
        "recmg_replay_workspace_bytes": (ctypes.c_int, [cfgp, i64, i32, i32, i32, i32,
                                                        ctypes.POINTER(sz)]),
        "recmg_replay": (ctypes.c_int, [cfgp, vp, vp, i64, i32, i32, i32, vp, vp, i32, vp, vp,
                                        vp, vp, vp, sz, vp]),
        "recmg_coverage_mean": (ctypes.c_double, [vp, vp, i64]),
        "recmg_coverage_accumulate": (ctypes.c_double, [vp, vp, i64, ctypes.c_double]),
        "recmg_embedding_bag_a2a": (ctypes.c_int, [cfgp, vp, vp, vp, i64, vp, vp, i32, i32, i32,
                                                   i32, i32, vp, vp, vp, vp, ctypes.c_uint64,
                                                   vp, vp]),
        "recmg_peer_alloc": (ctypes.c_int, [sz, ctypes.POINTER(ctypes.c_void_p)]),
        "recmg_peer_free": (ctypes.c_int, [vp]),
        "recmg_peer_handle": (ctypes.c_int, [vp, ctypes.c_char_p]),
        "recmg_peer_open": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
        "recmg_peer_close": (ctypes.c_int, [vp]),
        "recmg_replay_chunks": (ctypes.c_int, [cfgp, vp, vp, i64, i32, i32, i32, i64, i64, i32,
                                               vp, vp, i32, vp, vp, vp, vp, vp, sz, vp]),
        "recmg_replay_chunks_ex": (ctypes.c_int, [cfgp, vp, vp, i64, i32, i32, i32, i64, i64,
                                                  i32, vp, vp, i32, vp, vp, vp, vp, vp, sz, i32,
                                                  vp]),
        "recmg_replay_chunks_lru": (ctypes.c_int, [cfgp, vp, vp, i64, i32, i32, i32, i64, i64,
                                                   i32, vp, vp, i32, vp, vp, vp, cfgp, vp, vp,
                                                   vp, sz, i32, vp]),
        "recmg_prefetch_stats": (ctypes.c_int, [vp, i64, i32, i32, i32, i64, i64, vp, i32, vp,
                                                vp, vp, vp]),
        "recmg_set_model_sm_budget": (ctypes.c_int, [ctypes.c_int]),
        "recmg_rows_refresh": (ctypes.c_int, [cfgp, vp, vp, vp, i32, vp, vp, vp]),
        "recmg_embedding_bag": (ctypes.c_int, [cfgp, vp, vp, vp, i64, vp, vp, i32, vp, vp, vp]),
        "recmg_model_forward_profile": (ctypes.c_int, [shp, vp, vp, vp, i64, vp, vp, sz, vp, vp]),
        "recmg_simulate_workspace_bytes": (ctypes.c_int, [cfgp, i64, ctypes.POINTER(sz)]),
        "recmg_simulate": (ctypes.c_int, [cfgp, vp, vp, i64, vp, vp, vp, sz, vp]),
        "recmg_simulate_ex": (ctypes.c_int, [cfgp, vp, vp, i64, vp, vp, vp, vp, sz, vp]),
        "recmg_buffer_op": (ctypes.c_int, [cfgp, vp, i32, i64, i64, i32, vp, vp]),
        "recmg_model_dense_floats": (i64, [shp]),
        "recmg_model_packed_bytes": (sz, [shp, i32]),
        "recmg_model_pack": (ctypes.c_int, [shp, vp, vp, i32, vp]),
        "recmg_model_forward": (ctypes.c_int, [shp, i32, vp, vp, vp, vp, i64, vp, vp, vp, vp,
                                               sz, vp]),
        "recmg_model_forward_ex": (ctypes.c_int, [shp, i32, vp, vp, vp, vp, i64, i64, vp, vp,
                                                  vp, vp, sz, vp]),
        "recmg_model_forward_signal": (ctypes.c_int, [shp, i32, vp, vp, vp, vp, i64, i64, vp,
                                                      vp, vp, vp, sz, vp, i64, vp]),
        "recmg_wait_progress": (ctypes.c_int, [vp, i64, i32, vp]),
        "recmg_trace_parse_text": (ctypes.c_int, [vp, i64, i64, vp, i32, vp, i64, vp, vp, vp]),
        "recmg_shard_local_ids": (ctypes.c_int, [vp, i64, vp, i32, vp, vp, vp, vp, vp]),
        "recmg_pcg64_uniforms": (ctypes.c_int, [vp, i64, i64, vp, i32]),
        "recmg_trace_guide": (ctypes.c_int, [vp, i64, i32, vp]),
        "recmg_trace_generate_block": (ctypes.c_int, [vp, i64, i64, i64, vp, i64, vp, i32, vp,
                                                      ctypes.c_double, i32, vp, vp, vp, i32]),
        "recmg_model_pack_tc": (ctypes.c_int, [shp, vp, vp, vp, vp, vp]),
        "recmg_model_workspace_bytes": (sz, [shp, i32, i64]),
        "recmg_table_ids": (ctypes.c_int, [vp, i64, vp, i32, vp, vp]),
        "recmg_trace_pool_pass": (ctypes.c_int, [vp, vp, vp, i64, ctypes.c_double, i32, vp]),
        "recmg_launch_count": (ctypes.c_uint64, []),
        "recmg_selftest_umma": (ctypes.c_int, [vp, vp, vp, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_int, vp]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("RECMG_LIB") and not hasattr(L, name):
            continue   # an older A/B build without this entry point
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(rc: int, what: str = "recmg"):
    """Map a status code onto the reference's exception taxonomy (errors.py)."""
    if rc == RECMG_OK:
        return
    msg = f"{what}: {lib().recmg_status_string(rc).decode()}"
    if rc == RECMG_E_INVALID_CONFIG:
        raise InvalidConfigError(msg)
    if rc == RECMG_E_VOCAB_MISMATCH:
        raise VocabularyMismatchError(msg)
    if rc == RECMG_E_OUT_OF_VOCAB:
        raise OutOfVocabularyError(msg)
    if rc == RECMG_E_BUFFER_STATE:
        raise ValueError(msg)
    if rc == RECMG_E_NON_FINITE:
        raise NumericalError(msg)
    raise EmbcacheError(msg)


def torch_cuda():
    """torch with a usable CUDA device, or a loud error (no CPU fallback)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2511_08568_b200 needs a CUDA (B200) device; "
                           "there is no CPU fallback on the product path")
    lib()
    return torch


def stream_handle(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def device_bytes(torch, nbytes: int):
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device="cuda")


def buffer_cfg(capacity, ways, eviction_speed, policy, total_ids) -> BufferCfg:
    return BufferCfg(int(capacity), int(ways or 0), int(eviction_speed), int(policy), 0,
                     int(total_ids))


def pool_pass(zipf_gids: np.ndarray, sticky: np.ndarray, pool_coin: np.ndarray,
              stickiness: float, pool_size: int) -> np.ndarray:
    """Host sequential pass of generate_trace (trace.py:144-160), in C."""
    z = np.ascontiguousarray(zipf_gids, dtype=np.int64)
    a = np.ascontiguousarray(sticky, dtype=np.float64)
    b = np.ascontiguousarray(pool_coin, dtype=np.float64)
    out = np.empty(len(z), dtype=np.int64)
    rc = lib().recmg_trace_pool_pass(z.ctypes.data, a.ctypes.data, b.ctypes.data, len(z),
                                     float(stickiness), int(pool_size), out.ctypes.data)
    check(rc, "trace_pool_pass")
    return out


def coverage_mean(num: np.ndarray, den: np.ndarray) -> float:
    num = np.ascontiguousarray(num, dtype=np.uint16)
    den = np.ascontiguousarray(den, dtype=np.uint16)
    return float(lib().recmg_coverage_mean(num.ctypes.data, den.ctypes.data, len(num)))


__all__ = ["lib", "check", "EXPORTS", "BufferCfg", "ModelShape", "CheckpointError"]
