"""Device-resident engines over the C ABI: buffer replay (K3), LRU
comparator (K4) and the model pipeline (K1+K2 -> K3).  They own their
device allocations so repeated calls (the bench's steps, batch-by-batch
serving) allocate nothing; every launch is stream-ordered on torch's
current stream and nothing synchronises until ``*.result()``.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .trace import num_chunks


class BufferReplay:
    """recmg_replay: chunked replay through the priority buffer."""

    def __init__(self, capacity, total_ids, eviction_speed=4, ways=None, n=0, l_in=15,
                 l_out=5, window_ratio=3, pf_stride=0, policy=None):
        torch = _native.torch_cuda()
        L = _native.lib()
        self.torch = torch
        self.cfg = _native.buffer_cfg(capacity, ways, eviction_speed,
                                      _native.POLICY_PRIORITY if policy is None else policy,
                                      total_ids)
        sb = L.recmg_buffer_state_bytes(ctypes.byref(self.cfg))
        if sb == 0:
            _native.check(_native.RECMG_E_INVALID_CONFIG, "buffer config")
        self.state = _native.device_bytes(torch, sb)
        self.counters = torch.zeros(8, dtype=torch.int64, device="cuda")
        self.l_in, self.l_out, self.window_ratio = int(l_in), int(l_out), int(window_ratio)
        self._ws = None
        self._ws_key = None
        self._cov = None
        self.K = 0
        self.reserve(n, pf_stride)
        self.reset()

    def reserve(self, n, pf_stride):
        key = (int(n), int(pf_stride))
        if self._ws_key is not None and self._ws_key[0] >= key[0] and self._ws_key[1] >= key[1]:
            return
        sz = ctypes.c_size_t(0)
        _native.check(_native.lib().recmg_replay_workspace_bytes(
            ctypes.byref(self.cfg), key[0], self.l_in, self.l_out, self.window_ratio, key[1],
            ctypes.byref(sz)), "replay_workspace_bytes")
        self._ws = _native.device_bytes(self.torch, sz.value)
        K = num_chunks(key[0], self.l_in, self.l_out, self.window_ratio)
        self._cov = self.torch.empty((2, max(K, 1)), dtype=self.torch.int16, device="cuda")
        self._ws_key = key

    def reset(self):
        _native.check(_native.lib().recmg_buffer_reset(
            ctypes.byref(self.cfg), _native.ptr(self.state),
            _native.stream_handle(self.torch)), "buffer_reset")
        self.counters.zero_()

    def run(self, gids, bits=None, pf=None, access_class=None):
        """gids: device int32 [n]; bits uint8 [K, l_in]; pf int32 [K, stride]."""
        n = gids.numel()
        stride = int(pf.shape[1]) if pf is not None else 0
        self.reserve(n, stride)
        self.K = num_chunks(n, self.l_in, self.l_out, self.window_ratio)
        _native.check(_native.lib().recmg_replay(
            ctypes.byref(self.cfg), _native.ptr(self.state), _native.ptr(gids), n, self.l_in,
            self.l_out, self.window_ratio, _native.ptr(bits), _native.ptr(pf), stride,
            _native.ptr(self.counters), _native.ptr(self._cov[0]), _native.ptr(self._cov[1]),
            _native.ptr(access_class), _native.ptr(self._ws), self._ws.numel(),
            _native.stream_handle(self.torch)), "replay")

    def run_chunks(self, gids, k0, k1, with_tail, bits=None, pf=None, skip_stats=False):
        """Replay chunks [k0, k1) (+ tail) of the trace on the current state
        (recmg_replay_chunks_ex); consecutive ranges == one run().  skip_stats:
        the range's prefetch statistics were produced by stats_chunks()."""
        n = gids.numel()
        stride = int(pf.shape[1]) if pf is not None else 0
        self.reserve(n, stride)
        self.K = num_chunks(n, self.l_in, self.l_out, self.window_ratio)
        _native.check(_native.lib().recmg_replay_chunks_ex(
            ctypes.byref(self.cfg), _native.ptr(self.state), _native.ptr(gids), n, self.l_in,
            self.l_out, self.window_ratio, int(k0), int(k1), 1 if with_tail else 0,
            _native.ptr(bits), _native.ptr(pf), stride, _native.ptr(self.counters),
            _native.ptr(self._cov[0]), _native.ptr(self._cov[1]), None, _native.ptr(self._ws),
            self._ws.numel(), _native.REPLAY_SKIP_STATS if skip_stats else 0,
            _native.stream_handle(self.torch)), "replay_chunks")

    def run_chunks_lru(self, gids, k0, k1, with_tail, lru, bits=None, pf=None,
                       skip_stats=False):
        """run_chunks with the LRU comparator `lru` (an LruSim over the same sets)
        fused into the replay launch (recmg_replay_chunks_lru): it replays the
        serves of this replay's own events.  False (nothing launched) when the
        geometries do not allow it."""
        n = gids.numel()
        stride = int(pf.shape[1]) if pf is not None else 0
        self.reserve(n, stride)
        self.K = num_chunks(n, self.l_in, self.l_out, self.window_ratio)
        rc = _native.lib().recmg_replay_chunks_lru(
            ctypes.byref(self.cfg), _native.ptr(self.state), _native.ptr(gids), n, self.l_in,
            self.l_out, self.window_ratio, int(k0), int(k1), 1 if with_tail else 0,
            _native.ptr(bits), _native.ptr(pf), stride, _native.ptr(self.counters),
            _native.ptr(self._cov[0]), _native.ptr(self._cov[1]), ctypes.byref(lru.cfg),
            _native.ptr(lru.state), _native.ptr(lru.hm), _native.ptr(self._ws),
            self._ws.numel(), _native.REPLAY_SKIP_STATS if skip_stats else 0,
            _native.stream_handle(self.torch))
        if rc == _native.RECMG_E_INVALID_CONFIG:
            return False
        _native.check(rc, "replay_chunks_lru")
        return True

    def fusable_lru(self, lru):
        """Whether run_chunks_lru can carry `lru` (same sets and ways <= 32)."""
        a, b = self.cfg, lru.cfg
        if b.policy != _native.POLICY_LRU or a.policy != _native.POLICY_PRIORITY:
            return False
        if a.total_ids != b.total_ids or a.ways <= 0 or a.ways > 32 or b.ways != a.ways:
            return False
        return a.capacity // a.ways == b.capacity // b.ways and a.capacity // a.ways >= 2

    def stats_chunks(self, gids, k0, k1, pf=None):
        """Prefetch statistics (counters + coverage counts) of chunks [k0, k1)
        alone (recmg_prefetch_stats): they need the decoded ids, not the buffer."""
        n = gids.numel()
        stride = int(pf.shape[1]) if pf is not None else 0
        self.reserve(n, stride)
        self.K = num_chunks(n, self.l_in, self.l_out, self.window_ratio)
        _native.check(_native.lib().recmg_prefetch_stats(
            _native.ptr(gids), n, self.l_in, self.l_out, self.window_ratio, int(k0), int(k1),
            _native.ptr(pf), stride, _native.ptr(self.counters), _native.ptr(self._cov[0]),
            _native.ptr(self._cov[1]), _native.stream_handle(self.torch)), "prefetch_stats")

    def cov_host(self):
        """(num, den) uint16 arrays of the last run, copied to the host."""
        c = self._cov[:, :self.K].cpu().numpy().view(np.uint16)
        return c[0], c[1]

    def result(self, with_coverage=True):
        """Synchronise; counters dict plus the float64 coverage of the last run."""
        ctr = self.counters.cpu().numpy()
        out = dict(zip(_native.COUNTER_FIELDS, (int(x) for x in ctr)))
        if not with_coverage:
            return out
        if self.K:
            num, den = self.cov_host()
            out["coverage"] = _native.coverage_mean(num, den)
        else:
            out["coverage"] = 0.0
        return out


class SetSim:
    """recmg_simulate_ex: LRU / LFU / SRRIP / OPTGEN over set = gid % S
    (cache_sim.py:92-249), any ways per set."""

    POLICIES = {"lru": _native.POLICY_LRU, "lfu": _native.POLICY_LFU,
                "srrip": _native.POLICY_SRRIP, "optgen": _native.POLICY_OPTGEN}

    def __init__(self, capacity, total_ids, ways=None, n=0, policy="lru", srrip_max_rrpv=3):
        torch = _native.torch_cuda()
        L = _native.lib()
        self.torch = torch
        self.policy = policy
        self.cfg = _native.buffer_cfg(capacity, ways, srrip_max_rrpv if policy == "srrip" else 1,
                                      self.POLICIES[policy], total_ids)
        sb = L.recmg_buffer_state_bytes(ctypes.byref(self.cfg))
        if sb == 0:
            _native.check(_native.RECMG_E_INVALID_CONFIG, "cache config")
        self.state = _native.device_bytes(torch, sb)
        self.hm = torch.zeros(2, dtype=torch.int64, device="cuda")
        self._ws = None
        self._n = -1
        self.reserve(n)
        self.reset()

    def reserve(self, n):
        if n <= self._n:
            return
        sz = ctypes.c_size_t(0)
        _native.check(_native.lib().recmg_simulate_workspace_bytes(
            ctypes.byref(self.cfg), int(n), ctypes.byref(sz)), "simulate_workspace_bytes")
        self._ws = _native.device_bytes(self.torch, sz.value)
        self._n = int(n)

    def reset(self):
        _native.check(_native.lib().recmg_buffer_reset(
            ctypes.byref(self.cfg), _native.ptr(self.state),
            _native.stream_handle(self.torch)), "buffer_reset")
        self.hm.zero_()

    def run(self, gids, per_access_hit=None, keep=None):
        n = gids.numel()
        self.reserve(n)
        _native.check(_native.lib().recmg_simulate_ex(
            ctypes.byref(self.cfg), _native.ptr(self.state), _native.ptr(gids), n,
            _native.ptr(per_access_hit), _native.ptr(keep), _native.ptr(self.hm),
            _native.ptr(self._ws), self._ws.numel(), _native.stream_handle(self.torch)),
            "simulate")

    def result(self):
        h, m = (int(x) for x in self.hm.cpu().numpy())
        return h, m


class LruSim(SetSim):
    """The 32-way LRU comparator (K4)."""

    def __init__(self, capacity, total_ids, ways=None, n=0):
        super().__init__(capacity, total_ids, ways, n, "lru")


class RowStore:
    """Embedding rows of the buffered tables: all rows in pinned, mapped host
    memory (read by the GPU over PCIe through UVA), one HBM row per buffer
    slot.  refresh() (K5) copies the rows of slots whose occupant changed in
    the last replay; pool() (K6) is EmbeddingBag(sum) reading resident rows
    from HBM and the rest from host memory."""

    def __init__(self, replay: "BufferReplay", host_rows):
        torch = _native.torch_cuda()
        self.torch = torch
        if not host_rows.is_pinned():
            raise ValueError("host_rows must be pinned (torch.Tensor.pin_memory())")
        if host_rows.dtype != torch.float32 or host_rows.dim() != 2:
            raise ValueError("host_rows must be float32 [total_ids, dim]")
        self.replay = replay
        self.host = host_rows
        self.dim = int(host_rows.shape[1])
        cap = int(replay.cfg.capacity)
        self.buf = torch.zeros((cap, self.dim), dtype=torch.float32, device="cuda")
        self.loaded = torch.full((cap,), -1, dtype=torch.int32, device="cuda")
        self.copied = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.src = torch.zeros(2, dtype=torch.int64, device="cuda")

    def refresh(self, state=None):
        """state: a buffer state blob of this replay's geometry (default: the
        live one), e.g. a HotPath hook snapshot."""
        _native.check(_native.lib().recmg_rows_refresh(
            ctypes.byref(self.replay.cfg), _native.ptr(self.replay.state if state is None else state),
            _native.ptr(self.loaded), ctypes.c_void_p(self.host.data_ptr()), self.dim,
            _native.ptr(self.buf), _native.ptr(self.copied),
            _native.stream_handle(self.torch)), "rows_refresh")

    def pool(self, gids, offsets, out=None, state=None):
        n_bags = offsets.numel() - 1
        if out is None:
            out = self.torch.empty((n_bags, self.dim), dtype=self.torch.float32, device="cuda")
        _native.check(_native.lib().recmg_embedding_bag(
            ctypes.byref(self.replay.cfg),
            _native.ptr(self.replay.state if state is None else state), _native.ptr(gids),
            _native.ptr(offsets), n_bags, _native.ptr(self.buf),
            ctypes.c_void_p(self.host.data_ptr()), self.dim, _native.ptr(out),
            _native.ptr(self.src), _native.stream_handle(self.torch)), "embedding_bag")
        return out


def to_device_gids(torch, gids: np.ndarray):
    g = np.asarray(gids)
    if g.size and (g.min() < 0 or g.max() >= (1 << 30) - 1):
        raise ValueError("global ids must lie in [0, 2^30 - 1)")
    return torch.from_numpy(np.ascontiguousarray(g, dtype=np.int32)).cuda()
