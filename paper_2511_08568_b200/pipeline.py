"""HotPath: the whole per-access hot path resident on one GPU.

One object holds both models (K1/K2 weights in HBM), the buffer replay
engine (K3), the LRU comparator (K4) and every scratch buffer, so a replay
of a trace is a fixed sequence of stream-ordered launches with no
allocation and no host synchronisation until the report is read:

    tid      = recmg_table_ids(gids)                 (trace.py:86)
    bits     = K1 caching forward, logit >= 0        (runtime.py:181-193)
    pf       = K2 prefetch forward + fp64 decode     (runtime.py:196-210)
    counters = K3 replay(gids, bits, pf)             (runtime.py:220-283)
    lru      = K4 simulate(gids, C32 LRU, 32 ways)   (cache_sim.py:92-106)

``replay_host`` is the end-to-end entry (host gids in, BreakdownReport
out): H2D copy, the launches above, D2H of counters and per-chunk coverage
numerators, and the float64 coverage mean on the host.
"""
from __future__ import annotations

import numpy as np

from . import _native
from .engine import BufferReplay, LruSim
from .model import CACHING, PREFETCH, DeviceModel, ModelParameters
from .trace import num_chunks


class HotPath:
    STAGES = ("table_ids", "caching_fwd", "prefetch_fwd", "replay", "lru")

    def __init__(self, caching: ModelParameters | DeviceModel | None,
                 prefetch: ModelParameters | DeviceModel | None, table_sizes, capacity: int,
                 n_max: int, ways: int | None = 32, eviction_speed: int = 4,
                 lru_capacity: int | None = None, lru_ways: int | None = 32, l_in: int = 15,
                 l_out: int = 5, window_ratio: int = 3):
        torch = _native.torch_cuda()
        self.torch = torch
        self.table_sizes = [int(s) for s in table_sizes]
        self.total_ids = int(sum(self.table_sizes))
        self.caching = caching if (caching is None or isinstance(caching, DeviceModel)) \
            else DeviceModel(caching)
        self.prefetch = prefetch if (prefetch is None or isinstance(prefetch, DeviceModel)) \
            else DeviceModel(prefetch)
        for m, kind in ((self.caching, CACHING), (self.prefetch, PREFETCH)):
            if m is not None and (m.kind != kind or m.params.table_sizes != self.table_sizes):
                raise ValueError(f"{kind} model does not match the table layout")
        self.l_in, self.l_out, self.window_ratio = l_in, l_out, window_ratio
        self.n_max = int(n_max)
        self.K_max = num_chunks(self.n_max, l_in, l_out, window_ratio)
        from .trace import table_offsets
        self.offsets = torch.from_numpy(table_offsets(self.table_sizes)).cuda()
        self.gids = torch.empty(max(self.n_max, 1), dtype=torch.int32, device="cuda")
        self.tid = torch.empty(max(self.K_max * l_in, 1), dtype=torch.int32, device="cuda")
        self.bits = torch.empty((max(self.K_max, 1), l_in), dtype=torch.uint8, device="cuda")
        self.pf = torch.empty((max(self.K_max, 1), l_out), dtype=torch.int32, device="cuda")
        self.clog = torch.empty((max(self.K_max, 1), l_in), dtype=torch.float32, device="cuda")
        self.plog = torch.empty((max(self.K_max, 1), l_out), dtype=torch.float32, device="cuda")
        self.buffer = BufferReplay(capacity, self.total_ids, eviction_speed, ways, self.n_max,
                                   l_in, l_out, window_ratio,
                                   l_out if self.prefetch is not None else 0)
        self.lru = None
        if lru_capacity:
            self.lru = LruSim(lru_capacity, self.total_ids, lru_ways, self.n_max)
        self.events = None

    def enable_stage_timing(self, on=True):
        t = self.torch
        self.events = [(t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True))
                       for _ in self.STAGES] if on else None
        self.stage_ms = {s: [] for s in self.STAGES}

    def _mark(self, i, end):
        if self.events is not None:
            self.events[i][1 if end else 0].record()

    def collect_stage_times(self):
        if self.events is None:
            return
        for i, s in enumerate(self.STAGES):
            a, b = self.events[i]
            self.stage_ms[s].append(a.elapsed_time(b))

    def launch(self, n: int):
        """Stream-ordered launches over self.gids[:n] (device-resident)."""
        L = _native.lib()
        K = num_chunks(n, self.l_in, self.l_out, self.window_ratio)
        g = self.gids[:n]
        bits = pf = None
        self.buffer.reset()
        if self.lru is not None:
            self.lru.reset()
        self._mark(0, False)
        if K and (self.caching is not None or self.prefetch is not None):
            gk = g[:K * self.l_in].view(K, self.l_in)
            tk = self.tid[:K * self.l_in].view(K, self.l_in)
            _native.check(L.recmg_table_ids(_native.ptr(gk), K * self.l_in,
                                            _native.ptr(self.offsets), len(self.table_sizes),
                                            _native.ptr(tk), _native.stream_handle(self.torch)))
        self._mark(0, True)
        self._mark(1, False)
        if K and self.caching is not None:
            bits = self.bits[:K]
            self.caching.forward(gk, tk, logits=self.clog[:K], bits=bits)
        self._mark(1, True)
        self._mark(2, False)
        if K and self.prefetch is not None:
            pf = self.pf[:K]
            self.prefetch.forward(gk, tk, logits=self.plog[:K], pf_gid=pf)
        self._mark(2, True)
        self._mark(3, False)
        self.buffer.run(g, bits, pf)
        self._mark(3, True)
        self._mark(4, False)
        if self.lru is not None:
            self.lru.run(g)
        self._mark(4, True)
        self.K = K
        self.n = n

    def report(self):
        """Synchronise and return (BreakdownReport, lru (hits, misses) or None)."""
        from .runtime import BreakdownReport
        r = self.buffer.result()
        rep = BreakdownReport(r["cache_hits"], r["prefetch_hits"], r["on_demand"],
                              r["prefetch_issued"], r["prefetch_useful"], r["coverage"],
                              r["evictions"], r["prefetch_inserts"])
        lru = self.lru.result() if self.lru is not None else None
        return rep, lru

    def replay_host(self, host_gids):
        """End to end: pinned/host int32 gids -> BreakdownReport (+ LRU)."""
        n = int(host_gids.numel()) if hasattr(host_gids, "numel") else len(host_gids)
        if n > self.n_max:
            raise ValueError("trace longer than the HotPath was sized for")
        src = host_gids if hasattr(host_gids, "numel") else self.torch.from_numpy(
            np.ascontiguousarray(host_gids, dtype=np.int32))
        self.gids[:n].copy_(src, non_blocking=True)
        self.launch(n)
        return self.report()

    def d2h_bytes(self):
        """Bytes read back per replay_host: counters, LRU pair, coverage num/den."""
        return 8 * 8 + (16 if self.lru is not None else 0) + 2 * self.K
