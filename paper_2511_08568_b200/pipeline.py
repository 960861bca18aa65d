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

import os

import numpy as np

from . import _native
from .engine import BufferReplay, LruSim
from .model import CACHING, PREFETCH, DeviceModel, ModelParameters
from .trace import num_chunks


# Per piece the prefetch forward runs before the caching forward, so each
# piece's replay (side stream) overlaps the next piece's prefetch forward
# rather than the caching forward, whose L2-resident attention scratch is the
# more sensitive to the replay's event streams (config 2: +0.9% per step, two
# A/B pairs).  RECMG_PF_FIRST=0 restores caching-first for A/B runs.
_PF_FIRST = os.environ.get("RECMG_PF_FIRST", "1") == "1"
# Streamed mode (the default for a plain pieces > 1 replay): each model runs
# ONE forward over the whole trace and the second one releases a per-piece
# progress counter as its tiles finish (recmg_model_forward_signal); piece i's
# replay waits on that counter (recmg_wait_progress) on the replay stream.
# The forwards then never end between pieces, so the replay's kernels cannot
# take the SMs a forward launch boundary frees (measured with 8 per-piece
# launch pairs: +36% prefetch / +4% caching forward time).  RECMG_STREAMED=0
# restores per-piece forward launches.
_STREAMED = os.environ.get("RECMG_STREAMED", "0") == "1"
# replay_host() through a CUDA graph of the step's launches (see there)
_GRAPHS = os.environ.get("RECMG_GRAPHS", "1") == "1"
# In the serial schedule the LRU comparator is launched after the forwards (it
# then shares the GPU with the replay) instead of at the start, where its
# kernels take SMs at the forward launch boundary (config 2: +1.8%).
_LRU_LATE = os.environ.get("RECMG_LRU_LATE", "1") == "1"
_LRU_PRIO = os.environ.get("RECMG_LRU_PRIO", "1") == "1"
# Serial schedule: the LRU comparator runs inside the replay launch, on the
# serves of the replay's own partitioned events (recmg_replay_chunks_lru), so
# it builds and partitions no events of its own (RECMG_LRU_FUSED=0: its own
# launches on the LRU stream)
_LRU_FUSED = os.environ.get("RECMG_LRU_FUSED", "1") == "1"


class HotPath:
    STAGES = ("table_ids", "caching_fwd", "prefetch_fwd", "replay", "lru", "tail", "hook")

    def __init__(self, caching: ModelParameters | DeviceModel | None,
                 prefetch: ModelParameters | DeviceModel | None, table_sizes, capacity: int,
                 n_max: int, ways: int | None = 32, eviction_speed: int = 4,
                 lru_capacity: int | None = None, lru_ways: int | None = 32, l_in: int = 15,
                 l_out: int = 5, window_ratio: int = 3, pieces: int | None = None,
                 model_sms: int = 136,
                 shard=None, replay_priority: bool = True, piece_chunks: int | None = None,
                 piece_hook=None, hook_snapshot: bool = True):
        """pieces = None picks the schedule from the buffer geometry: one
        replay after both forwards (pieces = 1, `_launch_serial`) when the
        buffer has at least 256 sets -- the replay is then throughput-bound and
        a replay beside the forwards only takes SMs they need -- and 8 pipelined
        pieces for fewer, longer sets (the fully associative buffer: one chain
        that only hides under the forwards).

        pieces > 1 pipelines the replay: chunks are scored in `pieces`
        ranges on the main stream while earlier ranges replay on a side stream
        (recmg_replay_chunks continues the buffer state, so the result is the
        same as one replay); the LRU comparator runs on a third stream from
        the start.  The TC forwards then use `model_sms` SMs, leaving the rest
        to the replay CTAs.  piece_chunks fixes the piece length in chunks (a
        serving batch) instead of dividing the trace into `pieces`;
        piece_hook(k0, k1, last, state) runs after each piece's replay (the
        DLRM embedding stage: K5 row refresh + K6 pooling of that batch) on the
        buffer state as that replay left it, so it overlaps the next piece's
        forwards.  With hook_snapshot (the default) the state is a copy taken
        on the replay stream (double-buffered, 5 MB at config 2) and the hook
        runs on its own stream, so the next piece's replay overlaps this
        piece's hook as well (the hook sees exactly the state it would see
        in line; config 4: the replay stream no longer carries replay + K5 +
        K6 per batch); without it, the hook runs in line on the replay stream
        with state = the live buffer state.

        shard (shard.TableShard): the models are a table shard's, packed over
        its local vocabulary (shard.init_params_shard, DeviceModel with
        decode_ids = the global id count); the forwards then read local ids
        made on the device by recmg_shard_local_ids, the replay global ones."""
        torch = _native.torch_cuda()
        self.torch = torch
        self.table_sizes = [int(s) for s in table_sizes]
        self.total_ids = int(sum(self.table_sizes))
        self.caching = caching if (caching is None or isinstance(caching, DeviceModel)) \
            else DeviceModel(caching)
        self.prefetch = prefetch if (prefetch is None or isinstance(prefetch, DeviceModel)) \
            else DeviceModel(prefetch)
        self.shard = shard
        model_sizes = self.table_sizes if shard is None else list(shard.local_sizes)
        if shard is not None and list(shard.table_sizes) != self.table_sizes:
            raise ValueError("shard does not match the table layout")
        for m, kind in ((self.caching, CACHING), (self.prefetch, PREFETCH)):
            if m is not None and (m.kind != kind or m.params.table_sizes != model_sizes):
                raise ValueError(f"{kind} model does not match the table layout")
            if m is not None and shard is not None and m.decode_ids != shard.total_ids:
                raise ValueError(f"{kind} shard model must decode over the global ids")
        self.l_in, self.l_out, self.window_ratio = l_in, l_out, window_ratio
        self.n_max = int(n_max)
        self.K_max = num_chunks(self.n_max, l_in, l_out, window_ratio)
        from .trace import table_offsets
        self.offsets = torch.from_numpy(table_offsets(self.table_sizes)).cuda()
        self.gids = torch.empty(max(self.n_max, 1), dtype=torch.int32, device="cuda")
        self.tid = torch.empty(max(self.K_max * l_in, 1), dtype=torch.int32, device="cuda")
        self.lgid = None
        if shard is not None:
            self.lgid = torch.empty(max(self.K_max * l_in, 1), dtype=torch.int32, device="cuda")
            self.table_local = torch.from_numpy(shard.table_local).cuda()
            self.local_offsets = torch.from_numpy(shard.local_offsets).cuda()
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
        if pieces is None:
            sets = capacity // (ways or capacity) if capacity else 1
            pieces = 1 if sets >= 256 else 8
        self.pieces = max(1, int(pieces))
        self.piece_chunks = int(piece_chunks) if piece_chunks else None
        self.piece_hook = piece_hook
        self.hook_snapshot = bool(hook_snapshot) and piece_hook is not None
        self.model_sms = int(model_sms) if (self.pieces > 1 or self.piece_chunks) else 148
        # the replay and the LRU run under the forwards on the SMs they leave;
        # high priority makes the block scheduler hand freed SMs to them first
        # (at every forward launch boundary), so the replay does not lag
        prio = torch.cuda.Stream.priority_range()[1] if replay_priority else 0
        self.s_replay = torch.cuda.Stream(priority=prio)
        self.s_copy = torch.cuda.Stream()
        self.cov_host = torch.empty((2, max(self.K_max, 1)), dtype=torch.int16, pin_memory=True)
        self._cov_events = []
        # the LRU comparator yields the SMs to the replay's own event build and
        # partition (RECMG_LRU_PRIO=1: the replay stream's priority)
        self.s_lru = torch.cuda.Stream(priority=prio if _LRU_PRIO else 0)
        self.s_hook = torch.cuda.Stream(priority=prio) if self.hook_snapshot else None
        self._snaps = ([torch.empty_like(self.buffer.state) for _ in range(2)]
                       if self.hook_snapshot else None)
        self.events = None
        self.stage_ms = {}

    def enable_stage_timing(self, on=True):
        self.events = {} if on else None

    def _ev(self, key, stream):
        if self.events is None:
            return
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(stream)
        self.events.setdefault(key, []).append(e)

    def stage_times(self):
        """ms per stage of the last launch (sum over pieces; stages overlap)."""
        out = {}
        for s in self.STAGES:
            ev = self.events.get(s, []) if self.events else []
            out[s] = sum(ev[i].elapsed_time(ev[i + 1]) for i in range(0, len(ev) - 1, 2))
        return out

    def _piece_bounds(self, K):
        if self.piece_chunks:
            b = list(range(0, K, self.piece_chunks)) + [K]
            return [(b[i], b[i + 1]) for i in range(len(b) - 1)]
        if self.pieces <= 1 or K < 128 * self.pieces:
            return [(0, K)]
        step = (K // self.pieces + 127) // 128 * 128
        b = list(range(0, K, step)) + [K]
        return [(b[i], b[i + 1]) for i in range(len(b) - 1)]

    def _ids_of(self, g, k0, k1):
        """(ids the forwards read, table ids) of chunks [k0, k1): recmg_table_ids,
        or for a table shard recmg_shard_local_ids (global -> local rows)."""
        torch = self.torch
        L = _native.lib()
        m = (k1 - k0) * self.l_in
        gk = g[k0 * self.l_in:k1 * self.l_in].view(k1 - k0, self.l_in)
        tk = self.tid[k0 * self.l_in:k1 * self.l_in].view(k1 - k0, self.l_in)
        if self.shard is None:
            _native.check(L.recmg_table_ids(
                _native.ptr(gk), m, _native.ptr(self.offsets), len(self.table_sizes),
                _native.ptr(tk), _native.stream_handle(torch)))
            return gk, tk
        lk = self.lgid[k0 * self.l_in:k1 * self.l_in].view(k1 - k0, self.l_in)
        _native.check(L.recmg_shard_local_ids(
            _native.ptr(gk), m, _native.ptr(self.offsets), len(self.table_sizes),
            _native.ptr(self.table_local), _native.ptr(self.local_offsets), _native.ptr(lk),
            _native.ptr(tk), _native.stream_handle(torch)))
        return lk, tk

    def launch(self, n: int, host_src=None):
        """Stream-ordered launches over self.gids[:n].

        host_src (pinned host int32 ids, the end-to-end path): the ids are
        copied in two parts on a copy stream -- the first piece's chunks, then
        the rest -- so the first forwards start after a fraction of the H2D
        copy; every piece's per-chunk coverage counts are copied back as soon
        as its replay is done, so report() sums them while later pieces run."""
        torch = self.torch
        L = _native.lib()
        K = num_chunks(n, self.l_in, self.l_out, self.window_ratio)
        g = self.gids[:n]
        main = torch.cuda.current_stream()
        pieces = self._piece_bounds(K) if K else [(0, 0)]
        has_models = self.caching is not None or self.prefetch is not None
        serial = (K > 0 and has_models and len(pieces) == 1 and self.piece_hook is None
                  and not self.piece_chunks)
        # serial mode: the first forward starts after the first eighth of the ids
        serial_split = min(K, (K // 8 + 127) // 128 * 128) if (serial and host_src is not None) \
            else K
        all_ids = torch.cuda.Event()
        if host_src is not None:
            first = (min(n, serial_split * self.l_in) if serial else
                     min(n, pieces[0][1] * self.l_in) if K else n)
            self.s_copy.wait_stream(main)       # earlier readers of self.gids
            first_ids = torch.cuda.Event()
            with torch.cuda.stream(self.s_copy):
                self.gids[:first].copy_(host_src[:first], non_blocking=True)
                first_ids.record(self.s_copy)
                if n > first:
                    self.gids[first:n].copy_(host_src[first:n], non_blocking=True)
                all_ids.record(self.s_copy)
            main.wait_event(first_ids)
        else:
            all_ids.record(main)
        self._cov_events = []
        hook_done = [None, None]   # per snapshot slot: the hook that last read it
        # K4: the LRU comparator depends only on the ids
        def run_lru(after):
            self.s_lru.wait_event(after)
            with torch.cuda.stream(self.s_lru):
                self._ev("lru", self.s_lru)
                self.lru.reset()
                self.lru.run(g)
                self._ev("lru", self.s_lru)

        # late only in the serial schedule: pipelined runs (few-set buffers, config
        # 3's one-hot-set shards) have chain-bound LRUs that must hide under the forwards
        # (every schedule but the streamed one: each replay call carries the
        # comparator over its chunk range, the states continue across calls)
        self._lru_fused = (_LRU_FUSED and self.lru is not None and K > 0 and has_models
                           and not (_STREAMED and len(pieces) > 1 and self.piece_hook is None
                                    and not self.piece_chunks)
                           and self.buffer.fusable_lru(self.lru))
        lru_late = _LRU_LATE and self.lru is not None and serial and not self._lru_fused
        # (the SM budget first: a replay-engine launch made under a budget below
        # the SM count -- beside the forwards -- spreads over every free SM)
        prev = L.recmg_set_model_sm_budget(self.model_sms)
        try:
            if self.lru is not None and not lru_late and not self._lru_fused:
                run_lru(all_ids)
            self.s_replay.wait_event(all_ids)
            with torch.cuda.stream(self.s_replay):
                self.buffer.reset()
                if self._lru_fused:
                    self.lru.reset()
            bits = self.bits[:K] if (K and self.caching is not None) else None
            pf = self.pf[:K] if (K and self.prefetch is not None) else None
            models = K > 0 and (self.caching is not None or self.prefetch is not None)
            # table ids in (at most) two launches: the first piece's as soon as
            # its ids are in, the rest once all ids are
            split = pieces[0][1] if host_src is not None else K
            if serial:
                split = serial_split
            if models:
                self._ev("table_ids", main)
                gk, tk = self._ids_of(g, 0, split)
                self._ev("table_ids", main)
            if serial:
                self._launch_serial(g, K, host_src, all_ids, main, bits, pf, split)
                pieces = []
            streamed = (_STREAMED and models and len(pieces) > 1 and self.piece_hook is None
                        and not self.piece_chunks and all(
                            m is None or m.prec in (_native.PREC_TC32, _native.PREC_TC16)
                            for m in (self.caching, self.prefetch)))
            if streamed:
                self._launch_streamed(g, K, pieces, host_src, all_ids, main, bits, pf, split)
                pieces = []
            for i, (k0, k1) in enumerate(pieces):
                if i == 1 and host_src is not None:
                    main.wait_event(all_ids)
                    if models:
                        self._ev("table_ids", main)
                        self._ids_of(g, split, K)
                        self._ev("table_ids", main)
                if k1 > k0 and models:
                    gk = (self.lgid if self.shard is not None else self.gids)[
                        :K * self.l_in].view(K, self.l_in)
                    tk = self.tid[:K * self.l_in].view(K, self.l_in)
                    def fwd_caching():
                        self._ev("caching_fwd", main)
                        self.caching.forward(gk[k0:k1], tk[k0:k1], logits=self.clog[k0:k1],
                                             bits=self.bits[k0:k1])
                        self._ev("caching_fwd", main)

                    def fwd_prefetch():
                        self._ev("prefetch_fwd", main)
                        self.prefetch.forward(gk[k0:k1], tk[k0:k1], logits=self.plog[k0:k1],
                                              pf_gid=self.pf[k0:k1])
                        self._ev("prefetch_fwd", main)

                    order = ((fwd_prefetch, self.prefetch), (fwd_caching, self.caching)) \
                        if _PF_FIRST else ((fwd_caching, self.caching), (fwd_prefetch, self.prefetch))
                    for fn, model in order:
                        if model is not None:
                            fn()
                scored = torch.cuda.Event()
                scored.record(main)
                self.s_replay.wait_event(scored)
                with torch.cuda.stream(self.s_replay):
                    self._ev("replay", self.s_replay)
                    last = i == len(pieces) - 1
                    if not (self._lru_fused and self.buffer.run_chunks_lru(
                            g, k0, k1, last, self.lru, bits, pf)):
                        self.buffer.run_chunks(g, k0, k1, last, bits, pf)
                        if self._lru_fused:
                            raise RuntimeError("recmg_replay_chunks_lru refused a fusable LRU")
                    self._ev("replay", self.s_replay)
                    if self.piece_hook is not None and not self.hook_snapshot:
                        self._ev("hook", self.s_replay)
                        self.piece_hook(k0, k1, i == len(pieces) - 1, self.buffer.state)
                        self._ev("hook", self.s_replay)
                    if self.hook_snapshot:
                        slot = i & 1
                        if hook_done[slot] is not None:   # the hook two pieces back is done with it
                            self.s_replay.wait_event(hook_done[slot])
                        self._snaps[slot].copy_(self.buffer.state, non_blocking=True)
                        snapped = torch.cuda.Event()
                        snapped.record(self.s_replay)
                    if host_src is not None and k1 > k0:
                        for r in range(2):   # contiguous rows: plain async D2H copies
                            self.cov_host[r, k0:k1].copy_(self.buffer._cov[r, k0:k1],
                                                          non_blocking=True)
                        e = torch.cuda.Event(external=True)   # an event node in a graph
                        e.record(self.s_replay)
                        self._cov_events.append((k0, k1, e))
                if self.hook_snapshot:
                    self.s_hook.wait_event(snapped)
                    with torch.cuda.stream(self.s_hook):
                        self._ev("hook", self.s_hook)
                        self.piece_hook(k0, k1, i == len(pieces) - 1, self._snaps[slot])
                        self._ev("hook", self.s_hook)
                        hook_done[slot] = torch.cuda.Event()
                        hook_done[slot].record(self.s_hook)
        finally:
            L.recmg_set_model_sm_budget(prev)
        if lru_late:   # after the forwards: beside the replay's single-warp chain
            fwd_done = torch.cuda.Event()
            fwd_done.record(main)
            run_lru(fwd_done)
        self._ev("tail", main)          # forwards done ...
        main.wait_stream(self.s_replay)
        if self.s_hook is not None:
            main.wait_stream(self.s_hook)
        if self.lru is not None and not self._lru_fused:
            main.wait_stream(self.s_lru)
        self._ev("tail", main)          # ... -> last replay piece and LRU done
        self.K = K
        self.n = n

    def _launch_serial(self, g, K, host_src, all_ids, main, bits, pf, split):
        """One replay after both forwards (pieces == 1; measured the fastest
        schedule: a replay beside the forwards takes the SMs they need, the
        replay and forwards are both throughput-bound).  The prefetch forward
        runs first (in two launches on the end-to-end path: the first eighth
        starts once its ids are in); its prefetch statistics and coverage counts
        need only the decoded ids, so they run right after it on the replay
        stream and are copied back while the caching forward runs."""
        torch = self.torch
        gk = (self.lgid if self.shard is not None else self.gids)[
            :K * self.l_in].view(K, self.l_in)
        tk = self.tid[:K * self.l_in].view(K, self.l_in)

        def fwd(model, k0, k1):
            if model is None or k1 <= k0:
                return
            if model is self.caching:
                self._ev("caching_fwd", main)
                model.forward(gk[k0:k1], tk[k0:k1], logits=self.clog[k0:k1],
                              bits=self.bits[k0:k1])
                self._ev("caching_fwd", main)
            else:
                self._ev("prefetch_fwd", main)
                model.forward(gk[k0:k1], tk[k0:k1], logits=self.plog[k0:k1],
                              pf_gid=self.pf[k0:k1])
                self._ev("prefetch_fwd", main)

        first, second = ((self.prefetch, self.caching) if self.prefetch is not None
                         else (self.caching, None))
        fwd(first, 0, split)
        if split < K:
            main.wait_event(all_ids)
            self._ev("table_ids", main)
            self._ids_of(g, split, K)
            self._ev("table_ids", main)
            fwd(first, split, K)
        early_stats = self.prefetch is not None
        if early_stats:
            pf_done = torch.cuda.Event()
            pf_done.record(main)
            self.s_replay.wait_event(pf_done)
            with torch.cuda.stream(self.s_replay):
                self.buffer.stats_chunks(g, 0, K, pf)
                if host_src is not None:
                    for r in range(2):
                        self.cov_host[r, :K].copy_(self.buffer._cov[r, :K], non_blocking=True)
                    e = torch.cuda.Event(external=True)   # an event node in a graph
                    e.record(self.s_replay)
                    self._cov_events.append((0, K, e))
        fwd(second, 0, K)
        scored = torch.cuda.Event()
        scored.record(main)
        self.s_replay.wait_event(scored)
        with torch.cuda.stream(self.s_replay):
            self._ev("replay", self.s_replay)
            if self._lru_fused and not self.buffer.run_chunks_lru(
                    g, 0, K, True, self.lru, bits, pf, skip_stats=early_stats):
                self.buffer.run_chunks(g, 0, K, True, bits, pf, skip_stats=early_stats)
                self.lru.reset()
                self.lru.run(g)
            elif not self._lru_fused:
                self.buffer.run_chunks(g, 0, K, True, bits, pf, skip_stats=early_stats)
            self._ev("replay", self.s_replay)
            if host_src is not None and not early_stats:
                for r in range(2):
                    self.cov_host[r, :K].copy_(self.buffer._cov[r, :K], non_blocking=True)
                e = torch.cuda.Event(external=True)   # an event node in a graph
                e.record(self.s_replay)
                self._cov_events.append((0, K, e))

    def _launch_streamed(self, g, K, pieces, host_src, all_ids, main, bits, pf, split):
        """The streamed pipeline (see _STREAMED): the first model's forward
        over all chunks (two launches on the end-to-end path, so it starts
        after the first piece's ids), then the second model's with progress
        signals; the replay stream runs piece i once its tiles are done."""
        torch = self.torch
        L = _native.lib()
        gk = (self.lgid if self.shard is not None else self.gids)[
            :K * self.l_in].view(K, self.l_in)
        tk = self.tid[:K * self.l_in].view(K, self.l_in)
        step = pieces[0][1] - pieces[0][0]
        progress = torch.zeros(len(pieces), dtype=torch.int32, device="cuda")   # on main
        zeroed = torch.cuda.Event()
        zeroed.record(main)
        self.s_replay.wait_event(zeroed)   # the waits below must see this launch's zeros

        def fwd(model, key, k0, k1, signal):
            self._ev(key, main)
            kw = {"progress": progress, "piece_chunks": step} if signal else {}
            if model is self.caching:
                model.forward(gk[k0:k1], tk[k0:k1], logits=self.clog[k0:k1],
                              bits=self.bits[k0:k1], **kw)
            else:
                model.forward(gk[k0:k1], tk[k0:k1], logits=self.plog[k0:k1],
                              pf_gid=self.pf[k0:k1], **kw)
            self._ev(key, main)

        order = [(self.prefetch, "prefetch_fwd"), (self.caching, "caching_fwd")]
        if not _PF_FIRST:
            order.reverse()
        order = [(m, k) for m, k in order if m is not None]
        (m0, k0name), (m1, k1name) = (order[0], order[-1]) if len(order) > 1 else (
            (None, None), order[0])
        if m0 is not None:
            if host_src is not None and split < K:
                fwd(m0, k0name, 0, split, False)
                main.wait_event(all_ids)
                self._ev("table_ids", main)
                self._ids_of(g, split, K)
                self._ev("table_ids", main)
                fwd(m0, k0name, split, K, False)
            else:
                fwd(m0, k0name, 0, K, False)
        if host_src is not None and m0 is None and split < K:
            main.wait_event(all_ids)
            self._ids_of(g, split, K)
        fwd(m1, k1name, 0, K, True)
        for i, (a, b) in enumerate(pieces):
            with torch.cuda.stream(self.s_replay):
                _native.check(L.recmg_wait_progress(
                    _native.ptr(progress), i, (b - a + 127) // 128,
                    _native.stream_handle(torch)), "wait_progress")
                self._ev("replay", self.s_replay)
                self.buffer.run_chunks(g, a, b, i == len(pieces) - 1, bits, pf)
                self._ev("replay", self.s_replay)
                if host_src is not None and b > a:
                    for r in range(2):
                        self.cov_host[r, a:b].copy_(self.buffer._cov[r, a:b], non_blocking=True)
                    e = torch.cuda.Event(external=True)   # an event node in a graph
                    e.record(self.s_replay)
                    self._cov_events.append((a, b, e))
        self._progress = progress   # keep the counters alive until the stream is done

    def report(self):
        """Synchronise and return (BreakdownReport, lru (hits, misses) or None).
        After launch(host_src=...) the float64 coverage is accumulated piece by
        piece, in chunk order (runtime.py:276, 282), as the counts arrive."""
        from .runtime import BreakdownReport
        cov = None
        if getattr(self, "_cov_events", None):
            L = _native.lib()
            acc = 0.0
            base = self.cov_host.data_ptr()
            stride = self.cov_host.stride(0) * 2
            for k0, k1, e in self._cov_events:
                e.synchronize()
                acc = L.recmg_coverage_accumulate(base + 2 * k0, base + stride + 2 * k0, k1 - k0, acc)
            cov = acc / self.K if self.K else 0.0
        r = self.buffer.result(with_coverage=cov is None)
        if cov is not None:
            r["coverage"] = cov
        rep = BreakdownReport(r["cache_hits"], r["prefetch_hits"], r["on_demand"],
                              r["prefetch_issued"], r["prefetch_useful"], r["coverage"],
                              r["evictions"], r["prefetch_inserts"])
        lru = self.lru.result() if self.lru is not None else None
        return rep, lru

    def replay_host(self, host_gids):
        """End to end: pinned/host int32 gids -> BreakdownReport (+ LRU).

        With a pinned source the step's launches (H2D copies, forwards, stats,
        replay, LRU, coverage copies-back, on their four streams) are captured
        once into a CUDA graph per (n, source buffer) and replayed as one graph
        launch, so a synchronous caller does not pay the host launch sequence
        every step; report() then waits on the graph's coverage event nodes.
        RECMG_GRAPHS=0 (or a capture failure) runs the launches eagerly."""
        n = int(host_gids.numel()) if hasattr(host_gids, "numel") else len(host_gids)
        if n > self.n_max:
            raise ValueError("trace longer than the HotPath was sized for")
        src = host_gids if hasattr(host_gids, "numel") else self.torch.from_numpy(
            np.ascontiguousarray(host_gids, dtype=np.int32))
        if _GRAPHS and self.events is None and src.is_pinned():
            key = (n, src.data_ptr())
            if getattr(self, "_graph_key", None) != key:
                self._graph, self._graph_key = None, key
                self.launch(n, host_src=src)     # eager once: workspaces settle
                self.report()
                torch = self.torch
                g = torch.cuda.CUDAGraph()
                try:
                    with torch.cuda.graph(g):
                        self.launch(n, host_src=src)
                    self._graph = g
                    self._graph_state = (list(self._cov_events), self.K, self.n)
                except Exception as e:   # not capturable here: stay eager
                    import warnings
                    warnings.warn(f"HotPath: CUDA graph capture failed, running eagerly ({e})")
                    self._graph = None
                    torch.cuda.synchronize()
            if self._graph is not None:
                self._cov_events, self.K, self.n = (list(self._graph_state[0]),
                                                    self._graph_state[1], self._graph_state[2])
                self._graph.replay()
                return self.report()
        self.launch(n, host_src=src)
        return self.report()

    def d2h_bytes(self):
        """Bytes read back per replay_host: counters, LRU pair, coverage num/den."""
        return 8 * 8 + (16 if self.lru is not None else 0) + 2 * 2 * self.K
