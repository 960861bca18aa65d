"""Trace data model (trace.py of the reference), array-backed.

The reference keeps a Python ``EmbeddingIndex`` object per access
(trace.py:54-77); at 25 M-500 M accesses that is the bottleneck, so here a
``Trace`` is its int64 ``gid_array`` plus ``table_sizes`` and materialises
``accesses`` only on demand.  Any object with ``gid_array`` and
``table_sizes`` (including a reference ``embcache.Trace``) is accepted by
the replay API.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace

import numpy as np

from . import _native
from .errors import InvalidConfigError, TraceParseError, TraceValidationError


@dataclass(frozen=True, slots=True)
class EmbeddingIndex:
    """trace.py:18-24."""
    table_id: int
    row_id: int
    global_id: int


def table_offsets(table_sizes) -> np.ndarray:
    """trace.py:27-29."""
    return np.concatenate(([0], np.cumsum(np.asarray(table_sizes, dtype=np.int64))))


def make_index(table_id: int, row_id: int, table_sizes) -> EmbeddingIndex:
    """trace.py:32-41."""
    if not 0 <= table_id < len(table_sizes):
        raise TraceValidationError(f"table_id {table_id} out of range")
    if not 0 <= row_id < table_sizes[table_id]:
        raise TraceValidationError(
            f"row_id {row_id} out of range for table {table_id} (size {table_sizes[table_id]})")
    return EmbeddingIndex(table_id, row_id, int(sum(table_sizes[:table_id])) + row_id)


def index_of_global(global_id: int, table_sizes) -> EmbeddingIndex:
    """trace.py:44-51."""
    total = int(sum(table_sizes))
    if not 0 <= global_id < total:
        raise TraceValidationError(f"global_id {global_id} out of range [0, {total})")
    offsets = table_offsets(table_sizes)
    t = int(np.searchsorted(offsets, global_id, side="right")) - 1
    return EmbeddingIndex(t, int(global_id - offsets[t]), int(global_id))


class Trace:
    """Ordered accesses over a fixed table layout (trace.py:54-77)."""

    def __init__(self, gid_array, table_sizes):
        self.gid_array = np.ascontiguousarray(gid_array, dtype=np.int64)
        self.table_sizes = [int(s) for s in table_sizes]
        self._unique = None

    @property
    def unique_count(self) -> int:
        if self._unique is None:
            self._unique = int(np.unique(self.gid_array).size)
        return self._unique

    def __len__(self) -> int:
        return len(self.gid_array)

    @property
    def total_ids(self) -> int:
        return int(sum(self.table_sizes))

    @property
    def table_ids(self) -> np.ndarray:
        off = table_offsets(self.table_sizes)
        return np.searchsorted(off, self.gid_array, side="right") - 1

    @property
    def accesses(self) -> list[EmbeddingIndex]:
        off = table_offsets(self.table_sizes)
        t = self.table_ids
        return [EmbeddingIndex(int(a), int(g - off[a]), int(g))
                for a, g in zip(t, self.gid_array)]

    def __eq__(self, other):
        return (list(self.table_sizes) == list(other.table_sizes)
                and np.array_equal(self.gid_array, other.gid_array))


def trace_from_gids(gids, table_sizes) -> Trace:
    """trace.py:80-91."""
    offsets = table_offsets(table_sizes)
    gids = np.asarray(gids, dtype=np.int64)
    if gids.size and (gids.min() < 0 or gids.max() >= offsets[-1]):
        raise TraceValidationError("global id out of range for table layout")
    return Trace(gids, table_sizes)


@dataclass
class TraceGenConfig:
    """trace.py:94-121."""
    table_sizes: list
    total_accesses: int
    zipf_exponent: float = 1.1
    markov_stickiness: float = 0.0
    correlation_pool_size: int = 32
    rng_seed: int = 0

    def validate(self):
        if not self.table_sizes or any(s <= 0 for s in self.table_sizes):
            raise InvalidConfigError("table_sizes must be non-empty and positive")
        if self.total_accesses <= 0:
            raise InvalidConfigError("total_accesses must be positive")
        if self.zipf_exponent < 0:
            raise InvalidConfigError("zipf_exponent must be >= 0")
        if not 0.0 <= self.markov_stickiness <= 1.0:
            raise InvalidConfigError("markov_stickiness must be in [0, 1]")
        if self.correlation_pool_size < 1:
            raise InvalidConfigError("correlation_pool_size must be >= 1")


def generate_trace(cfg: TraceGenConfig) -> Trace:
    """Bit-identical to the reference generate_trace (trace.py:124-161).

    The draws use the same numpy Generator calls in the same order
    (permutation, then ``choice(p=...)`` — restated as numpy's own
    ``cdf.searchsorted(random(n), 'right')`` — then the two coin arrays);
    the sequential sticky-pool pass (:144-160) runs in C
    (recmg_trace_pool_pass).
    """
    cfg.validate()
    total = int(sum(cfg.table_sizes))
    n = int(cfg.total_accesses)
    if n >= (1 << 20) and total < np.iinfo(np.int32).max:
        # same draws through the multi-threaded streamed path (TraceStream)
        return Trace(generate_trace_streamed(cfg), cfg.table_sizes)
    rng = np.random.default_rng(cfg.rng_seed)
    ranks = np.arange(1, total + 1, dtype=np.float64)
    weights = ranks ** (-cfg.zipf_exponent)
    probs = weights / weights.sum()
    rank_to_gid = rng.permutation(total)
    # Generator.choice(total, size=n, p=probs) for 1-D p: cdf = cumsum(p),
    # cdf /= cdf[-1], uniform = random(n), idx = cdf.searchsorted(u, 'right')
    cdf = probs.cumsum()
    cdf /= cdf[-1]
    zipf_ranks = cdf.searchsorted(rng.random(n), side="right")
    sticky_coin = rng.random(n)
    pool_coin = rng.random(n)
    zipf_gids = rank_to_gid[zipf_ranks].astype(np.int64)
    gids = _native.pool_pass(zipf_gids, sticky_coin, pool_coin, cfg.markov_stickiness,
                             cfg.correlation_pool_size)
    return Trace(gids, cfg.table_sizes)


class TraceStream:
    """generate_trace (trace.py:124-161) streamed block by block, bit-exact.

    For traces the reference cannot materialise (config 3: 5e8 accesses over
    8.56e7 ids).  The permutation is numpy's own (the same call on the same
    default_rng); the PCG64 state right after it seeds the three random()
    streams, which recmg_trace_generate_block reaches at outputs i0, n+i0
    and 2n+i0 by jump-ahead.  Blocks must be drawn in order (the sticky pool
    carries over); every block is int32 gids.
    """

    GUIDE_LOG2 = 24

    def __init__(self, cfg: TraceGenConfig, threads: int | None = None):
        import os
        cfg.validate()
        self.cfg = cfg
        self.n = int(cfg.total_accesses)
        self.V = int(sum(cfg.table_sizes))
        if self.V > np.iinfo(np.int32).max:
            raise InvalidConfigError("streamed traces need fewer than 2^31 ids")
        rng = np.random.default_rng(cfg.rng_seed)
        ranks = np.arange(1, self.V + 1, dtype=np.float64)
        weights = ranks ** (-cfg.zipf_exponent)
        del ranks
        probs = weights / weights.sum()
        del weights
        self.rank_to_gid = rng.permutation(self.V)
        cdf = probs.cumsum()
        del probs
        cdf /= cdf[-1]
        self.cdf = cdf
        st = rng.bit_generator.state["state"]
        m64 = (1 << 64) - 1
        self.pcg = np.array([st["state"] >> 64, st["state"] & m64, st["inc"] >> 64,
                             st["inc"] & m64], dtype=np.uint64)
        self.guide_log2 = self.GUIDE_LOG2 if self.V > 4096 else 12
        self.guide = np.empty((1 << self.guide_log2) + 1, dtype=np.int64)
        _native.check(_native.lib().recmg_trace_guide(self.cdf.ctypes.data, self.V,
                                                      self.guide_log2, self.guide.ctypes.data),
                      "trace_guide")
        self.pool = np.zeros(cfg.correlation_pool_size, dtype=np.int64)
        self.pool_len = np.zeros(1, dtype=np.int32)
        self.pos = 0
        self.threads = threads or max(1, min(16, len(os.sched_getaffinity(0))))

    def next_block(self, count: int) -> np.ndarray:
        count = min(int(count), self.n - self.pos)
        out = np.empty(count, dtype=np.int32)
        if count:
            _native.check(_native.lib().recmg_trace_generate_block(
                self.pcg.ctypes.data, self.n, self.pos, count, self.cdf.ctypes.data, self.V,
                self.guide.ctypes.data, self.guide_log2, self.rank_to_gid.ctypes.data,
                float(self.cfg.markov_stickiness), int(self.cfg.correlation_pool_size),
                self.pool.ctypes.data, self.pool_len.ctypes.data, out.ctypes.data,
                self.threads), "trace_generate_block")
        self.pos += count
        return out

    def blocks(self, block: int = 1 << 24):
        while self.pos < self.n:
            yield self.next_block(block)

    def uniforms(self, skip: int, count: int) -> np.ndarray:
        """Generator.random() outputs [skip, skip+count) after the permutation."""
        out = np.empty(int(count), dtype=np.float64)
        _native.check(_native.lib().recmg_pcg64_uniforms(self.pcg.ctypes.data, int(skip),
                                                         int(count), out.ctypes.data,
                                                         self.threads), "pcg64_uniforms")
        return out


def generate_trace_streamed(cfg: TraceGenConfig, block: int = 1 << 24) -> np.ndarray:
    """All gids of generate_trace(cfg) as int32, drawn block by block."""
    s = TraceStream(cfg)
    out = np.empty(s.n, dtype=np.int32)
    for b in s.blocks(block):
        out[s.pos - len(b):s.pos] = b
    return out


@dataclass
class SequenceSample:
    """trace.py:207-223."""
    input: list
    origin: int
    cache_labels: list | None = None
    prefetch_targets: list | None = None
    window: list | None = None

    def with_labels(self, **kw) -> "SequenceSample":
        return replace(self, **kw)


def num_chunks(n: int, l_in: int = 15, l_out: int = 5, window_ratio: int = 3) -> int:
    """len(chunk(trace, ...)) without building samples (trace.py:238-250)."""
    l_win = window_ratio * l_out
    if n < l_in + l_win:
        return 0
    return (n - l_in - l_win) // l_in + 1


def chunk(trace, l_in: int = 15, l_out: int = 5, window_ratio: int = 3) -> list:
    """trace.py:226-250 (materialises Python samples: for callables only)."""
    if l_in < 1 or l_out < 1:
        raise InvalidConfigError("l_in and l_out must be >= 1")
    if window_ratio < 1:
        raise InvalidConfigError("window_ratio must be >= 1")
    l_win = window_ratio * l_out
    acc = trace.accesses
    out = []
    for k in range(num_chunks(len(acc), l_in, l_out, window_ratio)):
        o = k * l_in
        out.append(SequenceSample(input=acc[o:o + l_in], origin=o,
                                  window=acc[o + l_in:o + l_in + l_win]))
    return out


# ---- trace files (trace.py:164-204) and a binary form for 1e8+ accesses ----
_LINE_BREAKS = bytes([0x0B, 0x0C, 0x0D, 0x1C, 0x1D, 0x1E, 0x85, 0xA8, 0xA9])


def write_trace(trace, path: str):
    """trace.py:164-169: header 'tables: n1,n2,...' then 'table_id,row_id' lines."""
    sizes = [int(s) for s in trace.table_sizes]
    g = np.asarray(trace.gid_array, dtype=np.int64)
    off = table_offsets(sizes)
    t = np.searchsorted(off, g, side="right") - 1
    with open(path, "w", encoding="utf-8") as f:
        f.write("tables: " + ",".join(str(s) for s in sizes) + "\n")
        blk = 1 << 20
        for i in range(0, len(g), blk):
            tt, rr = t[i:i + blk], g[i:i + blk] - off[t[i:i + blk]]
            f.write("".join(f"{a},{b}\n" for a, b in zip(tt.tolist(), rr.tolist())))


def _parse_line(raw, lineno, table_sizes, offsets):
    """The reference's per-line rules (trace.py:186-203); None for blank lines."""
    if not raw.strip():
        return None
    parts = raw.split(",")
    if len(parts) != 2:
        raise TraceParseError(f"expected 'table_id,row_id', got {raw!r}", line=lineno)
    try:
        table_id, row_id = int(parts[0]), int(parts[1])
    except ValueError:
        raise TraceParseError(f"non-integer field in {raw!r}", line=lineno)
    if not 0 <= table_id < len(table_sizes):
        raise TraceValidationError(f"table_id {table_id} out of range", line=lineno)
    if not 0 <= row_id < table_sizes[table_id]:
        raise TraceValidationError(
            f"row_id {row_id} out of range for table {table_id}", line=lineno)
    return int(offsets[table_id]) + row_id


def _parse_header(first):
    if not first.startswith("tables: "):
        raise TraceParseError("expected header 'tables: n1,n2,...'", line=1)
    try:
        sizes = [int(tok) for tok in first[len("tables: "):].split(",")]
    except ValueError as e:
        raise TraceParseError(f"bad table size list: {e}", line=1)
    if not sizes or any(s <= 0 for s in sizes):
        raise TraceValidationError("table sizes must be positive", line=1)
    return sizes


def read_trace(path: str) -> Trace:
    """trace.py:172-204, same errors and line numbers.  The body is parsed in
    C (recmg_trace_parse_text) wherever lines have the plain 'int,int' form;
    any other line is read with the reference's rules, which raise or accept
    it exactly as the reference does."""
    with open(path, "rb") as f:
        data = f.read()
    if any(b in data for b in _LINE_BREAKS):
        # str.splitlines() separators beyond '\n' (or non-ASCII text): the
        # reference's own line splitting, line by line
        lines = data.decode("utf-8").splitlines()
        if not lines:
            raise TraceParseError("expected header 'tables: n1,n2,...'", line=1)
        sizes = _parse_header(lines[0])
        off = table_offsets(sizes)
        out = [g for i, raw in enumerate(lines[1:], start=2)
               if (g := _parse_line(raw, i, sizes, off)) is not None]
        return Trace(np.asarray(out, dtype=np.int64), sizes)
    if not data.isascii():
        data.decode("utf-8")    # the reference reads text: invalid UTF-8 raises here too
    nl = data.find(b"\n")
    first = (data if nl < 0 else data[:nl]).decode("utf-8")
    if not data:
        raise TraceParseError("expected header 'tables: n1,n2,...'", line=1)
    sizes = _parse_header(first)
    off = np.ascontiguousarray(table_offsets(sizes), dtype=np.int64)
    cap = data.count(b"\n") + 1
    out = np.empty(cap, dtype=np.int32)
    buf = np.frombuffer(data, dtype=np.uint8)
    pos, lineno, L = (len(data) if nl < 0 else nl + 1), 2, _native.lib()
    n, stop, done = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
    while pos < len(data):
        _native.check(L.recmg_trace_parse_text(buf.ctypes.data, len(data), pos, off.ctypes.data,
                                               len(sizes), out.ctypes.data, cap,
                                               ctypes.byref(n), ctypes.byref(stop),
                                               ctypes.byref(done)),
                      "trace_parse_text")
        lineno += done.value
        pos = stop.value
        if pos >= len(data):
            break
        e = data.find(b"\n", pos)
        e = len(data) if e < 0 else e
        g = _parse_line(data[pos:e].decode("utf-8"), lineno, sizes, off)
        if g is not None:
            out[n.value] = g
            n.value += 1
        lineno += 1
        pos = e + 1
    return Trace(out[:n.value].astype(np.int64), sizes)


_BIN_MAGIC = b"RECMGTR1"


def write_trace_binary(trace, path: str):
    """Binary trace: magic, n_tables (int64), table sizes (int64), n (int64),
    gids (int32, little endian) -- 4 bytes per access instead of ~10 of text."""
    sizes = np.asarray([int(s) for s in trace.table_sizes], dtype="<i8")
    g = np.asarray(trace.gid_array)
    with open(path, "wb") as f:
        f.write(_BIN_MAGIC)
        f.write(np.asarray([len(sizes)], dtype="<i8").tobytes())
        f.write(sizes.tobytes())
        f.write(np.asarray([len(g)], dtype="<i8").tobytes())
        blk = 1 << 24
        for i in range(0, len(g), blk):
            f.write(np.ascontiguousarray(g[i:i + blk], dtype="<i4").tobytes())


def read_trace_binary(path: str, mmap: bool = False):
    """Inverse of write_trace_binary; mmap=True maps the gids (int32) without
    reading them, for traces larger than host memory."""
    with open(path, "rb") as f:
        if f.read(8) != _BIN_MAGIC:
            raise TraceParseError("not a binary trace (bad magic)", line=None)
        nt = int(np.frombuffer(f.read(8), dtype="<i8")[0])
        sizes = np.frombuffer(f.read(8 * nt), dtype="<i8").tolist()
        n = int(np.frombuffer(f.read(8), dtype="<i8")[0])
        start = f.tell()
    if not sizes or any(s <= 0 for s in sizes):
        raise TraceValidationError("table sizes must be positive", line=None)
    if mmap:
        g = np.memmap(path, dtype="<i4", mode="r", offset=start, shape=(n,))
        return g, sizes
    g = np.fromfile(path, dtype="<i4", count=n, offset=start)
    if len(g) != n:
        raise TraceParseError("binary trace truncated", line=None)
    if n and (g.min() < 0 or g.max() >= sum(sizes)):
        raise TraceValidationError("global id out of range for table layout")
    return Trace(g.astype(np.int64), sizes)
