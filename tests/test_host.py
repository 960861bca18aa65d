"""Host-side logic and the C ABI library, no GPU needed."""
import ctypes
import hashlib
import json
import os
import re

import numpy as np
import pytest

import paper_2511_08568_b200 as rb
from paper_2511_08568_b200 import _native
from conftest import ROOT, golden


def header_functions():
    text = open(os.path.join(ROOT, "include", "recmg.h")).read()
    return sorted(set(re.findall(r"\b(recmg_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = _native.lib()
    names = header_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(_native.EXPORTS)


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_native.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_status_strings_and_categories():
    L = _native.lib()
    assert L.recmg_status_category(-1) == b"invalid-config"
    assert L.recmg_status_category(-2) == b"vocabulary-mismatch"
    assert L.recmg_status_category(-3) == b"out-of-vocabulary"
    assert L.recmg_status_string(0) == b"ok"
    with pytest.raises(rb.InvalidConfigError):
        _native.check(-1)
    with pytest.raises(rb.VocabularyMismatchError):
        _native.check(-2)
    with pytest.raises(ValueError):
        _native.check(-4)


def test_num_chunks_matches_reference_rule():
    L = _native.lib()
    for n in (0, 14, 29, 30, 44, 45, 46, 1000, 10 ** 6):
        for l_in, l_out, wr in ((15, 5, 3), (10, 5, 2), (7, 3, 1)):
            l_win = l_out * wr
            want, o = 0, 0
            while o + l_in + l_win <= n:
                want += 1
                o += l_in
            assert L.recmg_num_chunks(n, l_in, l_out, wr) == want
            assert rb.num_chunks(n, l_in, l_out, wr) == want


def test_sizes_and_workspaces():
    L = _native.lib()
    cfg = _native.buffer_cfg(3136, 32, 4, _native.POLICY_PRIORITY, 16000)
    assert L.recmg_buffer_state_bytes(ctypes.byref(cfg)) >= 3136 * 12
    bad = _native.buffer_cfg(100, 32, 4, _native.POLICY_PRIORITY, 16000)  # 32 does not divide
    assert L.recmg_buffer_state_bytes(ctypes.byref(bad)) == 0
    sz = ctypes.c_size_t(0)
    assert L.recmg_replay_workspace_bytes(ctypes.byref(cfg), 10 ** 6, 15, 5, 3, 5,
                                          ctypes.byref(sz)) == 0
    assert sz.value >= 4 * (66665 * 35)
    assert L.recmg_replay_workspace_bytes(ctypes.byref(cfg), 10, 0, 5, 3, 5,
                                          ctypes.byref(sz)) == -1
    lru = _native.buffer_cfg(3136, 32, 1, _native.POLICY_LRU, 16000)
    assert L.recmg_simulate_workspace_bytes(ctypes.byref(lru), 1000, ctypes.byref(sz)) == 0


def test_model_dense_floats_matches_shapes():
    L = _native.lib()
    for kind, dim, stacks in (("caching", 64, 1), ("prefetch", 64, 2), ("caching", 5, 1)):
        p = rb.init_params(kind, [4, 100, 60], dim=dim)
        shape = _native.ModelShape(0 if kind == "caching" else 1, dim, stacks, 15, 5, 3, 164)
        want = sum(a.size for n, a in p.arrays.items() if n != "embed_id")
        assert L.recmg_model_dense_floats(ctypes.byref(shape)) == want
        assert L.recmg_model_packed_bytes(ctypes.byref(shape), 0) >= 4 * want


def test_init_params_matches_reference_fixture():
    m = golden("models.npz")
    sizes = [int(s) for s in m["table_sizes"]]
    for kind, dim, seed, scale in m["cases"]:
        kind = "caching" if kind == 0 else "prefetch"
        p = rb.init_params(kind, sizes, dim=int(dim), seed=int(seed), init_scale=float(scale))
        ws = np.array([float(np.sum(a)) for a in p.arrays.values()])
        assert np.array_equal(ws, m[f"{kind}_{int(dim)}_{int(seed)}_wsum"])


def test_generate_trace_bit_exact():
    z = golden("traces.npz")
    i = 0
    while f"cfg{i}" in z:
        ts, n, s, p, pool, seed = json.loads(str(z[f"cfg{i}"]))
        t = rb.generate_trace(rb.TraceGenConfig(ts, n, s, p, pool, seed))
        assert hashlib.sha256(t.gid_array.astype(np.int64).tobytes()).hexdigest() == str(z[f"sha{i}"])
        assert t.unique_count == int(z[f"unique{i}"])
        if f"gids{i}" in z:
            assert np.array_equal(t.gid_array, z[f"gids{i}"])
        i += 1


def test_streamed_generator_matches_reference_hashes():
    """TraceStream (block-wise, PCG64 jump-ahead, guide-table searchsorted)
    reproduces the reference generate_trace outputs (golden sha256 made by
    running the reference, tests/golden/make_golden.py)."""
    from paper_2511_08568_b200.trace import generate_trace_streamed
    z = golden("traces.npz")
    i = 0
    while f"cfg{i}" in z:
        ts, n, s, p, pool, seed = json.loads(str(z[f"cfg{i}"]))
        for block in (997, 1 << 20):
            g = generate_trace_streamed(rb.TraceGenConfig(ts, n, s, p, pool, seed), block)
            assert hashlib.sha256(g.astype(np.int64).tobytes()).hexdigest() == str(z[f"sha{i}"])
        i += 1
    c1 = golden("config1.npz")
    g = generate_trace_streamed(rb.TraceGenConfig([2000] * 8, 1_000_000, 1.05, 0.4, 32, 0),
                                 300_001)
    assert hashlib.sha256(g.astype(np.int64).tobytes()).hexdigest() == str(c1["sha"])


def test_pcg64_jump_ahead_matches_numpy():
    from paper_2511_08568_b200.trace import TraceStream
    s = TraceStream(rb.TraceGenConfig([100] * 3, 1000, 1.05, 0.4, 32, 5))
    rng = np.random.default_rng(5)
    rng.permutation(300)
    u = rng.random(5000)
    assert np.array_equal(s.uniforms(0, 5000), u)
    assert np.array_equal(s.uniforms(4321, 600), u[4321:4921])


def test_coverage_mean_is_sequential_float64():
    rng = np.random.default_rng(0)
    num = rng.integers(0, 600, 5000).astype(np.uint16)
    den = rng.integers(600, 1600, 5000).astype(np.uint16)
    acc = 0.0
    for a, b in zip(num, den):
        acc += int(a) / int(b)
    assert _native.coverage_mean(num, den) == acc / 5000


def test_chunk_and_trace_model():
    t = rb.trace_from_gids(list(range(45)), [50])
    s = rb.chunk(t)
    assert [x.origin for x in s] == [0, 15]
    assert [a.global_id for a in s[1].window] == list(range(30, 45))
    assert rb.chunk(rb.trace_from_gids(list(range(14)), [20])) == []
    with pytest.raises(rb.TraceValidationError):
        rb.trace_from_gids([0, 5], [5])
    idx = rb.index_of_global(6, [5, 6])
    assert (idx.table_id, idx.row_id) == (1, 1)
    assert [d.global_id for d in rb.decode_indices([0.0, 1.0, 0.5, -3.0, 7.0], [5, 6])] == \
        [0, 10, 5, 0, 10]


def test_replay_validates_before_device_work():
    t = rb.trace_from_gids(list(range(60)), [64])
    with pytest.raises(rb.InvalidConfigError):
        rb.replay(t, rb.BufferConfig(0))
    with pytest.raises(rb.InvalidConfigError):
        rb.replay(t, rb.BufferConfig(4, eviction_speed=0))
    with pytest.raises(rb.InvalidConfigError):
        rb.replay(t, rb.BufferConfig(10, ways=3))
    with pytest.raises(ValueError):
        rb.replay(t, rb.BufferConfig(8), caching_fn=lambda s: [2] * 15)
    with pytest.raises(ValueError):
        rb.replay(t, rb.BufferConfig(8), caching_fn=lambda s: [1] * 14)
    p = rb.init_params("prefetch", [4, 100, 61], dim=4)
    with pytest.raises(rb.VocabularyMismatchError):
        rb.replay(rb.trace_from_gids([0, 1], [4, 100, 60]), rb.BufferConfig(8), prefetch_params=p)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    t = rb.trace_from_gids(list(range(60)), [64])
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rb.replay(t, rb.BufferConfig(8))


@pytest.mark.parametrize("cfg", [
    ([7] * 3, 3000, 1.2, 1.0, 4, 2),            # always sticky once the pool has an id
    ([100_000] * 3, 40_000, 1.05, 0.4, 32, 9),  # V > 4096: the 2^24-bucket guide table
    ([1], 100, 0.5, 0.5, 3, 1),                 # a single id
    ([3, 9000, 1], 25_000, 0.0, 0.7, 64, 4),    # uniform popularity, a wide pool
])
def test_streamed_generator_equals_numpy_path(cfg):
    """The streamed generator (TraceStream) and the numpy restatement of
    generate_trace agree on edge-case configurations, block size 1 included."""
    from paper_2511_08568_b200.trace import generate_trace_streamed
    c = rb.TraceGenConfig(*cfg)
    want = rb.generate_trace(c).gid_array
    for block in (1, 4097, 1 << 20):
        if block == 1 and len(want) > 5000:
            continue
        assert np.array_equal(generate_trace_streamed(c, block), want), block


def test_pad_params_is_exact_in_float64():
    """pad_params (d < 64 models on the d = 64 tcgen05 kernels): the float64
    forwards of the padded model equal the d-unit model's."""
    from oracle import model_oracle as mo
    from paper_2511_08568_b200.model import pad_params
    sizes = [40, 25, 60]
    rng = np.random.default_rng(3)
    gid = rng.integers(0, 125, (33, 15))
    tid = np.searchsorted(np.cumsum([0] + sizes), gid, side="right") - 1
    for d in (8, 32):
        cp = rb.init_params("caching", sizes, dim=d, seed=0, init_scale=0.6)
        pp = rb.init_params("prefetch", sizes, dim=d, seed=1, init_scale=0.6)
        a = mo.caching_logits(cp.arrays, d, 1, gid, tid)
        b = mo.caching_logits(pad_params(cp).arrays, 64, 1, gid, tid)
        assert np.max(np.abs(a - b)) < 1e-12
        a = mo.prefetch_logits(pp.arrays, d, 2, 5, gid, tid)
        b = mo.prefetch_logits(pad_params(pp).arrays, 64, 2, 5, gid, tid)
        assert np.max(np.abs(a - b)) < 1e-12
