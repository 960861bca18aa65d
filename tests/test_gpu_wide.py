"""Buffers wider than 4096 ways (replay_wide_kernel: global-memory ways, an
id -> slot map, the victim scan by a whole CTA), the GPU labeler, and the
chunk-length handling of the model-driven replay; against reference-made
fixtures (tests/golden/wide.npz, make_golden.py:make_wide) and the oracle."""
import hashlib

import numpy as np
import pytest

import oracle
import paper_2511_08568_b200 as rb
from conftest import golden
from oracle import model_oracle as mo

pytestmark = pytest.mark.gpu

NAMES = ("cache_hits", "prefetch_hits", "on_demand", "prefetch_issued", "prefetch_useful",
         "evictions", "prefetch_inserts")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def _counts(rep):
    return [rep.cache_hits, rep.prefetch_hits, rep.on_demand, rep.prefetch_issued,
            rep.prefetch_useful, rep.evictions, rep.prefetch_inserts]


@pytest.fixture(scope="module")
def wide():
    return golden("wide.npz")


@pytest.fixture(scope="module")
def config1():
    z = golden("config1.npz")
    t = rb.generate_trace(rb.TraceGenConfig([2000] * 8, 1_000_000, 1.05, 0.4, 32, 0))
    K = int(z["bits_shape"][0])
    bits = np.unpackbits(z["bits_packed"])[:K * 15].reshape(K, 15)
    return t, bits, z["pf"]


def test_wide_fully_associative_replay_vs_reference(wide, config1):
    """The reference's own buffer (ways=None) at 30% / 40% of the unique ids
    (4,741 / 6,321 ways): every counter and the coverage equal the
    reference replay with its own config-1 decisions."""
    t, bits, pf = config1
    cfn = lambda s: bits[s.origin // 15]
    pfn = lambda s: pf[s.origin // 15]
    for case, cnt, cov in zip(wide["fa_cases"], wide["fa_counts"], wide["fa_coverage"]):
        C, es = (int(x) for x in case)
        assert C > 4096
        rep = rb.replay(t, rb.BufferConfig(C, es), caching_fn=cfn, prefetch_fn=pfn)
        assert _counts(rep) == list(cnt[:7]), case
        assert rep.coverage == float(cov), case


def test_wide_set_associative_vs_reference_composition(wide, config1):
    t, bits, pf = config1
    cap, ways, es = (int(x) for x in wide["sa_case"])
    rep = rb.replay(t, rb.BufferConfig(cap, es, ways), caching_fn=lambda s: bits[s.origin // 15],
                    prefetch_fn=lambda s: pf[s.origin // 15])
    got = [rep.cache_hits, rep.prefetch_hits, rep.on_demand, rep.evictions, rep.prefetch_inserts]
    assert got == list(wide["sa_counts"][:5])


@pytest.mark.parametrize("seed", range(3))
def test_wide_random_replays_vs_oracle(seed):
    """Random Zipf traces, ragged prefetch lists, capacities past 4096 ways:
    counters, coverage and the per-access class against the C oracle."""
    rng = np.random.default_rng(300 + seed)
    V = int(rng.integers(9000, 30000))
    n = int(rng.integers(60000, 150000))
    gids = (rng.zipf(1.05, n) - 1) % V
    K = rb.num_chunks(n)
    bits = rng.integers(0, 2, (K, 15)).astype(np.uint8)
    pf = rng.integers(0, V, (K, 5))
    pf[np.arange(5)[None, :] >= rng.integers(0, 6, K)[:, None]] = -1
    t = rb.trace_from_gids(gids, [V])
    for ways, cap in ((None, int(rng.integers(4097, 7000))), (4160, 4160 * 2)):
        es = int(rng.choice([1, 4, cap]))
        rep, cls = rb.replay(t, rb.BufferConfig(cap, es, ways),
                             caching_fn=lambda s: bits[s.origin // 15],
                             prefetch_fn=lambda s: [int(g) for g in pf[s.origin // 15] if g >= 0],
                             return_access_class=True)
        ref, cov, rcls = oracle.replay(gids, V, cap, ways or 0, es, bits=bits, pf=pf,
                                       access_class=True)
        assert _counts(rep) == [ref[k] for k in NAMES], (ways, cap, es)
        assert rep.coverage == cov
        assert np.array_equal(cls, rcls), (ways, cap, es)
        # fully associative / wide-set LRU against the oracle, per access
        res = rb.simulate(gids, rb.CacheConfig(cap, rb.Policy.LRU, ways))
        h, pa = oracle.lru(gids, V, cap, ways or 0, per_access=True)
        assert res.hits == h and res.per_access_hit == pa.tolist(), (ways, cap)


def test_wide_policies_vs_reference(wide, config1):
    """simulate() fully associative past 4096 ways: LRU / LFU / OPTGEN on
    config 1 (per-access hits and optgen keep bits by sha256), SRRIP / LFU /
    LRU / OPTGEN on a smaller trace (per-access vectors), and the LRU +
    prefetch baseline (replay_policy_only) with the optgen-miss prefetcher."""
    t, _, _ = config1
    C = int(np.floor(0.4 * t.unique_count))
    for name, pol in (("lru", rb.Policy.LRU), ("lfu", rb.Policy.LFU),
                      ("optgen", rb.Policy.OPTGEN)):
        res = rb.simulate(t, rb.CacheConfig(C, pol))
        assert res.hits == int(wide[f"{name}_hits"]), name
        assert sha(np.array(res.per_access_hit)) == str(wide[f"{name}_pa_sha"]), name
        if pol == rb.Policy.OPTGEN:
            assert sha(np.array(res.keep_decisions)) == str(wide["optgen_keep_sha"])
    ts = rb.trace_from_gids(wide["small_gids"], [int(x) for x in wide["small_table_sizes"]])
    n = len(ts)
    for name, pol in (("srrip", rb.Policy.SRRIP), ("lfu", rb.Policy.LFU), ("lru", rb.Policy.LRU),
                      ("optgen", rb.Policy.OPTGEN)):
        res = rb.simulate(ts, rb.CacheConfig(4160, pol))
        want = np.unpackbits(wide[f"small_{name}_per_access"])[:n]
        assert res.hits == int(wide[f"small_{name}_hits"]), name
        assert np.array_equal(np.array(res.per_access_hit, dtype=np.uint8), want), name
    pf = wide["small_lrupf_pf"]
    rep = rb.replay_policy_only(ts, rb.CacheConfig(4200, rb.Policy.LRU),
                                prefetch_fn=lambda s: [int(g) for g in pf[s.origin // 15] if g >= 0])
    assert [rep.cache_hits, rep.prefetch_hits, rep.on_demand, rep.prefetch_issued,
            rep.prefetch_useful] == list(wide["small_lrupf_counts"])
    assert rep.coverage == float(wide["small_lrupf_coverage"])


def test_labels_vs_reference(wide, config1):
    """label_caching / label_prefetch (labeler.py:43-83) on config 1 at 80%
    of the 20% buffer (2,528 ways: shared-memory kernel) and of the 40%
    buffer (5,056 ways: global-memory kernel), list API and array API."""
    t, _, _ = config1
    U = t.unique_count
    samples = rb.chunk(t)
    for name, gc in (("c20", int(np.floor(0.2 * U))), ("c40", int(np.floor(0.4 * U)))):
        assert [gc, int(np.floor(0.8 * gc))] == [int(x) for x in wide[f"label_{name}_cap"]]
        lc = rb.label_caching(t, samples, gc)
        lab = np.array([s.cache_labels for s in lc.samples], dtype=np.uint8)
        assert sha(lab) == str(wide[f"label_{name}_caching_sha"]), name
        arr, cap = rb.caching_label_array(t, gc)
        assert np.array_equal(arr, lab) and cap == lc.label_capacity
        lp = rb.label_prefetch(t, samples, gc, l_out=5)
        tg = np.array([[a.global_id for a in s.prefetch_targets] for s in lp.samples])
        assert sha(tg) == str(wide[f"label_{name}_prefetch_sha"]), name
        assert lp.dropped == int(wide[f"label_{name}_prefetch_dropped"])
        org, tga, dropped, _ = rb.prefetch_target_array(t, gc)
        assert sha(org) == str(wide[f"label_{name}_prefetch_origin_sha"])
        assert np.array_equal(tga, tg) and dropped == lp.dropped


def test_replay_with_model_at_another_chunk_length():
    """replay(l_in=10) with models packed for l_in=15: the
    models run over 10-access chunks (the reference's forwards take any
    length), the prefetch model still emits its own l_out ids; counters
    equal the oracle replay of the float64 decisions at that length."""
    t = rb.generate_trace(rb.TraceGenConfig([250] * 8, 12000, 1.05, 0.4, 32, 4))
    V = t.total_ids
    for dim in (64, 16):
        cp = rb.init_params("caching", t.table_sizes, dim=dim, seed=0, init_scale=0.4)
        pp = rb.init_params("prefetch", t.table_sizes, dim=dim, seed=1, l_out=3, init_scale=0.4)
        L, lo, wr = 10, 4, 2
        rep = rb.replay(t, rb.BufferConfig(400, 4, 16), cp, pp, l_in=L, l_out=lo,
                        window_ratio=wr)
        K = rb.num_chunks(len(t), L, lo, wr)
        gid = t.gid_array[:K * L].reshape(K, L)
        tid = t.table_ids[:K * L].reshape(K, L)
        lc = rb.forward_caching_batch(cp, gid, tid).logits
        rc = mo.caching_logits(cp.arrays, dim, 1, gid, tid)
        assert np.max(np.abs(lc - rc) / np.maximum(np.abs(rc), 1e-2)) <= 1e-3
        bits = (lc >= 0).astype(np.uint8)
        lp = rb.forward_prefetch_batch(pp, gid, tid).logits
        assert lp.shape == (K, 3)
        pf = mo.decode_gids(mo.sigmoid(lp.astype(np.float64)), V)
        ref, cov = oracle.replay(t.gid_array, V, 400, 16, 4, l_in=L, l_out=lo, window_ratio=wr,
                                 bits=bits, pf=pf)
        assert _counts(rep) == [ref[k] for k in NAMES], dim
        assert rep.coverage == cov
        # replay_policy_only's l_out is the window only: a 3-id model with the
        # default l_out=5 runs (the reference accepts it, runtime.py:286-339)
        r2 = rb.replay_policy_only(t, rb.CacheConfig(300, rb.Policy.LRU), prefetch_params=pp)
        assert r2.prefetch_issued == 3 * rb.num_chunks(len(t))


def test_wide_coverage_window_past_255():
    """Windows longer than 255 accesses (uint16 coverage counts)."""
    rng = np.random.default_rng(7)
    V, n = 500, 30000
    gids = (rng.zipf(1.1, n) - 1) % V
    t = rb.trace_from_gids(gids, [V])
    K = rb.num_chunks(n, 15, 5, 60)
    pf = rng.integers(0, V, (K, 5))
    rep = rb.replay(t, rb.BufferConfig(64, 4, 32), l_out=5, window_ratio=60,
                    prefetch_fn=lambda s: [int(g) for g in pf[s.origin // 15]])
    ref, cov = oracle.replay(gids, V, 64, 32, 4, window_ratio=60, pf=pf)
    assert _counts(rep) == [ref[k] for k in NAMES]
    assert rep.coverage == cov


def test_device_models_are_reused_until_weights_change():
    """replay / forward_*_batch reuse the packed model across calls; an
    in-place update of the arrays (as the reference trainer does,
    neural/train.py:203) is seen by the next call."""
    from paper_2511_08568_b200 import model as mdl
    t = rb.generate_trace(rb.TraceGenConfig([250] * 4, 3000, 1.05, 0.4, 32, 2))
    cp = rb.init_params("caching", t.table_sizes, dim=64, seed=0, init_scale=0.4)
    K = rb.num_chunks(len(t))
    gid = t.gid_array[:K * 15].reshape(K, 15)
    tid = t.table_ids[:K * 15].reshape(K, 15)
    a = mdl.device_model(cp)
    assert mdl.device_model(cp) is a
    l0 = rb.forward_caching_batch(cp, gid, tid).logits
    cp.arrays["head_b"] += 0.5
    b = mdl.device_model(cp)
    assert b is not a
    l1 = rb.forward_caching_batch(cp, gid, tid).logits
    assert np.allclose(l1 - l0, 0.5, atol=1e-4)


def test_priority_bound_after_every_chunk():
    """test_runtime.py:139-154 on the GPU state: replaying chunk by chunk
    (recmg_replay_chunks continues the state), no resident priority exceeds
    eviction_speed + 1 after any chunk's update, fully associative and
    32-way, and the piecewise replay equals the one-shot replay."""
    import torch
    from paper_2511_08568_b200.engine import BufferReplay, to_device_gids
    t = rb.generate_trace(rb.TraceGenConfig([4, 100, 60], 4000, 1.05, 0.4, 24, 11))
    n = len(t)
    K = rb.num_chunks(n)
    bits = torch.ones((K, 15), dtype=torch.uint8, device="cuda")
    g = to_device_gids(torch, t.gid_array)
    for cap, ways in ((24, None), (64, 32)):
        eng = BufferReplay(cap, t.total_ids, 4, ways, n)
        S = cap // (ways or cap)
        W = ways or cap
        off = 64 + ((4 * S * W + 255) // 256) * 256
        top = 0
        for k in range(K):
            eng.run_chunks(g, k, k + 1, k == K - 1, bits=bits)
            tags = eng.state[64:64 + 4 * S * W].view(torch.int32)
            meta = eng.state[off:off + 8 * S * W].view(torch.int64)
            pr = (meta & 0xFFFFFFFF)[tags >= 0]
            if pr.numel():
                top = max(top, int(pr.max()))
                assert top <= 5, (cap, ways, k)
        r = eng.result()
        one = rb.replay(t, rb.BufferConfig(cap, 4, ways), caching_fn=lambda s: [1] * 15)
        assert r["on_demand"] == one.on_demand and r["cache_hits"] == one.cache_hits
        assert top == 5
