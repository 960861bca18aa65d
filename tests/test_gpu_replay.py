"""K3 / K4 on the B200 through the C ABI, bit-exact against the reference's
fixtures and the oracle."""
import numpy as np
import pytest

import oracle
import paper_2511_08568_b200 as rb
from conftest import golden, letters

pytestmark = pytest.mark.gpu

NAMES = ("cache_hits", "prefetch_hits", "on_demand", "prefetch_issued", "prefetch_useful",
         "evictions", "prefetch_inserts")


def _fns(bits, pf):
    cfn = (lambda s: bits[s.origin // 15]) if bits is not None else None
    pfn = (lambda s: [int(g) for g in pf[s.origin // 15] if g >= 0]) if pf is not None else None
    return cfn, pfn


def _counts(rep):
    return [rep.cache_hits, rep.prefetch_hits, rep.on_demand, rep.prefetch_issued,
            rep.prefetch_useful, rep.evictions, rep.prefetch_inserts]


def test_fa_replay_bit_exact_vs_reference(small):
    t = rb.trace_from_gids(small["gids"], [int(x) for x in small["table_sizes"]])
    for case, cnt, cov in zip(small["fa_cases"], small["fa_counts"], small["fa_coverage"]):
        cap, es, ub, up = (int(x) for x in case)
        cfn, pfn = _fns(small["bits"] if ub else None, small["pf"] if up else None)
        rep = rb.replay(t, rb.BufferConfig(cap, es), caching_fn=cfn, prefetch_fn=pfn)
        assert _counts(rep) == list(cnt[:7]), case
        assert rep.coverage == cov, case


def test_set_associative_bit_exact_vs_reference_composition(small):
    t = rb.trace_from_gids(small["gids"], [int(x) for x in small["table_sizes"]])
    cfn, pfn = _fns(small["bits"], small["pf"])
    for case, cnt in zip(small["sa_cases"], small["sa_counts"]):
        cap, ways, es = (int(x) for x in case)
        rep = rb.replay(t, rb.BufferConfig(cap, es, ways), caching_fn=cfn, prefetch_fn=pfn)
        got = [rep.cache_hits, rep.prefetch_hits, rep.on_demand, rep.evictions,
               rep.prefetch_inserts]
        assert got == list(cnt[:5]), case


def test_variable_length_prefetch_lists(small):
    t = rb.trace_from_gids(small["gids"], [int(x) for x in small["table_sizes"]])
    cfn, pfn = _fns(small["opt_bits"], small["opt_pf"])
    rep = rb.replay(t, rb.BufferConfig(int(small["opt_cap"])), caching_fn=cfn, prefetch_fn=pfn)
    assert _counts(rep) == list(small["opt_counts"][:7])
    assert rep.coverage == float(small["opt_coverage"])


@pytest.mark.parametrize("seed", range(6))
def test_random_replays_vs_oracle(seed):
    rng = np.random.default_rng(seed)
    V = int(rng.integers(40, 3000))
    n = int(rng.integers(200, 20000))
    gids = (rng.zipf(1.2, n) - 1) % V
    K = rb.num_chunks(n)
    bits = rng.integers(0, 2, (K, 15)).astype(np.uint8)
    pf = rng.integers(0, V, (K, 5))
    lens = rng.integers(0, 6, K)             # ragged prefetch lists (-1 padded)
    pf[np.arange(5)[None, :] >= lens[:, None]] = -1
    t = rb.trace_from_gids(gids, [V])
    for ways, cap in ((None, int(rng.integers(1, 200))), (32, 32 * int(rng.integers(1, 9))),
                      (8, 8 * int(rng.integers(1, 20))), (1, int(rng.integers(1, 50))),
                      (64, 64 * int(rng.integers(1, 4)))):
        es = int(rng.choice([1, 4, cap]))
        rep, cls = rb.replay(t, rb.BufferConfig(cap, es, ways), caching_fn=lambda s: bits[s.origin // 15],
                             prefetch_fn=lambda s: [int(g) for g in pf[s.origin // 15] if g >= 0],
                             return_access_class=True)
        ref, cov, rcls = oracle.replay(gids, V, cap, ways or 0, es, bits=bits, pf=pf,
                                       access_class=True)
        assert _counts(rep) == [ref[k] for k in NAMES], (ways, cap, es)
        assert rep.coverage == cov
        assert np.array_equal(cls, rcls), (ways, cap, es)


def test_empty_and_tiny_traces():
    t = rb.trace_from_gids(list(range(37)), [64])
    rep = rb.replay(t, rb.BufferConfig(capacity=8))
    assert rep.total == 37 and rep.on_demand == 37           # test_runtime.py:123-128
    t = rb.trace_from_gids([3] * 10, [8])
    rep = rb.replay(t, rb.BufferConfig(capacity=1))
    assert (rep.on_demand, rep.cache_hits) == (1, 9)
    assert rb.replay(rb.trace_from_gids([], [8]), rb.BufferConfig(4)).total == 0


def test_lru_vs_reference(small):
    t = rb.trace_from_gids(small["gids"], [int(x) for x in small["table_sizes"]])
    for case, hits, pa in zip(small["lru_cases"], small["lru_hits"], small["lru_per_access"]):
        cap, ways = int(case[0]), int(case[1]) or None
        res = rb.simulate(t, rb.CacheConfig(cap, rb.Policy.LRU, ways))
        assert res.hits == hits and res.per_access_hit == pa.tolist(), case


def test_lru_known_answers():
    # test_cache_sim.py:13-16 and 108-112
    t = rb.trace_from_gids(letters("ABCABC"), [3])
    assert rb.simulate(t, rb.CacheConfig(2)).hits == 0
    assert rb.simulate(t, rb.CacheConfig(3)).hits == 3
    t = rb.trace_from_gids([0, 2, 0, 1, 1], [4])
    assert rb.simulate(t, rb.CacheConfig(2, rb.Policy.LRU, 1)).per_access_hit == [0, 0, 0, 0, 1]


@pytest.mark.parametrize("seed", range(4))
def test_lru_random_vs_oracle(seed):
    rng = np.random.default_rng(100 + seed)
    V = int(rng.integers(50, 50000))
    n = int(rng.integers(1000, 200000))
    gids = (rng.zipf(1.1, n) - 1) % V
    for ways, cap in ((32, 32 * int(rng.integers(1, 64))), (None, int(rng.integers(1, 300))),
                      (4, 4 * int(rng.integers(1, 100)))):
        res = rb.simulate(gids, rb.CacheConfig(cap, rb.Policy.LRU, ways))
        h, pa = oracle.lru(gids, V, cap, ways or 0, per_access=True)
        assert res.hits == h and res.per_access_hit == pa.tolist(), (ways, cap)


def test_priority_buffer_unit_examples():
    # Alg. 1 / Alg. 2 worked examples: test_runtime.py:24-88, test_acceptance.py:392-408
    def filled(prios, capacity=None, total=32):
        buf = rb.PriorityBuffer(capacity or len(prios), total)
        for g, p in prios.items():
            buf.add(g, p)
        return buf

    buf = filled({0: 0, 1: 0, 2: 0}, capacity=4)
    rb.load_embeddings(buf, [0, 1, 2], [1, 0, 1], [])
    assert buf.entries == {0: 5, 1: 4, 2: 5}
    buf = filled({3: 1, 7: 2}, capacity=2)
    rb.load_embeddings(buf, [], [], [7])
    assert buf.entries == {3: 1, 7: 4} and len(buf) == 2
    buf = filled({0: 5, 1: 4, 2: 5}, capacity=3)
    rb.load_embeddings(buf, [], [], [9])
    assert 9 in buf and 1 not in buf and len(buf) == 3 and buf.priority_of(9) == 4
    buf = filled({0: 5, 1: 4, 2: 5})
    assert rb.gpu_buffer_populate(buf) == 1 and buf.entries == {0: 4, 2: 4}
    buf = filled({3: 0, 5: 0, 7: 0})
    assert rb.gpu_buffer_populate(buf) == 3 and buf.entries == {5: 0, 7: 0}
    buf = filled({6: 2})
    assert rb.gpu_buffer_populate(buf) == 6
    with pytest.raises(ValueError):
        rb.gpu_buffer_populate(buf)
    buf = filled({0: 1}, capacity=1)
    with pytest.raises(ValueError):
        buf.add(0, 1)
    with pytest.raises(ValueError):
        buf.add(1, 1)
    with pytest.raises(KeyError):
        buf.priority_of(9)
    buf = rb.PriorityBuffer(2, 16)
    buf.add(4, 4, prefetched=True)
    assert buf.reference(4) is True and buf.reference(4) is False


def test_replay_deterministic_and_partition():
    t = rb.generate_trace(rb.TraceGenConfig([4, 100, 60], 4000, 1.05, 0.4, 24, 11))
    a = rb.replay(t, rb.BufferConfig(24), caching_fn=lambda s: [1] * 15)
    b = rb.replay(t, rb.BufferConfig(24), caching_fn=lambda s: [1] * 15)
    assert a == b and a.total == len(t)


def test_config1_golden_counts_on_gpu():
    z = golden("config1.npz")
    t = rb.generate_trace(rb.TraceGenConfig([2000] * 8, 1_000_000, 1.05, 0.4, 32, 0))
    K = int(z["bits_shape"][0])
    bits = np.unpackbits(z["bits_packed"])[:K * 15].reshape(K, 15)
    pf = z["pf"]
    C, C32 = int(z["C"]), int(z["C32"])
    cfn = lambda s: bits[s.origin // 15]
    pfn = lambda s: pf[s.origin // 15]
    for es_name, es in (("4", 4), ("C", C)):
        rep = rb.replay(t, rb.BufferConfig(C, es), caching_fn=cfn, prefetch_fn=pfn)
        assert _counts(rep) == list(z[f"fa_es{es_name}"][:7])
        assert rep.coverage == float(z[f"fa_es{es_name}_coverage"])
    for es_name, es in (("4", 4), ("C", C32)):
        rep = rb.replay(t, rb.BufferConfig(C32, es, 32), caching_fn=cfn, prefetch_fn=pfn)
        assert [rep.cache_hits, rep.prefetch_hits, rep.on_demand, rep.evictions,
                rep.prefetch_inserts] == list(z[f"w32_es{es_name}"][:5])
    res = rb.simulate(t, rb.CacheConfig(C32, rb.Policy.LRU, 32), per_access=False)
    assert res.misses == int(z["lru32_misses"])


def test_lru_plus_prefetch_vs_reference(small):
    """replay_policy_only with a prefetcher (runtime.py:304-349) == reference."""
    t = rb.trace_from_gids(small["gids"], [int(x) for x in small["table_sizes"]])
    pf = small["opt_pf"]
    rep = rb.replay_policy_only(t, rb.CacheConfig(24, rb.Policy.LRU),
                                prefetch_fn=lambda s: [int(g) for g in pf[s.origin // 15] if g >= 0])
    assert [rep.cache_hits, rep.prefetch_hits, rep.on_demand, rep.prefetch_issued,
            rep.prefetch_useful] == list(small["lrupf_counts"])
    assert rep.coverage == float(small["lrupf_coverage"])


@pytest.mark.parametrize("seed", range(3))
def test_lru_plus_prefetch_random_vs_oracle(seed):
    rng = np.random.default_rng(50 + seed)
    V = int(rng.integers(50, 2000))
    n = int(rng.integers(500, 30000))
    gids = (rng.zipf(1.2, n) - 1) % V
    K = rb.num_chunks(n)
    pf = rng.integers(0, V, (K, 5))
    pf[np.arange(5)[None, :] >= rng.integers(0, 6, K)[:, None]] = -1
    t = rb.trace_from_gids(gids, [V])
    for cap in (1, 7, int(rng.integers(8, 300))):
        rep = rb.replay_policy_only(t, rb.CacheConfig(cap, rb.Policy.LRU),
                                    prefetch_fn=lambda s: [int(g) for g in pf[s.origin // 15] if g >= 0])
        ref, cov = oracle.lru_prefetch(gids, V, cap, pf)
        assert [rep.cache_hits, rep.prefetch_hits, rep.on_demand, rep.prefetch_issued,
                rep.prefetch_useful] == [ref[k] for k in NAMES[:5]], cap
        assert rep.coverage == cov


def test_lfu_srrip_optgen_vs_reference(small):
    """simulate() for LFU / SRRIP / OPTGEN (cache_sim.py:109-249) == reference,
    incl. per-access hits and optgen keep decisions."""
    t = rb.trace_from_gids(small["gids"], [int(x) for x in small["table_sizes"]])
    pols = (rb.Policy.LFU, rb.Policy.SRRIP, rb.Policy.OPTGEN)
    for case, hits, pa, keep in zip(small["pol_cases"], small["pol_hits"],
                                    small["pol_per_access"], small["pol_keep"]):
        pol, cap, ways = pols[int(case[0])], int(case[1]), int(case[2]) or None
        res = rb.simulate(t, rb.CacheConfig(cap, pol, ways))
        assert res.hits == hits and res.per_access_hit == pa.tolist(), (pol, cap, ways)
        if pol == rb.Policy.OPTGEN:
            assert res.keep_decisions == keep.tolist(), (cap, ways)


def test_optgen_known_answers():
    # test_cache_sim.py:33-42
    res = rb.simulate_optgen(rb.trace_from_gids(letters("ABCABC"), [3]), 2)
    assert res.hits == 2 and res.per_access_hit == [0, 0, 0, 1, 0, 1]
    assert rb.simulate_optgen(rb.trace_from_gids([0, 0, 0], [2]), 1).hits == 2
    res = rb.simulate_optgen(rb.trace_from_gids(letters("ABACB"), [3]), 2)
    assert res.per_access_hit == [0, 0, 1, 0, 1] and res.keep_decisions == [1, 1, 0, 0, 0]
    # test_cache_sim.py:19-24 (LFU keeps the hot block)
    res = rb.simulate(rb.trace_from_gids(letters("AABCA"), [3]), rb.CacheConfig(2, rb.Policy.LFU))
    assert res.per_access_hit == [0, 1, 0, 0, 1]


def test_hot_runs_vs_reference():
    """One id carries 85% of the trace (long single-gid runs): the replay
    kernels' uniform-run fast path against the reference per-set buffer,
    simulate() for LRU/LFU/SRRIP/OPTGEN (per-access hits, keep bits) and
    replay_policy_only with prefetches; access classes against the oracle."""
    z = golden("hot_runs.npz")
    gids, bits, pf = z["gids"], z["bits"], z["pf"]
    t = rb.trace_from_gids(gids, [400])
    cfn, pfn = _fns(bits, pf)
    for case, cnt in zip(z["sa_cases"], z["sa_counts"]):
        cap, ways, es = (int(x) for x in case)
        rep, cls = rb.replay(t, rb.BufferConfig(cap, es, ways), caching_fn=cfn, prefetch_fn=pfn,
                             return_access_class=True)
        got = [rep.cache_hits, rep.prefetch_hits, rep.on_demand, rep.evictions,
               rep.prefetch_inserts]
        assert got == list(cnt[:5]), case
        _, _, rcls = oracle.replay(gids, 400, cap, ways, es, bits=bits, pf=pf, access_class=True)
        assert np.array_equal(cls, rcls), case
    pols = (rb.Policy.LRU, rb.Policy.LFU, rb.Policy.SRRIP, rb.Policy.OPTGEN)
    for case, hits, pa, keep in zip(z["pol_cases"], z["pol_hits"], z["pol_per_access"],
                                    z["pol_keep"]):
        pol, cap, ways = pols[int(case[0])], int(case[1]), int(case[2]) or None
        res = rb.simulate(t, rb.CacheConfig(cap, pol, ways))
        assert res.hits == hits and res.per_access_hit == pa.tolist(), (pol, cap, ways)
        if pol == rb.Policy.OPTGEN:
            assert res.keep_decisions == keep.tolist(), (cap, ways)
    for row in z["lrupf_counts"]:
        cap = int(row[0])
        rep = rb.replay_policy_only(t, rb.CacheConfig(cap, rb.Policy.LRU), prefetch_fn=pfn)
        assert [rep.cache_hits, rep.prefetch_hits, rep.on_demand, rep.prefetch_issued,
                rep.prefetch_useful] == [int(x) for x in row[1:]], cap
