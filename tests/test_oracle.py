"""The oracle (test infrastructure) against the reference's own outputs.

Every fixture in tests/golden/ was produced by running the reference package
(tests/golden/make_golden.py); these CPU tests pin the C and numpy
restatements to them before any GPU result is compared with the oracle.
"""
import numpy as np
import pytest

import oracle
from oracle import model_oracle as mo
from conftest import golden, letters


def test_fa_replay_matches_reference(small):
    g, V = small["gids"], int(small["table_sizes"].sum())
    for case, cnt, cov in zip(small["fa_cases"], small["fa_counts"], small["fa_coverage"]):
        cap, es, ub, up = (int(x) for x in case)
        for dense in (True, False):
            r, c = oracle.replay(g, V, cap, 0, es, bits=small["bits"] if ub else None,
                                 pf=small["pf"] if up else None, dense=dense)
            assert [r[k] for k in oracle.COUNTER_NAMES] == list(cnt), (case, dense)
            assert c == cov  # float64 coverage, bit-exact


def test_per_set_replay_matches_reference_composition(small):
    g, V = small["gids"], int(small["table_sizes"].sum())
    for case, cnt in zip(small["sa_cases"], small["sa_counts"]):
        cap, ways, es = (int(x) for x in case)
        for dense in (True, False):
            r, _ = oracle.replay(g, V, cap, ways, es, bits=small["bits"], pf=small["pf"],
                                 dense=dense)
            got = [r["cache_hits"], r["prefetch_hits"], r["on_demand"], r["evictions"],
                   r["prefetch_inserts"]]
            assert got == list(cnt[:5]), (case, dense)


def test_lru_matches_reference(small):
    g, V = small["gids"], int(small["table_sizes"].sum())
    for case, hits, pa in zip(small["lru_cases"], small["lru_hits"], small["lru_per_access"]):
        h, p = oracle.lru(g, V, int(case[0]), int(case[1]), per_access=True)
        assert h == hits and np.array_equal(p, pa), case


def test_variable_length_prefetch_lists(small):
    g, V = small["gids"], int(small["table_sizes"].sum())
    r, c = oracle.replay(g, V, int(small["opt_cap"]), 0, 4, bits=small["opt_bits"],
                         pf=small["opt_pf"])
    assert [r[k] for k in oracle.COUNTER_NAMES] == list(small["opt_counts"])
    assert c == float(small["opt_coverage"])


def test_lru_plus_prefetch(small):
    g, V = small["gids"], int(small["table_sizes"].sum())
    r, c = oracle.lru_prefetch(g, V, 24, small["opt_pf"])
    assert [r[k] for k in oracle.COUNTER_NAMES[:5]] == list(small["lrupf_counts"])
    assert c == float(small["lrupf_coverage"])


def test_model_restatement_exact():
    m = golden("models.npz")
    sizes = [int(s) for s in m["table_sizes"]]
    for kind, dim, seed, scale in m["cases"]:
        kind = "caching" if kind == 0 else "prefetch"
        dim, seed = int(dim), int(seed)
        arr = mo.init_arrays(kind, sizes, dim, seed=seed, init_scale=float(scale))
        assert np.array_equal(np.array([float(np.sum(a)) for a in arr.values()]),
                              m[f"{kind}_{dim}_{seed}_wsum"])
        if kind == "caching":
            logit = mo.caching_logits(arr, dim, 1, m["gid"], m["tid"])
        else:
            logit = mo.prefetch_logits(arr, dim, 2, 5, m["gid"], m["tid"])
            assert np.array_equal(mo.decode_gids(mo.sigmoid(logit), sum(sizes)),
                                  m[f"{kind}_{dim}_{seed}_decoded"])
        assert np.abs(mo.sigmoid(logit) - m[f"{kind}_{dim}_{seed}_probs"]).max() == 0.0


def test_known_answers():
    # cache_sim tests: test_cache_sim.py:13-16, 108-112
    abc = np.array(letters("ABCABC"))
    assert oracle.lru(abc, 3, 2) == 0
    assert oracle.lru(abc, 3, 3) == 3
    _, pa = oracle.lru(np.array([0, 2, 0, 1, 1]), 4, 2, ways=1, per_access=True)
    assert pa.tolist() == [0, 0, 0, 0, 1]
    # replay tail: test_runtime.py:123-128
    r, _ = oracle.replay(np.arange(37), 64, 8)
    assert r["on_demand"] == 37 and r["cache_hits"] + r["prefetch_hits"] == 0
    # chunk counts: SPEC trace examples (45 -> 2, 14 -> 0)
    assert oracle.num_chunks(45) == 2 and oracle.num_chunks(14) == 0
    assert oracle.num_chunks(30, 10, 5, 2) == 2


def test_config1_golden_counts_oracle():
    z = golden("config1.npz")
    from paper_2511_08568_b200.trace import TraceGenConfig, generate_trace
    import hashlib
    t = generate_trace(TraceGenConfig([2000] * 8, 1_000_000, 1.05, 0.4, 32, 0))
    assert hashlib.sha256(t.gid_array.tobytes()).hexdigest() == str(z["sha"])
    K = int(z["bits_shape"][0])
    bits = np.unpackbits(z["bits_packed"])[:K * 15].reshape(K, 15)
    pf = z["pf"].astype(np.int64)
    C, C32 = int(z["C"]), int(z["C32"])
    r, cov = oracle.replay(t.gid_array, 16000, C, 0, 4, bits=bits, pf=pf)
    assert [r[k] for k in oracle.COUNTER_NAMES] == list(z["fa_es4"])
    assert cov == float(z["fa_es4_coverage"])
    r, _ = oracle.replay(t.gid_array, 16000, C32, 32, 4, bits=bits, pf=pf)
    assert [r["cache_hits"], r["prefetch_hits"], r["on_demand"], r["evictions"],
            r["prefetch_inserts"]] == list(z["w32_es4"][:5])
    assert 1_000_000 - oracle.lru(t.gid_array, 16000, C32, 32) == int(z["lru32_misses"])


def test_oracle_hot_runs_vs_reference():
    """The C oracle on the hot-run fixture (one id = 85% of accesses) equals
    the reference's per-set buffer and LRU."""
    z = golden("hot_runs.npz")
    gids, bits, pf = z["gids"], z["bits"], z["pf"]
    for case, cnt in zip(z["sa_cases"], z["sa_counts"]):
        cap, ways, es = (int(x) for x in case)
        ref, _ = oracle.replay(gids, 400, cap, ways, es, bits=bits, pf=pf)
        got = [ref[k] for k in ("cache_hits", "prefetch_hits", "on_demand", "evictions",
                                "prefetch_inserts")]
        assert got == list(cnt[:5]), case
    for case, hits, pa in zip(z["pol_cases"], z["pol_hits"], z["pol_per_access"]):
        if int(case[0]) != 0:
            continue
        cap, ways = int(case[1]), int(case[2])
        h, p = oracle.lru(gids, 400, cap, ways, per_access=True)
        assert h == hits and np.array_equal(p, pa), case


def test_trace_oracle_matches_reference_hashes():
    """oracle.trace_oracle (the reference arm's workload generator, no product
    import) reproduces the reference generate_trace outputs."""
    import hashlib
    import json
    from oracle import trace_oracle
    z = golden("traces.npz")
    i = 0
    while f"cfg{i}" in z:
        ts, n, s, p, pool, seed = json.loads(str(z[f"cfg{i}"]))
        g = trace_oracle.generate_gids(ts, n, s, p, pool, seed)
        assert hashlib.sha256(g.astype(np.int64).tobytes()).hexdigest() == str(z[f"sha{i}"])
        assert np.unique(g).size == int(z[f"unique{i}"])
        for block in (997, 1 << 20):
            gb = np.concatenate(list(trace_oracle.generate_gid_blocks(ts, n, s, p, pool, seed,
                                                                      block)))
            assert np.array_equal(gb, g)
        i += 1
    c1 = golden("config1.npz")
    g = trace_oracle.generate_gids([2000] * 8, 1_000_000, 1.05, 0.4, 32, 0)
    assert hashlib.sha256(g.astype(np.int64).tobytes()).hexdigest() == str(c1["sha"])


def test_oracle_wide_buffers_match_reference():
    """The C oracle at the fully associative capacities past 4096 ways
    (tests/golden/wide.npz, reference replay with the config-1 decisions)."""
    from oracle import trace_oracle
    z = golden("wide.npz")
    c1 = golden("config1.npz")
    g = trace_oracle.generate_gids([2000] * 8, 1_000_000, 1.05, 0.4, 32, 0)
    K = int(c1["bits_shape"][0])
    bits = np.unpackbits(c1["bits_packed"])[:K * 15].reshape(K, 15)
    pf = c1["pf"].astype(np.int64)
    for case, cnt, cov in zip(z["fa_cases"], z["fa_counts"], z["fa_coverage"]):
        C, es = (int(x) for x in case)
        ref, c = oracle.replay(g, 16000, C, 0, es, bits=bits, pf=pf)
        assert [ref[k] for k in oracle.COUNTER_NAMES] == list(cnt), case
        assert c == float(cov)
