"""Generate the golden fixtures by running the REFERENCE package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py [--skip-config1]

Everything in tests/golden/*.npz comes from the reference's own code
(/root/reference/pkg/src/embcache): its trace generator, its models, its
``replay`` / ``simulate`` / ``replay_policy_only`` and its ``PriorityBuffer``.
The only glue written here is the per-set composition loop, which mirrors
runtime.py:254-280 line for line but keeps one reference ``PriorityBuffer``
per set — it is checked to equal ``replay`` at one set.
Evictions and prefetch inserts are counted by spying on the reference's
``PriorityBuffer.populate`` / ``add`` (the test_runtime.py:139-154 pattern).

Versions are recorded in each file (numpy's Generator streams are not
promised stable across numpy versions).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import embcache  # noqa: E402
from embcache import runtime as rt  # noqa: E402
from embcache import cache_sim  # noqa: E402
from embcache.neural import model as ref_model  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
META = {"numpy": np.__version__, "reference": getattr(embcache, "__version__", "?")}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


class Spy:
    """Counts populate() and prefetched add() calls on reference buffers."""

    def __init__(self):
        self.evictions = 0
        self.inserts = 0
        self.max_occ = 0

    def __enter__(self):
        self._pop = rt.PriorityBuffer.populate
        self._add = rt.PriorityBuffer.add
        spy = self

        def populate(buf):
            spy.evictions += 1
            return spy._pop(buf)

        def add(buf, gid, priority, prefetched=False):
            if prefetched:
                spy.inserts += 1
            r = spy._add(buf, gid, priority, prefetched)
            spy.max_occ = max(spy.max_occ, len(buf))
            return r

        rt.PriorityBuffer.populate = populate
        rt.PriorityBuffer.add = add
        return self

    def __exit__(self, *a):
        rt.PriorityBuffer.populate = self._pop
        rt.PriorityBuffer.add = self._add


def ref_replay(trace, capacity, es, bits, pf, l_in=15, l_out=5, window_ratio=3):
    """The reference replay with decisions injected; counters + spy counts."""
    samples = embcache.chunk(trace, l_in, l_out, window_ratio)
    idx = {s.origin: k for k, s in enumerate(samples)}
    cfn = (lambda s: [int(b) for b in bits[idx[s.origin]]]) if bits is not None else None
    pfn = (lambda s: [int(g) for g in pf[idx[s.origin]]]) if pf is not None else None
    with Spy() as spy:
        r = rt.replay(trace, rt.BufferConfig(capacity, es), l_in=l_in, l_out=l_out,
                      window_ratio=window_ratio, caching_fn=cfn, prefetch_fn=pfn)
    return [r.cache_hits, r.prefetch_hits, r.on_demand, r.prefetch_issued,
            r.prefetch_useful, spy.evictions, spy.inserts, spy.max_occ], r.coverage


def per_set_replay(trace, capacity, ways, es, bits, pf, l_in=15, l_out=5, window_ratio=3):
    """Per-set composition of reference PriorityBuffers; mirrors runtime.py:254-280."""
    S = capacity // ways
    V = trace.total_ids
    bufs = [rt.PriorityBuffer(ways, V, es) for _ in range(S)]
    ctr = dict(cache_hits=0, prefetch_hits=0, on_demand=0)
    gids = trace.gid_array
    samples = embcache.chunk(trace, l_in, l_out, window_ratio)

    def serve(g):
        buf = bufs[g % S]
        if g in buf:
            if buf.reference(g):
                ctr["prefetch_hits"] += 1
            else:
                ctr["cache_hits"] += 1
        else:
            ctr["on_demand"] += 1
            if buf.full:
                buf.populate()
            buf.add(g, buf.eviction_speed, prefetched=False)

    with Spy() as spy:
        for k, sample in enumerate(samples):
            chunk_gids = [int(gids[i]) for i in range(sample.origin, sample.origin + l_in)]
            for g in chunk_gids:
                serve(g)
            b = [int(x) for x in bits[k]] if bits is not None else [0] * l_in
            for g, bit in zip(chunk_gids, b):              # load_embeddings :126-130
                buf = bufs[g % S]
                if g in buf:
                    buf.set_priority(g, bit + buf.eviction_speed)
            for g in (list(pf[k]) if pf is not None else []):   # :131-137
                g = int(g)
                buf = bufs[g % S]
                if g in buf:
                    buf.set_priority(g, buf.eviction_speed)
                    continue
                if buf.full:
                    buf.populate()
                buf.add(g, buf.eviction_speed, prefetched=True)
        for i in range(len(samples) * l_in, len(gids)):
            serve(int(gids[i]))
    occ = sum(len(b) for b in bufs)
    return [ctr["cache_hits"], ctr["prefetch_hits"], ctr["on_demand"],
            spy.evictions, spy.inserts, occ]


def decisions(trace, cparams, pparams, l_in=15, l_out=5, window_ratio=3):
    samples = embcache.chunk(trace, l_in, l_out, window_ratio)
    bits = np.array(rt._model_bits(cparams, None, samples), dtype=np.uint8) \
        if cparams is not None else None
    pf = np.array(rt._model_prefetches(pparams, None, samples, trace.table_sizes),
                  dtype=np.int64) if pparams is not None else None
    return bits, pf


def pad(lists, stride):
    out = np.full((len(lists), stride), -1, dtype=np.int64)
    for k, p in enumerate(lists):
        out[k, :len(p)] = p
    return out


def make_small():
    """correlated_trace (conftest.py:23-29) + small models + many buffer configs."""
    cfg = embcache.TraceGenConfig(table_sizes=[4, 100, 60], total_accesses=4000,
                                  zipf_exponent=1.05, markov_stickiness=0.4,
                                  correlation_pool_size=24, rng_seed=11)
    t = embcache.generate_trace(cfg)
    cp = embcache.init_params("caching", t.table_sizes, dim=8, seed=3, init_scale=0.4)
    pp = embcache.init_params("prefetch", t.table_sizes, dim=8, seed=4, init_scale=0.4)
    bits, pf = decisions(t, cp, pp)
    out = {"gids": t.gid_array, "table_sizes": np.array(t.table_sizes),
           "bits": bits, "pf": pf}
    fa_cases, fa_counts, fa_cov = [], [], []
    for cap in (8, 24, 33, 64):
        for es in (4, 1, cap):
            for use_b, use_p in ((1, 1), (1, 0), (0, 1), (0, 0)):
                c, cov = ref_replay(t, cap, es, bits if use_b else None, pf if use_p else None)
                fa_cases.append([cap, es, use_b, use_p])
                fa_counts.append(c)
                fa_cov.append(cov)
    out["fa_cases"] = np.array(fa_cases)
    out["fa_counts"] = np.array(fa_counts)
    out["fa_coverage"] = np.array(fa_cov)
    # sanity: the per-set glue equals the reference at one set
    for cap, es in ((24, 4), (33, 33)):
        a = per_set_replay(t, cap, cap, es, bits, pf)
        b, _ = ref_replay(t, cap, es, bits, pf)
        assert a[:3] == b[:3] and a[3] == b[5] and a[4] == b[6], (a, b)
    sa_cases, sa_counts = [], []
    for cap, ways in ((32, 32), (64, 32), (64, 8), (24, 4), (30, 1), (96, 32)):
        for es in (4, cap):
            sa_cases.append([cap, ways, es])
            sa_counts.append(per_set_replay(t, cap, ways, es, bits, pf))
    out["sa_cases"] = np.array(sa_cases)
    out["sa_counts"] = np.array(sa_counts)
    # set-associative / fully associative LRU  (cache_sim.py:92-106)
    lru_cases, lru_hits, lru_pa = [], [], []
    for cap, ways in ((24, None), (24, 1), (24, 4), (32, 32), (64, 32), (96, 32), (7, None)):
        r = cache_sim.simulate(t, cache_sim.CacheConfig(cap, cache_sim.Policy.LRU, ways))
        lru_cases.append([cap, 0 if ways is None else ways])
        lru_hits.append(r.hits)
        lru_pa.append(np.array(r.per_access_hit, dtype=np.uint8))
    out["lru_cases"] = np.array(lru_cases)
    out["lru_hits"] = np.array(lru_hits)
    out["lru_per_access"] = np.stack(lru_pa)
    # LFU / SRRIP / optgen comparators (cache_sim.py:109-249), set-assoc and FA
    pol_cases, pol_hits, pol_pa, pol_keep = [], [], [], []
    for pi, pol in enumerate((cache_sim.Policy.LFU, cache_sim.Policy.SRRIP, cache_sim.Policy.OPTGEN)):
        for cap, ways in ((24, None), (24, 4), (32, 32), (64, 8), (96, 32), (7, None), (30, 1)):
            r = cache_sim.simulate(t, cache_sim.CacheConfig(cap, pol, ways))
            pol_cases.append([pi, cap, 0 if ways is None else ways])
            pol_hits.append(r.hits)
            pol_pa.append(np.array(r.per_access_hit, dtype=np.uint8))
            pol_keep.append(np.array(r.keep_decisions if r.keep_decisions is not None
                                     else [0] * len(t), dtype=np.uint8))
    out["pol_cases"] = np.array(pol_cases)
    out["pol_hits"] = np.array(pol_hits)
    out["pol_per_access"] = np.stack(pol_pa)
    out["pol_keep"] = np.stack(pol_keep)
    # variable-length prefetch lists from the optgen miss oracle
    # (test_runtime.py:157-171) with optgen keep bits
    cap = max(1, int(0.2 * t.unique_count))
    keep = cache_sim.simulate_optgen(t, cap).keep_decisions
    oracle = rt.optgen_miss_oracle(t, cap, l_out=5)
    samples = embcache.chunk(t)
    obits = np.array([keep[s.origin:s.origin + 15] for s in samples], dtype=np.uint8)
    opf = pad([oracle(s) for s in samples], 5)
    lists = [[int(g) for g in row if g >= 0] for row in opf]
    with Spy() as spy:
        r = rt.replay(t, rt.BufferConfig(cap), caching_fn=lambda s: keep[s.origin:s.origin + 15],
                      prefetch_fn=oracle)
    out["opt_cap"] = np.array(cap)
    out["opt_bits"] = obits
    out["opt_pf"] = opf
    out["opt_counts"] = np.array([r.cache_hits, r.prefetch_hits, r.on_demand,
                                  r.prefetch_issued, r.prefetch_useful, spy.evictions,
                                  spy.inserts, spy.max_occ])
    out["opt_coverage"] = np.array(r.coverage)
    lp = rt.replay_policy_only(t, cache_sim.CacheConfig(24, cache_sim.Policy.LRU),
                               prefetch_fn=lambda s: lists[s.origin // 15])
    out["lrupf_counts"] = np.array([lp.cache_hits, lp.prefetch_hits, lp.on_demand,
                                    lp.prefetch_issued, lp.prefetch_useful])
    out["lrupf_coverage"] = np.array(lp.coverage)
    out["meta"] = np.array(json.dumps(META))
    np.savez_compressed(os.path.join(HERE, "small_replay.npz"), **out)
    print("small_replay.npz written")


def make_hot():
    """A trace dominated by one id (85% of accesses, long runs): the replay
    kernels' uniform-run fast path (csrc/replay.cu) against the reference
    per-set buffer, simulate() policies and replay_policy_only."""
    rng = np.random.default_rng(77)
    V, n = 400, 12000
    gids = np.where(rng.random(n) < 0.85, 7, rng.integers(0, V, n)).astype(np.int64)
    gids[3000:3700] = 7                       # a run longer than any batch
    gids[5000:5400] = 7 + 64                  # a second hot id sharing set 7 (mod 32/64)
    t = embcache.trace_from_gids(gids, [V])
    K = len(embcache.chunk(t))
    bits = rng.integers(0, 2, (K, 15)).astype(np.uint8)
    pf = rng.integers(0, V, (K, 5))
    pf[rng.random((K, 5)) < 0.3] = 7          # full rows: per_set_replay takes them raw
    lists = [[int(g) for g in row] for row in pf]
    out = {"gids": gids, "bits": bits, "pf": pf}
    sa_cases, sa_counts = [], []
    for cap, ways in ((32, 32), (64, 32), (24, 4), (8, 8)):
        for es in (4, cap):
            sa_cases.append([cap, ways, es])
            sa_counts.append(per_set_replay(t, cap, ways, es, bits, pf))
    out["sa_cases"] = np.array(sa_cases)
    out["sa_counts"] = np.array(sa_counts)
    pol_cases, pol_hits, pol_pa, pol_keep = [], [], [], []
    for pi, pol in enumerate((cache_sim.Policy.LRU, cache_sim.Policy.LFU, cache_sim.Policy.SRRIP,
                              cache_sim.Policy.OPTGEN)):
        for cap, ways in ((32, 32), (64, 32), (24, 4), (40, None)):
            r = cache_sim.simulate(t, cache_sim.CacheConfig(cap, pol, ways))
            pol_cases.append([pi, cap, 0 if ways is None else ways])
            pol_hits.append(r.hits)
            pol_pa.append(np.array(r.per_access_hit, dtype=np.uint8))
            pol_keep.append(np.array(r.keep_decisions if r.keep_decisions is not None
                                     else [0] * len(t), dtype=np.uint8))
    out["pol_cases"] = np.array(pol_cases)
    out["pol_hits"] = np.array(pol_hits)
    out["pol_per_access"] = np.stack(pol_pa)
    out["pol_keep"] = np.stack(pol_keep)
    lp_counts = []
    for cap in (16, 100):
        lp = rt.replay_policy_only(t, cache_sim.CacheConfig(cap, cache_sim.Policy.LRU),
                                   prefetch_fn=lambda s: lists[s.origin // 15])
        lp_counts.append([cap, lp.cache_hits, lp.prefetch_hits, lp.on_demand,
                          lp.prefetch_issued, lp.prefetch_useful])
    out["lrupf_counts"] = np.array(lp_counts)
    out["meta"] = np.array(json.dumps(META))
    np.savez_compressed(os.path.join(HERE, "hot_runs.npz"), **out)
    print("hot_runs.npz written")


def make_artifacts():
    """Reference-written artifacts: a checkpoint (save_checkpoint,
    checkpoint.py:27-45), a text trace (write_trace, trace.py:164-169) and
    the reference's outcome (gids or error class + message) of read_trace on
    malformed traces."""
    p = embcache.init_params("prefetch", [30, 5, 70, 12], dim=8, seed=9, init_scale=0.4)
    embcache.save_checkpoint(p, os.path.join(HERE, "ref_ckpt_prefetch.npz"))
    t = embcache.generate_trace(embcache.TraceGenConfig([300, 50, 7], 3000, 1.05, 0.4, 32, 1))
    embcache.write_trace(t, os.path.join(HERE, "ref_trace.txt"))
    cases = {"hdr": "tbl: 1,2\n0,0\n", "badsize": "tables: 3,x\n", "neg": "tables: 3,0\n",
             "fields": "tables: 3,4\n0,1\n1,2,3\n", "nonint": "tables: 3,4\n0,1\n\n a , 2\n",
             "range": "tables: 3,4\n0,1\n2,0\n", "row": "tables: 3,4\n1,4\n",
             "ok_ws": "tables: 3,4\n 1 , 3 \n\n+0,2\n1_0,1\n",
             "crlf": "tables: 3,4\r\n0,1\r\n1,3\r\n\r\n1,9\r\n", "empty": "",
             "tail_blank": "tables: 3,4\n0,1\n   \n1,0\n\n"}
    out = {}
    import tempfile
    for k, body in cases.items():
        with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as f:
            f.write(body)
        try:
            r = embcache.read_trace(f.name)
            out[k] = {"body": body, "ok": [a.global_id for a in r.accesses],
                      "sizes": r.table_sizes}
        except Exception as e:  # noqa: BLE001 -- record the reference's outcome
            out[k] = {"body": body, "error": type(e).__name__, "msg": str(e)}
        os.unlink(f.name)
    with open(os.path.join(HERE, "ref_trace_cases.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("artifacts written")


def make_models():
    """Reference forward outputs for several shapes / init scales."""
    out = {}
    sizes = [4, 100, 60]
    rng = np.random.default_rng(5)
    total = sum(sizes)
    offsets = np.concatenate(([0], np.cumsum(sizes)))
    gid = rng.integers(0, total, size=(37, 15))
    tid = np.searchsorted(offsets, gid, side="right") - 1
    out["table_sizes"] = np.array(sizes)
    out["gid"] = gid
    out["tid"] = tid
    cases = []
    for kind in ("caching", "prefetch"):
        for dim, scale, seed in ((8, 0.4, 1), (16, 0.6, 2), (64, 0.08, 0), (64, 0.4, 7),
                                 (64, 0.6, 9), (5, 0.4, 3)):
            p = ref_model.init_params(kind, sizes, dim=dim, seed=seed, init_scale=scale)
            if kind == "caching":
                v = ref_model.forward_caching_batch(p, gid, tid).value
            else:
                v = ref_model.forward_prefetch_batch(p, gid, tid).value
                out[f"{kind}_{dim}_{seed}_decoded"] = np.array(
                    [[d.global_id for d in ref_model.decode_indices(list(r), sizes)] for r in v])
            key = f"{kind}_{dim}_{seed}"
            out[key + "_probs"] = v
            out[key + "_wsum"] = np.array([float(np.sum(a)) for a in p.arrays.values()])
            cases.append([0 if kind == "caching" else 1, dim, seed, scale])
    out["cases"] = np.array(cases)
    out["meta"] = np.array(json.dumps(META))
    np.savez_compressed(os.path.join(HERE, "models.npz"), **out)
    print("models.npz written")


def make_traces():
    """Generator determinism fixtures (trace.py:124-161)."""
    out = {}
    cfgs = [([4, 100, 60], 4000, 1.05, 0.4, 24, 11),
            ([8, 120], 6000, 1.0, 0.45, 16, 23),
            ([250] * 8, 20000, 1.05, 0.5, 32, 31),
            ([5], 50, 0.0, 0.0, 1, 7),
            ([2000] * 8, 100000, 1.05, 0.4, 32, 0)]
    for i, (ts, n, s, p, pool, seed) in enumerate(cfgs):
        t = embcache.generate_trace(embcache.TraceGenConfig(ts, n, s, p, pool, seed))
        out[f"cfg{i}"] = np.array(json.dumps([ts, n, s, p, pool, seed]))
        out[f"sha{i}"] = np.array(sha(t.gid_array))
        out[f"unique{i}"] = np.array(t.unique_count)
        if n <= 6000:
            out[f"gids{i}"] = t.gid_array.astype(np.int32)
    out["meta"] = np.array(json.dumps(META))
    np.savez_compressed(os.path.join(HERE, "traces.npz"), **out)
    print("traces.npz written")


def make_config1():
    """Config 1: reference decisions at init 0.4 + golden counts."""
    t0 = time.time()
    cfg = embcache.TraceGenConfig([2000] * 8, 1_000_000, 1.05, 0.4, 32, 0)
    t = embcache.generate_trace(cfg)
    cp = embcache.init_params("caching", t.table_sizes, dim=64, seed=0, init_scale=0.4)
    pp = embcache.init_params("prefetch", t.table_sizes, dim=64, seed=1, init_scale=0.4)
    bits, pf = decisions(t, cp, pp)
    print(f"config1 decisions {time.time() - t0:.1f}s")
    C = int(np.floor(0.2 * t.unique_count))
    C32 = C - C % 32
    out = {"sha": np.array(sha(t.gid_array)), "unique": np.array(t.unique_count),
           "C": np.array(C), "C32": np.array(C32),
           "bits_packed": np.packbits(bits.reshape(-1)), "bits_shape": np.array(bits.shape),
           "pf": pf.astype(np.int32)}
    for es_name, es in (("4", 4), ("C", C)):
        c, cov = ref_replay(t, C, es, bits, pf)
        out[f"fa_es{es_name}"] = np.array(c)
        out[f"fa_es{es_name}_coverage"] = np.array(cov)
        print(f"FA es={es_name}: {c} cov={cov!r} {time.time() - t0:.1f}s")
    for es_name, es in (("4", 4), ("C", C32)):
        c = per_set_replay(t, C32, 32, es, bits, pf)
        out[f"w32_es{es_name}"] = np.array(c)
        print(f"32-way es={es_name}: {c} {time.time() - t0:.1f}s")
    r = cache_sim.simulate(t, cache_sim.CacheConfig(C32, cache_sim.Policy.LRU, 32))
    out["lru32_misses"] = np.array(r.misses)
    r = cache_sim.simulate(t, cache_sim.CacheConfig(C, cache_sim.Policy.LRU))
    out["lru_fa_misses"] = np.array(r.misses)
    out["meta"] = np.array(json.dumps(META))
    np.savez_compressed(os.path.join(HERE, "config1.npz"), **out)
    print(f"config1.npz written {time.time() - t0:.1f}s")


def config1_inputs():
    """Config-1 trace and the reference decisions stored in config1.npz."""
    cfg = embcache.TraceGenConfig([2000] * 8, 1_000_000, 1.05, 0.4, 32, 0)
    t = embcache.generate_trace(cfg)
    z = np.load(os.path.join(HERE, "config1.npz"))
    assert str(z["sha"]) == sha(t.gid_array)
    shape = tuple(int(x) for x in z["bits_shape"])
    bits = np.unpackbits(z["bits_packed"])[:shape[0] * shape[1]].reshape(shape)
    return t, bits, z["pf"].astype(np.int64)


def make_wide():
    """Buffers wider than 4096 ways (the GPU's global-memory set kernel):
    the reference fully associative replay on the config-1 trace at 30% / 40%
    of its unique ids (es = 4 and es = C) with the config-1 reference
    decisions, a 2-set x 4160-way per-set composition, the fully associative
    LRU / LFU / optgen comparators and the labeler at 80% of those buffers;
    SRRIP and the LRU+prefetch baseline on a smaller trace."""
    t0 = time.time()
    t, bits, pf = config1_inputs()
    U = t.unique_count
    out = {"sha": np.array(sha(t.gid_array))}
    fa_cases, fa_counts, fa_cov = [], [], []
    for frac in (0.3, 0.4):
        C = int(np.floor(frac * U))
        for es in (4, C):
            c, cov = ref_replay(t, C, es, bits, pf)
            fa_cases.append([C, es])
            fa_counts.append(c)
            fa_cov.append(cov)
            print(f"wide FA C={C} es={es}: {c} {time.time() - t0:.1f}s")
    out["fa_cases"] = np.array(fa_cases)
    out["fa_counts"] = np.array(fa_counts)
    out["fa_coverage"] = np.array(fa_cov)
    out["sa_case"] = np.array([8320, 4160, 4])
    out["sa_counts"] = np.array(per_set_replay(t, 8320, 4160, 4, bits, pf))
    print(f"wide 2x4160 per-set {time.time() - t0:.1f}s")
    C = int(np.floor(0.4 * U))
    pol = {}
    for name, policy in (("lru", cache_sim.Policy.LRU), ("lfu", cache_sim.Policy.LFU),
                         ("optgen", cache_sim.Policy.OPTGEN)):
        r = cache_sim.simulate(t, cache_sim.CacheConfig(C, policy))
        out[f"{name}_hits"] = np.array(r.hits)
        out[f"{name}_pa_sha"] = np.array(sha(np.array(r.per_access_hit)))
        if r.keep_decisions is not None:
            out[f"{name}_keep_sha"] = np.array(sha(np.array(r.keep_decisions)))
        print(f"wide FA {name} C={C}: hits {r.hits} {time.time() - t0:.1f}s")
    # labeler.py:43-83 at 80% of the 20% buffer (2528 ways, shared-memory
    # kernel) and of the 40% buffer (5056 ways, global-memory kernel)
    from embcache import labeler
    samples = embcache.chunk(t)
    for name, gc in (("c20", int(np.floor(0.2 * U))), ("c40", C)):
        lc = labeler.label_caching(t, samples, gc)
        lab = np.array([s.cache_labels for s in lc.samples], dtype=np.uint8)
        lp = labeler.label_prefetch(t, samples, gc, l_out=5)
        tg = np.array([[a.global_id for a in s.prefetch_targets] for s in lp.samples],
                      dtype=np.int64)
        org = np.array([s.origin for s in lp.samples], dtype=np.int64)
        out[f"label_{name}_cap"] = np.array([gc, lc.label_capacity])
        out[f"label_{name}_caching_sha"] = np.array(sha(lab))
        out[f"label_{name}_caching_ones"] = np.array(int(lab.sum()))
        out[f"label_{name}_prefetch_sha"] = np.array(sha(tg))
        out[f"label_{name}_prefetch_origin_sha"] = np.array(sha(org))
        out[f"label_{name}_prefetch_dropped"] = np.array(lp.dropped)
        print(f"labels {name}: cap {lc.label_capacity} ones {int(lab.sum())} "
              f"dropped {lp.dropped} {time.time() - t0:.1f}s")
    # SRRIP / LFU / LRU+prefetch past 4096 ways on a smaller trace
    ts = embcache.generate_trace(embcache.TraceGenConfig([3000] * 4, 120_000, 1.05, 0.4, 32, 21))
    out["small_gids"] = ts.gid_array.astype(np.int32)
    out["small_table_sizes"] = np.array(ts.table_sizes)
    for name, policy in (("srrip", cache_sim.Policy.SRRIP), ("lfu", cache_sim.Policy.LFU),
                         ("lru", cache_sim.Policy.LRU), ("optgen", cache_sim.Policy.OPTGEN)):
        r = cache_sim.simulate(ts, cache_sim.CacheConfig(4160, policy))
        out[f"small_{name}_per_access"] = np.packbits(np.array(r.per_access_hit, dtype=np.uint8))
        out[f"small_{name}_hits"] = np.array(r.hits)
        print(f"small FA {name}: hits {r.hits} {time.time() - t0:.1f}s")
    oracle = rt.optgen_miss_oracle(ts, 6000, l_out=5)
    s_samples = embcache.chunk(ts)
    lists = [oracle(s) for s in s_samples]
    out["small_lrupf_pf"] = pad(lists, 5).astype(np.int32)
    lp = rt.replay_policy_only(ts, cache_sim.CacheConfig(4200, cache_sim.Policy.LRU),
                               prefetch_fn=lambda s: lists[s.origin // 15])
    out["small_lrupf_counts"] = np.array([lp.cache_hits, lp.prefetch_hits, lp.on_demand,
                                          lp.prefetch_issued, lp.prefetch_useful])
    out["small_lrupf_coverage"] = np.array(lp.coverage)
    out["meta"] = np.array(json.dumps(META))
    np.savez_compressed(os.path.join(HERE, "wide.npz"), **out)
    print(f"wide.npz written {time.time() - t0:.1f}s")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-config1", action="store_true")
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    jobs = {"small": make_small, "models": make_models, "traces": make_traces,
            "config1": make_config1, "hot": make_hot, "artifacts": make_artifacts,
            "wide": make_wide}
    for name, fn in jobs.items():
        if a.only and name != a.only:
            continue
        if name in ("config1", "wide") and a.skip_config1:
            continue
        fn()
