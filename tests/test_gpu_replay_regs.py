"""The register-resident set replay (`replay_set_regs`, sets of <= 32 ways that
are not on the heavy list) against the oracle and against the shared-memory
path (`RECMG_REPLAY_REGS=0`) on the same inputs, at sizes where both paths
run in one launch: hundreds of sets, Zipf-skewed so the heavy list is full."""
import os

import numpy as np
import pytest

import oracle
import paper_2511_08568_b200 as rb

pytestmark = pytest.mark.gpu

NAMES = ("cache_hits", "prefetch_hits", "on_demand", "prefetch_issued", "prefetch_useful",
         "evictions", "prefetch_inserts")


def _counts(rep):
    return [rep.cache_hits, rep.prefetch_hits, rep.on_demand, rep.prefetch_issued,
            rep.prefetch_useful, rep.evictions, rep.prefetch_inserts]


class _regs:
    def __init__(self, on):
        self.on = on

    def __enter__(self):
        self.old = os.environ.get("RECMG_REPLAY_REGS")
        os.environ["RECMG_REPLAY_REGS"] = self.on if isinstance(self.on, str) else (
            "-1" if self.on else "0")

    def __exit__(self, *exc):
        if self.old is None:
            os.environ.pop("RECMG_REPLAY_REGS", None)
        else:
            os.environ["RECMG_REPLAY_REGS"] = self.old


def _workload(seed, V, n):
    rng = np.random.default_rng(seed)
    gids = (rng.zipf(1.05, n) - 1) % V
    K = rb.num_chunks(n)
    bits = rng.integers(0, 2, (K, 15)).astype(np.uint8)
    # prefetch ids drawn from the trace itself (so some are hits), ragged lists
    pf = gids[rng.integers(0, n, (K, 5))]
    lens = rng.integers(0, 6, K)
    pf[np.arange(5)[None, :] >= lens[:, None]] = -1
    return gids, bits, pf


@pytest.mark.parametrize("seed,V,n,ways,sets,es", [
    (0, 200_000, 2_000_000, 32, 500, 4),
    (1, 50_000, 1_000_000, 32, 300, 1),
    (2, 100_000, 1_500_000, 16, 400, 4),
    (3, 30_000, 600_000, 32, 40, 7),
    # 25-bit gids and es = 130: the priorities do not fit the one-word victim
    # key, so the two-word argmin runs
    (4, 1 << 25, 400_000, 32, 60, 130),
])
@pytest.mark.parametrize("mode", ["-1", "1"])
def test_priority_replay_regs_vs_oracle_and_smem(seed, V, n, ways, sets, es, mode):
    gids, bits, pf = _workload(seed, V, n)
    t = rb.trace_from_gids(gids, [V])
    cap = ways * sets
    cfg = rb.BufferConfig(cap, es, ways)
    kw = dict(caching_fn=lambda s: bits[s.origin // 15],
              prefetch_fn=lambda s: [int(g) for g in pf[s.origin // 15] if g >= 0],
              return_access_class=True)
    with _regs(mode):
        rep, cls = rb.replay(t, cfg, **kw)
    with _regs(False):
        rep0, cls0 = rb.replay(t, cfg, **kw)
    ref, cov, rcls = oracle.replay(gids, V, cap, ways, es, bits=bits, pf=pf, access_class=True)
    assert _counts(rep) == [ref[k] for k in NAMES]
    assert _counts(rep0) == _counts(rep)
    assert rep.coverage == cov
    assert np.array_equal(cls, rcls)
    assert np.array_equal(cls0, cls)


@pytest.mark.parametrize("seed,V,n,ways,sets", [
    (10, 200_000, 2_000_000, 32, 600),
    (11, 20_000, 500_000, 8, 200),
])
def test_lru_regs_vs_oracle_and_smem(seed, V, n, ways, sets):
    rng = np.random.default_rng(seed)
    gids = (rng.zipf(1.05, n) - 1) % V
    cfg = rb.CacheConfig(ways * sets, rb.Policy.LRU, ways)
    with _regs(True):
        res = rb.simulate(gids, cfg)
    with _regs(False):
        res0 = rb.simulate(gids, cfg)
    h, pa = oracle.lru(gids, V, ways * sets, ways, per_access=True)
    assert res.hits == h and res.per_access_hit == pa.tolist()
    assert res0.hits == h


def test_priority_state_after_piecewise_replay_matches_smem():
    """The buffer state a replay leaves (tags, priorities with the decay
    applied, prefetch tags, counts) is byte-identical on both paths, replayed
    in 3 chunk ranges that continue the state (recmg_replay_chunks_ex)."""
    import torch
    from paper_2511_08568_b200.engine import BufferReplay
    gids, bits, pf = _workload(7, 80_000, 900_000)
    n = len(gids)
    K = rb.num_chunks(n)
    dev = torch.device("cuda:0")
    g = torch.as_tensor(gids.astype(np.int32), device=dev)
    b = torch.as_tensor(bits, device=dev)
    p = torch.as_tensor(pf.astype(np.int32), device=dev)
    out = []
    for on in (True, False):
        with _regs(on):
            eng = BufferReplay(32 * 250, 80_000, 4, 32, n=n, pf_stride=5)
            cuts = [0, K // 3, 2 * K // 3, K]
            for k0, k1 in zip(cuts[:-1], cuts[1:]):
                eng.run_chunks(g, k0, k1, k1 == K, bits=b, pf=p)
            res = eng.result()
            raw = eng.state.cpu().numpy().copy()
            # header (64 B), tags [S*W] int32, meta [S*W] int64, count [S] int32,
            # each region 256-B aligned (common.cuh state_view); padding is not state
            S, W = 250, 32
            tags = raw[64:64 + 4 * S * W].view(np.int32)
            mo = 64 + -(-4 * S * W // 256) * 256
            meta = raw[mo:mo + 8 * S * W].view(np.int64)
            co = mo + -(-8 * S * W // 256) * 256
            count = raw[co:co + 4 * S].view(np.int32)
            out.append((res, tags, meta, count))
    assert out[0][0] == out[1][0]
    for x, y in zip(out[0][1:], out[1][1:]):
        assert np.array_equal(x, y)
    assert (out[0][1] >= 0).sum() == out[0][3].sum()


@pytest.mark.parametrize("seed,V,n,sets,pieces", [
    (20, 200_000, 2_000_000, 500, 1),
    (21, 60_000, 900_000, 120, 3),
    (22, 3_000, 100_000, 8, 2),
])
def test_lru_fused_into_replay(seed, V, n, sets, pieces):
    """recmg_replay_chunks_lru: the 32-way LRU comparator replayed on the serves
    of the priority replay's own events (collapsed repeat serves included as
    hits) equals simulate() and the oracle, with the priority replay itself
    unchanged; chunk ranges continue both states."""
    import torch
    from paper_2511_08568_b200.engine import BufferReplay, LruSim
    gids, bits, pf = _workload(seed, V, n)
    K = rb.num_chunks(n)
    dev = torch.device("cuda:0")
    g = torch.as_tensor(gids.astype(np.int32), device=dev)
    b = torch.as_tensor(bits, device=dev)
    p = torch.as_tensor(pf.astype(np.int32), device=dev)
    cap = 32 * sets
    fused, plain = BufferReplay(cap, V, 4, 32, n=n, pf_stride=5), BufferReplay(cap, V, 4, 32, n=n,
                                                                                pf_stride=5)
    lru = LruSim(cap, V, 32, n)
    assert fused.fusable_lru(lru)
    cuts = [K * i // pieces for i in range(pieces + 1)]
    for k0, k1 in zip(cuts[:-1], cuts[1:]):
        assert fused.run_chunks_lru(g, k0, k1, k1 == K, lru, bits=b, pf=p)
        plain.run_chunks(g, k0, k1, k1 == K, bits=b, pf=p)
    assert fused.result() == plain.result()
    h, m = lru.result()
    hr, _ = oracle.lru(gids, V, cap, 32, per_access=True)
    assert (h, m) == (hr, n - hr)
    assert rb.simulate(gids, rb.CacheConfig(cap, rb.Policy.LRU, 32)).hits == h
