"""HotPath (pipeline.py) on the B200: the pipelined end-to-end call
(replay_host: two-part H2D copy, per-piece coverage summed on the host in
chunk order) equals the device-resident launch, the one-shot replay() API
and the C oracle driven by the same model decisions."""
import numpy as np
import pytest

import oracle
import paper_2511_08568_b200 as rb
from paper_2511_08568_b200.pipeline import HotPath

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pieces", [1, 3, 8])
def test_replay_host_matches_device_and_oracle(pieces):
    import torch
    t = rb.generate_trace(rb.TraceGenConfig([3000] * 16, 200_000, 1.05, 0.4, 32, 13))
    cp = rb.init_params("caching", t.table_sizes, dim=64, seed=0, init_scale=0.4)
    pp = rb.init_params("prefetch", t.table_sizes, dim=64, seed=1, init_scale=0.4)
    n = len(t)
    C = int(0.2 * t.unique_count)
    C32 = C - C % 32
    hp = HotPath(cp, pp, t.table_sizes, C32, n, ways=32, lru_capacity=C32, lru_ways=32,
                 pieces=pieces)
    host = torch.from_numpy(t.gid_array.astype(np.int32)).pin_memory()
    rep_h, lru_h = hp.replay_host(host)
    from paper_2511_08568_b200 import pipeline
    if pipeline._GRAPHS:   # the pinned end-to-end call runs as one captured CUDA graph
        assert hp._graph is not None
        rep_g, lru_g = hp.replay_host(host)   # a graph replay
        assert rep_g == rep_h and lru_g == lru_h
    K = hp.K
    bits = hp.bits[:K].cpu().numpy()
    pf = hp.pf[:K].cpu().numpy()
    hp.gids[:n].copy_(host)
    hp.launch(n)
    rep_d, lru_d = hp.report()
    assert rep_h == rep_d and lru_h == lru_d
    assert (rep_h.evictions, rep_h.prefetch_inserts) == (rep_d.evictions, rep_d.prefetch_inserts)
    ref, cov = oracle.replay(t.gid_array, t.total_ids, C32, 32, 4, bits=bits, pf=pf)
    assert [rep_h.cache_hits, rep_h.prefetch_hits, rep_h.on_demand, rep_h.prefetch_issued,
            rep_h.prefetch_useful, rep_h.evictions, rep_h.prefetch_inserts] == \
        [ref[k] for k in ("cache_hits", "prefetch_hits", "on_demand", "prefetch_issued",
                          "prefetch_useful", "evictions", "prefetch_inserts")]
    assert rep_h.coverage == cov
    assert lru_h[0] == oracle.lru(t.gid_array, t.total_ids, C32, 32)


def test_replay_host_edge_sizes_and_reuse():
    """One HotPath reused for traces of every awkward length: shorter than one
    chunk (all accesses are tail, served demand-only, runtime.py:278-280),
    exactly one chunk, fewer chunks than pieces x 128, and a ragged tail;
    each equals the one-shot replay() of the same prefix and the LRU
    simulator, so no state leaks from a longer earlier replay."""
    t = rb.generate_trace(rb.TraceGenConfig([700] * 8, 40_000, 1.05, 0.4, 32, 21))
    cp = rb.init_params("caching", t.table_sizes, dim=64, seed=0, init_scale=0.4)
    pp = rb.init_params("prefetch", t.table_sizes, dim=64, seed=1, init_scale=0.4)
    C = int(0.2 * t.unique_count)
    C32 = C - C % 32
    hp = HotPath(cp, pp, t.table_sizes, C32, len(t), ways=32, lru_capacity=C32, lru_ways=32,
                 pieces=8)
    for n in (40_000, 29, 30, 45, 1_000, 8 * 128 * 15 + 29, 40_000 - 7):
        sub = rb.trace_from_gids(t.gid_array[:n], t.table_sizes)
        rep, (h, m) = hp.replay_host(t.gid_array[:n].astype(np.int32))
        ref = rb.replay(sub, rb.BufferConfig(C32, 4, 32), cp, pp)
        assert rep == ref and (rep.evictions, rep.prefetch_inserts) == \
            (ref.evictions, ref.prefetch_inserts), n
        assert rep.total == n and h + m == n, n
        assert m == rb.simulate(sub, rb.CacheConfig(C32, rb.Policy.LRU, 32),
                                per_access=False).misses, n


@pytest.mark.parametrize("pf_first", [True, False])
def test_streamed_schedule_matches_oracle(monkeypatch, pf_first):
    """The streamed schedule (one forward launch per model, the second one
    releasing per-piece progress counters that the replay stream waits on:
    recmg_model_forward_signal / recmg_wait_progress) gives the oracle's counts."""
    import torch
    from paper_2511_08568_b200 import pipeline
    monkeypatch.setattr(pipeline, "_STREAMED", True)
    monkeypatch.setattr(pipeline, "_PF_FIRST", pf_first)
    t = rb.generate_trace(rb.TraceGenConfig([3000] * 16, 200_000, 1.05, 0.4, 32, 17))
    cp = rb.init_params("caching", t.table_sizes, dim=64, seed=0, init_scale=0.4)
    pp = rb.init_params("prefetch", t.table_sizes, dim=64, seed=1, init_scale=0.4)
    n = len(t)
    C = int(0.2 * t.unique_count)
    C32 = C - C % 32
    hp = HotPath(cp, pp, t.table_sizes, C32, n, ways=32, pieces=8)
    host = torch.from_numpy(t.gid_array.astype(np.int32)).pin_memory()
    for _ in range(2):   # the second pass reuses the progress counters' memory
        rep, _ = hp.replay_host(host)
    K = hp.K
    bits = hp.bits[:K].cpu().numpy()
    pf = hp.pf[:K].cpu().numpy()
    ref, cov = oracle.replay(t.gid_array, t.total_ids, C32, 32, 4, bits=bits, pf=pf)
    assert [rep.cache_hits, rep.prefetch_hits, rep.on_demand, rep.prefetch_issued,
            rep.prefetch_useful, rep.evictions, rep.prefetch_inserts] == \
        [ref[k] for k in ("cache_hits", "prefetch_hits", "on_demand", "prefetch_issued",
                          "prefetch_useful", "evictions", "prefetch_inserts")]
    assert rep.coverage == cov


@pytest.mark.parametrize("snapshot", [True, False])
def test_batch_hook_pools_each_batch_like_embedding_bag(snapshot):
    """Serving batches (piece_chunks) with the K5 + K6 hook after each
    batch's replay: on the state snapshot (its own stream, overlapping the
    next batch's replay) or in line on the live state, every batch's pooled
    bags equal torch embedding_bag of the host rows, the rows of the
    snapshot's resident slots are in HBM, and the counters equal a hook-less
    run of the same trace."""
    import torch
    import torch.nn.functional as F
    from paper_2511_08568_b200.engine import RowStore
    t = rb.generate_trace(rb.TraceGenConfig([3000] * 16, 120_000, 1.05, 0.4, 32, 17))
    cp = rb.init_params("caching", t.table_sizes, dim=64, seed=0, init_scale=0.4)
    pp = rb.init_params("prefetch", t.table_sizes, dim=64, seed=1, init_scale=0.4)
    n, V, D, P = len(t), t.total_ids, 32, 2
    C = int(0.2 * t.unique_count)
    C32 = C - C % 32
    host = torch.from_numpy(np.random.default_rng(5).standard_normal((V, D))
                            .astype(np.float32)).pin_memory()
    got, resident_ok = {}, []
    st = {}

    def hook(k0, k1, last, state):
        a0, a1 = 15 * k0, (n if last else 15 * k1)
        nb = -(-(a1 - a0) // P)
        off = torch.arange(0, nb * P + 1, P, dtype=torch.int64, device="cuda")
        off[-1] = a1 - a0
        st["rows"].refresh(state)
        out = st["rows"].pool(st["hp"].gids[a0:a1], off, state=state)
        got[(a0, a1)] = (out, off, state.clone(), st["rows"].buf.clone())

    hp = HotPath(cp, pp, t.table_sizes, C32, n, ways=32, lru_capacity=C32, lru_ways=32,
                 piece_chunks=1024, piece_hook=hook, hook_snapshot=snapshot)
    st.update(hp=hp, rows=RowStore(hp.buffer, host))
    hp.gids[:n].copy_(torch.from_numpy(t.gid_array.astype(np.int32)))
    hp.launch(n)
    rep, lru = hp.report()
    assert len(got) == -(-hp.K // 1024) > 4
    S = C32 // 32
    for (a0, a1), (out, off, state, buf) in got.items():
        ids = torch.from_numpy(t.gid_array[a0:a1]).long()
        want = F.embedding_bag(ids, host, off[:-1].cpu(), mode="sum")
        assert torch.equal(out.cpu(), want), (a0, (out.cpu() - want).abs().max())
        tags = state[64:64 + 4 * S * 32].view(torch.int32).cpu().numpy()
        res = tags >= 0
        assert np.array_equal(buf.cpu().numpy()[res], host.numpy()[tags[res]])
    plain = HotPath(cp, pp, t.table_sizes, C32, n, ways=32, lru_capacity=C32, lru_ways=32,
                    piece_chunks=1024)
    plain.gids[:n].copy_(hp.gids[:n])
    plain.launch(n)
    assert plain.report() == (rep, lru)
