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
