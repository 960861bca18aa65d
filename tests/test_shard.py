"""Table shards with shard-local models.

CPU: the shard's parameters are init_params restricted to its tables
(bit-exact through the PCG64 jump-ahead), local ids map back to global ones,
and a world-2 gloo run of the streamed config-3 style generator gives every
rank the same assignment and a partition of the trace.
GPU: a shard's HotPath (local folded tables, decode over the global ids)
produces the same logits, decisions and replay counters as the unsharded
model run on the same sub-trace."""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2511_08568_b200 as rb
from paper_2511_08568_b200 import shard
from paper_2511_08568_b200.trace import generate_trace_streamed

SIZES = [900] * 10 + [300] * 6


def test_init_params_shard_is_init_params_restricted():
    tables = [1, 4, 5, 11, 15]
    sh = shard.TableShard(SIZES, tables)
    rows = np.concatenate([np.arange(sh.offsets[t], sh.offsets[t + 1]) for t in sh.tables])
    for kind, seed in (("caching", 0), ("prefetch", 1)):
        full = rb.init_params(kind, SIZES, dim=16, seed=seed, init_scale=0.4)
        p, emb = shard.init_params_shard(kind, SIZES, tables, dim=16, seed=seed,
                                         init_scale=0.4, device=False, block_rows=333)
        assert p.table_sizes == [SIZES[t] for t in sh.tables]
        assert np.array_equal(emb, full.arrays["embed_id"][rows].astype(np.float32))
        for k, v in p.arrays.items():
            want = full.arrays[k][sh.tables] if k == "embed_table" else full.arrays[k]
            assert np.array_equal(v, want), k


def test_local_ids_round_trip():
    sh = shard.TableShard(SIZES, [0, 7, 12])
    g = np.array([0, 899, 7 * 900, 7 * 900 + 5, 10 * 900 + 2 * 300 + 7, 900])
    lg, lt = sh.to_local(g)
    assert lt.tolist() == [0, 0, 1, 1, 2, -1]
    assert lg.tolist() == [0, 899, 900, 905, 1807, -1]


def _cfg3_small():
    return rb.TraceGenConfig(SIZES, 60_000, 1.05, 0.4, 32, 3)


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = generate_trace_streamed(_cfg3_small(), 7001)
    t = rb.trace_from_gids(g, SIZES)
    assign = shard.assign_tables(shard.table_access_counts(t), world)
    sub = shard.shard_trace(t, assign, rank)
    out[rank] = (assign.tolist(), sub.gid_array.tolist())
    dist.destroy_process_group()


def test_gloo_world2_streamed_shards_partition_trace():
    from test_dist import _free_port
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    ref = rb.generate_trace(_cfg3_small())
    assert out[0][0] == out[1][0]
    assign = np.asarray(out[0][0])
    tid = ref.table_ids
    for r in range(world):
        assert out[r][1] == ref.gid_array[assign[tid] == r].tolist()


@pytest.mark.gpu
@pytest.mark.parametrize("dim", [64, 16])
def test_shard_hotpath_matches_unsharded(dim):
    import torch
    from paper_2511_08568_b200.model import DeviceModel
    from paper_2511_08568_b200.pipeline import HotPath
    t = rb.generate_trace(rb.TraceGenConfig(SIZES, 40_000, 1.05, 0.4, 32, 5))
    assign = shard.assign_tables(shard.table_access_counts(t), 3)
    for r in range(3):
        sub = shard.shard_trace(t, assign, r)
        sh = shard.TableShard(SIZES, np.nonzero(assign == r)[0])
        cap = shard.shard_capacity(sub, 0.2, 32)
        full = [DeviceModel(rb.init_params(k, SIZES, dim=dim, seed=s, init_scale=0.4))
                for k, s in (("caching", 0), ("prefetch", 1))]
        loc = []
        for k, s in (("caching", 0), ("prefetch", 1)):
            p, emb = shard.init_params_shard(k, SIZES, sh, dim=dim, seed=s, init_scale=0.4)
            loc.append(DeviceModel(p, emb, decode_ids=sh.total_ids))
        a = HotPath(full[0], full[1], SIZES, cap, len(sub), lru_capacity=cap, pieces=3)
        b = HotPath(loc[0], loc[1], SIZES, cap, len(sub), lru_capacity=cap, pieces=3, shard=sh)
        ra = a.replay_host(sub.gid_array.astype(np.int32))
        rb_ = b.replay_host(sub.gid_array.astype(np.int32))
        torch.cuda.synchronize()
        assert ra == rb_
        assert (ra[0].evictions, ra[0].prefetch_inserts) == (rb_[0].evictions, rb_[0].prefetch_inserts)
        K = a.K
        assert torch.equal(a.clog[:K], b.clog[:K]) and torch.equal(a.plog[:K], b.plog[:K])
        assert torch.equal(a.bits[:K], b.bits[:K]) and torch.equal(a.pf[:K], b.pf[:K])
        assert int(a.pf[:K].max()) < sh.total_ids
