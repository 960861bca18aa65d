"""Multi-process (gloo, world size 2) coverage of the table-sharded path on
CPU: every rank builds the same assignment, replays its own shard (the
oracle stands in for the GPU replay here) and the summed counters equal the
single-process sum over shards."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2511_08568_b200 as rb
from paper_2511_08568_b200 import shard


def _trace():
    return rb.generate_trace(rb.TraceGenConfig([300] * 12 + [40] * 4, 30000, 1.05, 0.4, 32, 7))


def _shard_counts(t, assign, r):
    import oracle
    sub = shard.shard_trace(t, assign, r)
    cap = shard.shard_capacity(sub, 0.2, 32)
    res, _ = oracle.replay(sub.gid_array, t.total_ids, cap, 32, 4)
    return res


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = _trace()
    assign = shard.assign_tables(shard.table_access_counts(t), world)
    local = _shard_counts(t, assign, rank)
    total = shard.reduce_counters(local)
    out[rank] = (total, assign.tolist(), len(shard.shard_trace(t, assign, rank)))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_assignment_is_balanced_and_deterministic():
    t = _trace()
    counts = shard.table_access_counts(t)
    assert counts.sum() == len(t)
    for n in (2, 4, 8):
        a = shard.assign_tables(counts, n)
        assert np.array_equal(a, shard.assign_tables(counts, n))
        loads = np.bincount(a, weights=counts, minlength=n)
        # LPT bound: max load <= mean + the largest single table
        assert loads.max() <= counts.sum() / n + counts.max()
        # shards partition the trace, order preserved
        parts = [shard.shard_trace(t, a, r).gid_array for r in range(n)]
        assert sum(len(p) for p in parts) == len(t)
        merged = np.sort(np.concatenate(parts))
        assert np.array_equal(merged, np.sort(t.gid_array))


def test_gloo_world2_counters_sum():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    t = _trace()
    assign = shard.assign_tables(shard.table_access_counts(t), world)
    want = {k: 0 for k in shard.COUNTERS}
    for r in range(world):
        c = _shard_counts(t, assign, r)
        for k in shard.COUNTERS:
            want[k] += c[k]
    assert out[0][0] == want and out[1][0] == want
    assert out[0][1] == out[1][1] == assign.tolist()
    assert out[0][2] + out[1][2] == len(t)


def _dlrm_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    import torch.nn.functional as F
    from paper_2511_08568_b200 import dlrm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = _trace()
    assign = shard.assign_tables(shard.table_access_counts(t), world)
    rows = torch.from_numpy(np.random.default_rng(3).standard_normal((t.total_ids, 8))
                            .astype(np.float32))
    pool = lambda ids, offs: F.embedding_bag(ids.long(), rows, offs[:-1], mode="sum")
    stage = dlrm.DlrmEmbeddingStage(t.table_sizes, assign, rank, world, 8, pool)
    bags = torch.from_numpy(dlrm.build_bags(t, stage.local_tables, 6, 3, start=rank * 0))
    out[rank] = stage.forward(bags).numpy()
    dist.destroy_process_group()


def test_gloo_world2_dlrm_all_to_all():
    """Config-4 layout: table-sharded pooling + one all_to_all_single gives
    every rank the pooled rows of all tables for its block of samples."""
    import torch
    import torch.nn.functional as F
    from paper_2511_08568_b200 import dlrm
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_dlrm_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    t = _trace()
    rows = torch.from_numpy(np.random.default_rng(3).standard_normal((t.total_ids, 8))
                            .astype(np.float32))
    all_bags = dlrm.build_bags(t, list(range(len(t.table_sizes))), 6, 3)   # [6, T, 3]
    want = F.embedding_bag(torch.from_numpy(all_bags.reshape(-1, 3)), rows, mode="sum")
    want = want.reshape(6, len(t.table_sizes), 8).numpy()
    assert np.array_equal(out[0], want[:3]) and np.array_equal(out[1], want[3:])
