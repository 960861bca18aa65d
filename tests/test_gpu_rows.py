"""K5 host-row gathers + K6 EmbeddingBag vs torch.nn.functional.embedding_bag
on the CPU (the reference has no row data; parity unpinned by
the reference, oracle = torch embedding_bag(mode='sum'))."""
import numpy as np
import pytest

import paper_2511_08568_b200 as rb
from paper_2511_08568_b200.engine import BufferReplay, RowStore, to_device_gids

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dim,ways,bag", [(128, 32, 2), (16, 8, 5), (64, 32, 1), (256, 4, 3)])
def test_gather_and_pool_vs_torch(dim, ways, bag):
    import torch
    import torch.nn.functional as F
    rng = np.random.default_rng(dim + ways)
    t = rb.generate_trace(rb.TraceGenConfig([3000] * 4, 40_000, 1.05, 0.4, 32, dim))
    V = t.total_ids
    host = torch.from_numpy(rng.standard_normal((V, dim)).astype(np.float32)).pin_memory()
    C = int(0.2 * t.unique_count)
    C -= C % ways
    K = rb.num_chunks(len(t))
    bits = torch.from_numpy(rng.integers(0, 2, (K, 15)).astype(np.uint8)).cuda()
    pf = torch.from_numpy(rng.integers(0, V, (K, 5)).astype(np.int32)).cuda()
    rep = BufferReplay(C, V, 4, ways, len(t), pf_stride=5)
    rows = RowStore(rep, host)
    g = to_device_gids(torch, t.gid_array)
    half = (K // 2)
    pieces = [(0, half, False), (half, K, True)]
    n_bags = len(t) // bag
    offsets = torch.arange(0, (n_bags + 1) * bag, bag, dtype=torch.int64).cuda()
    want = F.embedding_bag(torch.from_numpy(t.gid_array[:n_bags * bag]).long(), host,
                           offsets[:-1].cpu(), mode="sum")
    for k0, k1, tail in pieces:
        rep.run_chunks(g, k0, k1, tail, bits, pf)
        rows.refresh()
        torch.cuda.synchronize()
        # every resident slot holds exactly its id's host row
        st = rep.state
        S, W = C // ways, ways
        tags = st[64:64 + 4 * S * W].view(torch.int32).cpu().numpy()
        buf = rows.buf.cpu().numpy()
        res = tags >= 0
        assert np.array_equal(buf[res], host.numpy()[tags[res]])
        out = rows.pool(g[:n_bags * bag], offsets)
        got = out.cpu()
        assert torch.equal(got, want), (got - want).abs().max()
    hb, hh = (int(x) for x in rows.src.cpu().numpy())
    assert hb + hh == 2 * n_bags * bag and hb > 0


def test_dlrm_stage_single_rank_nccl():
    """Config-4 stage on one GPU: replay the batch's accesses (K3), gather
    changed rows (K5), pool the bags (K6), all-to-all over NCCL (world 1)."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    import torch.nn.functional as F
    from paper_2511_08568_b200 import dlrm, shard
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        t = rb.generate_trace(rb.TraceGenConfig([2000] * 6, 30_000, 1.05, 0.4, 32, 8))
        V, D = t.total_ids, 128
        host = torch.from_numpy(np.random.default_rng(1).standard_normal((V, D))
                                .astype(np.float32)).pin_memory()
        assign = shard.assign_tables(shard.table_access_counts(t), 1)
        B, P = 64, 2
        bags = dlrm.build_bags(t, list(range(6)), B, P)
        flat = bags.reshape(-1)
        C = 32 * 20
        rep = BufferReplay(C, V, 4, 32, len(flat))
        rows = RowStore(rep, host)
        g = to_device_gids(torch, flat)
        rep.run(g)
        rows.refresh()
        stage = dlrm.DlrmEmbeddingStage(t.table_sizes, assign, 0, 1, D, rows.pool)
        got = stage.forward(torch.from_numpy(bags).cuda()).cpu()
        want = F.embedding_bag(torch.from_numpy(flat.reshape(-1, P)), host, mode="sum")
        assert torch.equal(got, want.reshape(B, 6, D))
    finally:
        dist.destroy_process_group()


def _a2a_worker(rank, world, port, out):
    import os
    import torch
    import torch.distributed as dist
    import torch.nn.functional as F
    from paper_2511_08568_b200 import dlrm, shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        t = rb.generate_trace(rb.TraceGenConfig([1500] * 7, 30_000, 1.05, 0.4, 32, 8))
        V, D, B, P = t.total_ids, 64, 32, 3
        host = torch.from_numpy(np.random.default_rng(1).standard_normal((V, D))
                                .astype(np.float32)).pin_memory()
        assign = shard.assign_tables(shard.table_access_counts(t), world)
        mine = [tt for tt in range(7) if assign[tt] == rank]
        bags = dlrm.build_bags(t, mine, B, P)
        flat = bags.reshape(-1)
        rep = BufferReplay(32 * 8, V, 4, 32, len(flat))
        rows = RowStore(rep, host)
        rep.run(to_device_gids(torch, flat))      # some rows resident in HBM, the rest host
        rows.refresh()
        ex = dlrm.PeerExchange(rows, t.table_sizes, assign, rank, world, B)
        res = []
        for _ in range(3):                        # both output buffers, reused
            res.append(ex.forward(torch.from_numpy(bags).cuda()).clone())
        torch.cuda.synchronize()
        allb = dlrm.build_bags(t, list(range(7)), B, P)
        want = F.embedding_bag(torch.from_numpy(allb.reshape(-1, P)), host, mode="sum")
        want = want.reshape(B, 7, D)[rank * B // world:(rank + 1) * B // world]
        out[rank] = all(torch.equal(r.cpu(), want) for r in res)
        dist.barrier()
        ex.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2])
def test_fused_pooled_all_to_all_over_peer_memory(world):
    """K7 fused (config 4): the pooling epilogue stores every pooled row into
    its owner's buffer through CUDA-IPC-mapped peer memory and a per-sender
    epoch flag completes the exchange; world 2 runs two processes on one GPU.
    The result equals EmbeddingBag over all tables for the rank's samples."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    out = mp.Manager().dict()
    mp.spawn(_a2a_worker, args=(world, port, out), nprocs=world, join=True)
    assert all(out[r] for r in range(world))
