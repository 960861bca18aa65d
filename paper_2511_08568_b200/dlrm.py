"""DLRM embedding stage across GPUs (config 4): table-sharded
buffers and pooling, one all-to-all of pooled embeddings per batch.

Rank g owns tables T_g (``shard.assign_tables``), their rows in pinned host
memory, its buffer shard and its slice of the access stream.  For a batch of
B samples, every sample has one bag of P ids per table (the synthetic trace
has no query boundaries, so the bag layout is builder-defined — SPEC.md:104):

1. the local accesses of the batch run through the hot path (models +
   buffer replay, ``HotPath``) and the changed buffer rows are gathered from
   host memory (K5, ``RowStore.refresh``);
2. K6 (``RowStore.pool``) sums each local bag, writing rows in
   (sample, local table) order — which is already peer-major: rank r needs
   samples [r*B/G, (r+1)*B/G), a contiguous block;
3. one ``all_to_all_single`` (NCCL over NVLink; no pack kernel) leaves rank
   r with [B/G, T, D]: every table's pooled row for its samples.

The pooling is injectable (``pool_fn``) so the multi-process host logic is
tested on CPU with gloo (tests/test_dist.py).

``PeerExchange`` is the fused form of steps 2-3 on the GPU: the pooling
kernel's epilogue stores each pooled row directly into its owner's output
over NVLink peer memory (CUDA IPC), so the all-to-all costs no extra pass
over the pooled rows and no collective launch (tests/test_gpu_rows.py runs
it with two processes sharing one GPU).
"""
from __future__ import annotations

import numpy as np

from .trace import table_offsets


def build_bags(trace, tables, batch: int, pooling: int, start: int = 0) -> np.ndarray:
    """[batch, len(tables), pooling] global ids: bag (b, t) = the
    (start+b)-th run of `pooling` consecutive accesses to table t in trace
    order (cyclic when a table's stream is shorter)."""
    off = table_offsets(trace.table_sizes)
    g = np.asarray(trace.gid_array)
    tid = np.searchsorted(off, g, side="right") - 1
    out = np.empty((batch, len(tables), pooling), dtype=np.int64)
    for j, t in enumerate(tables):
        stream = g[tid == t]
        if len(stream) == 0:
            stream = np.array([off[t]], dtype=np.int64)   # a never-accessed table: row 0
        idx = (np.arange(batch)[:, None] + start) * pooling + np.arange(pooling)[None, :]
        out[:, j, :] = stream[idx % len(stream)]
    return out


class DlrmEmbeddingStage:
    def __init__(self, table_sizes, assignment, rank: int, world: int, dim: int, pool_fn,
                 group=None):
        self.table_sizes = list(table_sizes)
        self.assignment = np.asarray(assignment)
        self.rank, self.world, self.dim = rank, world, dim
        self.pool_fn = pool_fn
        self.group = group
        self.local_tables = [t for t in range(len(self.table_sizes)) if self.assignment[t] == rank]
        self.tables_of = [[t for t in range(len(self.table_sizes)) if self.assignment[t] == r]
                          for r in range(world)]

    def forward(self, local_bags):
        """local_bags: [B, T_g, P] ids of this rank's tables (torch, on the
        pooling device).  Returns [B/G, T, D] pooled rows for this rank's
        samples, tables in global order."""
        import torch
        import torch.distributed as dist
        B, Tg, P = local_bags.shape
        G = self.world
        if B % G:
            raise ValueError("batch must split evenly across ranks")
        flat = local_bags.reshape(-1).to(torch.int32)
        offsets = torch.arange(0, B * Tg * P + 1, P, dtype=torch.int64, device=flat.device)
        pooled = self.pool_fn(flat, offsets)                        # [B*Tg, D], peer-major
        send = pooled.reshape(B * Tg * self.dim)
        splits_out = [B // G * len(ts) * self.dim for ts in self.tables_of]
        recv = torch.empty(sum(splits_out), dtype=pooled.dtype, device=pooled.device)
        if G > 1:
            dist.all_to_all_single(recv, send, output_split_sizes=splits_out,
                                   input_split_sizes=[B // G * Tg * self.dim] * G,
                                   group=self.group)
        else:
            recv.copy_(send)
        out = torch.empty((B // G, len(self.table_sizes), self.dim), dtype=pooled.dtype,
                          device=pooled.device)
        pos = 0
        for r, ts in enumerate(self.tables_of):
            n = B // G * len(ts) * self.dim
            if ts:
                out[:, ts, :] = recv[pos:pos + n].reshape(B // G, len(ts), self.dim)
            pos += n
        return out


class _DevPtrArray:
    """A raw device allocation seen by torch (__cuda_array_interface__)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": shape,
                                         "typestr": typestr, "version": 3}


class PeerExchange:
    """K7 fused: pooling whose epilogue IS the all-to-all (SURVEY.md §8(e),
    config 4).  Every rank allocates two output buffers [B/G, T, D] (even /
    odd exchanges) plus a flag array in one dedicated allocation, maps every
    other rank's allocation with CUDA IPC (NVLink P2P inside one B200 node),
    and ``forward`` runs ``recmg_embedding_bag_a2a``: each pooled row is
    stored straight into its owner's buffer, then a per-exchange epoch flag
    per sender replaces the collective's completion.  Double buffering keeps
    a peer's next exchange off the buffer this rank is still reading (a
    peer reaches exchange e+2 only after this rank signalled e+1, which is
    stream-ordered after this rank's consumers of e).

    Handles are exchanged once with ``all_gather_object`` (NCCL or gloo), so
    several ranks may even share one GPU (the 2-process GPU test).
    """

    def __init__(self, rowstore, table_sizes, assignment, rank, world, batch, group=None):
        import ctypes
        import torch
        import torch.distributed as dist
        from . import _native
        if batch % world:
            raise ValueError("batch must split evenly across ranks")
        self.rows, self.rank, self.world, self.batch = rowstore, rank, world, batch
        self.T = len(table_sizes)
        self.dim = rowstore.dim
        assignment = np.asarray(assignment)
        self.local_tables = [t for t in range(self.T) if assignment[t] == rank]
        L = _native.lib()
        per = batch // world
        self.out_elems = per * self.T * self.dim
        self.flag_off = (2 * self.out_elems * 4 + 255) // 256 * 256
        total = self.flag_off + 8 * (world + 1)
        p = ctypes.c_void_p()
        _native.check(L.recmg_peer_alloc(total, ctypes.byref(p)), "peer_alloc")
        self.base = p.value
        h = ctypes.create_string_buffer(64)
        _native.check(L.recmg_peer_handle(ctypes.c_void_p(self.base), h), "peer_handle")
        handles = [None] * world
        if world > 1:
            dist.all_gather_object(handles, h.raw, group=group)
        else:
            handles = [h.raw]
        self.peers = []
        for g in range(world):
            if g == rank:
                self.peers.append(self.base)
            else:
                q = ctypes.c_void_p()
                _native.check(L.recmg_peer_open(handles[g], ctypes.byref(q)), "peer_open")
                self.peers.append(q.value)
        self.tglob = torch.tensor(self.local_tables, dtype=torch.int32, device="cuda")
        self.flag_ptrs = torch.tensor([q + self.flag_off for q in self.peers], dtype=torch.int64,
                                      device="cuda")
        self.out_ptrs = [torch.tensor([q + b * self.out_elems * 4 for q in self.peers],
                                      dtype=torch.int64, device="cuda") for b in range(2)]
        self.epoch = 0
        if world > 1:
            dist.barrier(group=group)

    def output(self, parity):
        import torch
        arr = _DevPtrArray(self.base + parity * self.out_elems * 4,
                           (self.batch // self.world, self.T, self.dim), "<f4")
        return torch.as_tensor(arr, device="cuda")

    def forward(self, local_bags):
        """local_bags: [B, T_g, P] ids of this rank's tables (device).  Returns
        [B/G, T, D] pooled rows for this rank's samples (valid until the
        exchange after next)."""
        import ctypes
        import torch
        from . import _native
        B, Tg, P = local_bags.shape
        if B != self.batch or Tg != len(self.local_tables):
            raise ValueError("bags do not match the exchange's batch / tables")
        self.epoch += 1
        parity = self.epoch & 1
        flat = local_bags.reshape(-1).to(torch.int32).contiguous()
        offsets = torch.arange(0, B * Tg * P + 1, P, dtype=torch.int64, device=flat.device)
        rs = self.rows
        _native.check(_native.lib().recmg_embedding_bag_a2a(
            ctypes.byref(rs.replay.cfg), _native.ptr(rs.replay.state), _native.ptr(flat),
            _native.ptr(offsets), B * Tg, _native.ptr(rs.buf),
            ctypes.c_void_p(rs.host.data_ptr()), self.dim, B, self.world, self.rank, self.T,
            _native.ptr(self.tglob), _native.ptr(self.out_ptrs[parity]),
            _native.ptr(self.flag_ptrs), ctypes.c_void_p(self.base + self.flag_off),
            self.epoch, _native.ptr(rs.src), _native.stream_handle(torch)), "embedding_bag_a2a")
        return self.output(parity)

    def close(self):
        import ctypes
        from . import _native
        L = _native.lib()
        for g, q in enumerate(self.peers):
            if g != self.rank:
                L.recmg_peer_close(ctypes.c_void_p(q))
        L.recmg_peer_free(ctypes.c_void_p(self.base))
        self.peers = []
