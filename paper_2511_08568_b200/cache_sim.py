"""Cache simulators (cache_sim.py of the reference) on the GPU: LRU (the
32-way comparator, K4), LFU, SRRIP and the offline optimum (optgen / Belady
with keep decisions) as policies of the replay engine's shared-memory set
kernel (set = gid % set_count, cache_sim.py:33-35), any capacity: sets of up
to 4096 ways replay in shared memory, wider ones (fully associative at a
realistic capacity) in global memory.
"""
from __future__ import annotations

import csv
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _native
from .errors import InvalidConfigError


class Policy(str, Enum):
    LRU = "lru"
    LFU = "lfu"
    SRRIP = "srrip"
    OPTGEN = "optgen"


@dataclass
class CacheConfig:
    """cache_sim.py:30-58."""
    capacity: int
    policy: Policy = Policy.LRU
    ways: int | None = None
    srrip_max_rrpv: int = 3

    def validate(self):
        if self.capacity < 1:
            raise InvalidConfigError("capacity must be >= 1")
        if self.ways is not None:
            if self.ways < 1 or self.capacity % self.ways != 0:
                raise InvalidConfigError("ways must be >= 1 and divide capacity")
        if self.srrip_max_rrpv < 0:
            raise InvalidConfigError("srrip_max_rrpv must be >= 0")

    @property
    def set_count(self) -> int:
        return 1 if self.ways is None else self.capacity // self.ways

    @property
    def ways_per_set(self) -> int:
        return self.capacity if self.ways is None else self.ways


@dataclass
class SimResult:
    """cache_sim.py:61-71."""
    hits: int
    misses: int
    per_access_hit: list
    keep_decisions: list | None = None

    @property
    def hit_rate(self) -> float:
        total = self.hits + self.misses
        return self.hits / total if total else 0.0


def _gids_of(trace) -> np.ndarray:
    if hasattr(trace, "gid_array"):
        return np.asarray(trace.gid_array)
    return np.asarray(trace, dtype=np.int64)


def _run(trace, capacity, ways, policy, srrip_max_rrpv=3, per_access=True, keep=False):
    from .engine import SetSim, to_device_gids
    torch = _native.torch_cuda()
    gids = _gids_of(trace)
    if len(gids) == 0:
        return SimResult(0, 0, [], [] if keep else None)
    total_ids = int(gids.max()) + 1
    if hasattr(trace, "total_ids"):
        total_ids = max(total_ids, int(trace.total_ids))
    sim = SetSim(capacity, total_ids, ways, len(gids), policy, srrip_max_rrpv)
    pa = torch.empty(len(gids), dtype=torch.uint8, device="cuda") \
        if (per_access or keep) else None
    kd = torch.empty(len(gids), dtype=torch.uint8, device="cuda") if keep else None
    sim.run(to_device_gids(torch, gids), pa, kd)
    hits, misses = sim.result()
    return SimResult(hits, misses, pa.cpu().numpy().tolist() if per_access else [],
                     kd.cpu().numpy().tolist() if keep else None)


def simulate(trace, cfg: CacheConfig, per_access: bool = True) -> SimResult:
    """cache_sim.py:223-260 on the GPU."""
    cfg.validate()
    if cfg.policy == Policy.OPTGEN:
        return _run(trace, cfg.capacity if cfg.set_count > 1 else cfg.ways_per_set,
                    cfg.ways if cfg.set_count > 1 else None, "optgen", per_access=per_access,
                    keep=True)
    return _run(trace, cfg.capacity, cfg.ways, cfg.policy.value, cfg.srrip_max_rrpv,
                per_access=per_access)


def simulate_optgen(trace, capacity: int) -> SimResult:
    """cache_sim.py:199-220: fully associative Belady with keep decisions."""
    if capacity < 1:
        raise InvalidConfigError("capacity must be >= 1")
    return _run(trace, capacity, None, "optgen", keep=True)


def sweep(trace, policies, capacities, ways=None) -> list:
    """cache_sim.py:304-320."""
    rows = []
    for policy in policies:
        for cap in capacities:
            w = ways if ways is not None and policy != Policy.OPTGEN else None
            res = simulate(trace, CacheConfig(capacity=cap, policy=policy, ways=w),
                           per_access=False)
            rows.append({"policy": policy.value, "capacity": cap, "hits": res.hits,
                         "misses": res.misses, "hit_rate": res.hit_rate})
    return rows


def write_sweep_csv(rows: list, path: str):
    """cache_sim.py:323-329."""
    with open(path, "w", encoding="utf-8", newline="") as f:
        w = csv.writer(f)
        w.writerow(["policy", "capacity", "hits", "misses", "hit_rate"])
        for r in rows:
            w.writerow([r["policy"], r["capacity"], r["hits"], r["misses"],
                        f"{r['hit_rate']:.6f}"])


BRUTE_MAX_LEN = 14
BRUTE_MAX_CAP = 4


def brute_force_optimal(trace, capacity: int) -> int:
    """cache_sim.py:263-301: the maximum hit count over every victim choice,
    by exhaustive search -- an independent check of the offline optimum for
    tiny instances (at most 14 accesses, capacity 4), on the host."""
    from functools import lru_cache
    gids = tuple(int(g) for g in _gids_of(trace))
    if len(gids) > BRUTE_MAX_LEN or capacity > BRUTE_MAX_CAP:
        raise InvalidConfigError(
            f"brute force bounded to {BRUTE_MAX_LEN} accesses / capacity {BRUTE_MAX_CAP}")
    if capacity < 1:
        raise InvalidConfigError("capacity must be >= 1")

    @lru_cache(maxsize=None)
    def best(i: int, cached: frozenset) -> int:
        if i == len(gids):
            return 0
        g = gids[i]
        if g in cached:
            return 1 + best(i + 1, cached)
        if len(cached) < capacity:
            return best(i + 1, cached | {g})
        return max(best(i + 1, (cached - {v}) | {g}) for v in cached)

    return best(0, frozenset())
