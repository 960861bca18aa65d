"""Cache simulators (cache_sim.py of the reference): the LRU comparator on
the GPU (K4: recmg_simulate, set = gid % set_count, cache_sim.py:92-106).

LFU / SRRIP / optgen (cache_sim.py:109-220) are SURVEY.md §8(f) "next"
items and are not on the GPU path yet: asking for them raises.
"""
from __future__ import annotations

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


def simulate(trace, cfg: CacheConfig, per_access: bool = True) -> SimResult:
    """cache_sim.py:223-260 for Policy.LRU, on the GPU."""
    cfg.validate()
    if cfg.policy != Policy.LRU:
        raise NotImplementedError(f"{cfg.policy.value} is not on the GPU path yet "
                                  "(SURVEY.md §8(f) next #3/#4)")
    from .engine import LruSim, to_device_gids
    torch = _native.torch_cuda()
    gids = _gids_of(trace)
    if len(gids) == 0:
        return SimResult(0, 0, [])
    total_ids = int(gids.max()) + 1
    if hasattr(trace, "total_ids"):
        total_ids = max(total_ids, int(trace.total_ids))
    sim = LruSim(cfg.capacity, total_ids, cfg.ways, len(gids))
    pa = torch.empty(len(gids), dtype=torch.uint8, device="cuda") if per_access else None
    sim.run(to_device_gids(torch, gids), pa)
    hits, misses = sim.result()
    return SimResult(hits, misses, pa.cpu().numpy().tolist() if per_access else [])
