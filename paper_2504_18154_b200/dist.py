"""Cross-rank plumbing of the multi-GPU runs (one process per GPU, torchrun).

PaDG instances share no data-path state (no KV transmission between
instances), so the only collectives are the timing barrier and the reduction of
per-rank measurements: times are max-reduced, work is sum-reduced.
"""
from __future__ import annotations

from typing import Sequence, Tuple

import torch
import torch.distributed as dist


def reduce_max_sum(values: Sequence[float], device=None) -> Tuple[list, list]:
    """Returns (elementwise max over ranks, elementwise sum over ranks)."""
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return t.tolist(), t.tolist()
    mx, sm = t.clone(), t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return mx.tolist(), sm.tolist()


def shard_requests(n_total: int, rank: int, world: int) -> range:
    """Weak scaling: rank r owns request ids r, r+world, ... (disjoint, covering)."""
    return range(rank, n_total, world)
