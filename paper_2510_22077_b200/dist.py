"""Process-group plumbing for N > 1 (one process per GPU, torch.distributed).

Round 1 runs independent replicas of the workload per rank (weak scaling);
this module holds the host-side pieces shared by bench.py and the future slab
decomposition: rank/world discovery, device-time reduction (max over ranks),
and the slab ownership of primaries (primaries owned by the
z-slab containing their centroid, cut planes weighted by local-solve work).
No arithmetic of the method lives here.
"""
from __future__ import annotations

import os

import numpy as np


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device time) over the default process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def slab_owners(centroid_z: np.ndarray, work: np.ndarray, nz: int, world: int) -> np.ndarray:
    """Owner rank of each primary: z-slabs whose cut planes split the total
    local-solve work evenly; a primary belongs to the slab containing its
    centroid.  Deterministic (ties by primary index)."""
    centroid_z = np.asarray(centroid_z, dtype=float)
    work = np.asarray(work, dtype=float)
    if world <= 1 or centroid_z.size == 0:
        return np.zeros(centroid_z.size, dtype=np.int64)
    order = np.lexsort((np.arange(centroid_z.size), centroid_z))
    cum = np.cumsum(work[order])
    total = cum[-1]
    owner_sorted = np.minimum((cum - 0.5 * work[order]) * world // max(total, 1e-300), world - 1).astype(np.int64)
    owner = np.empty_like(owner_sorted)
    owner[order] = owner_sorted
    return owner
