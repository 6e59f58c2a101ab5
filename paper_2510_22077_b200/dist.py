"""Process-group plumbing for N > 1 (one process per GPU, torch.distributed).

bench.py runs ONE problem partitioned over the ranks (strong scaling): the
library (pmns_set_comm) owns the partition -- contiguous primary slabs cut by
sum n_i^2, interfaces with their smallest adjacent primary -- and the halo
exchanges of the Krylov phase (csrc/dist.inc).  This module holds only the
host-side plumbing: rank/world discovery and the device-time reduction (max
over ranks).  No arithmetic of the method lives here.
"""
from __future__ import annotations

import os


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
