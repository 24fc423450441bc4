"""Multi-GPU sharding of planning instances (one process per GPU).

Planning instances are independent, so ranks split them with
no data-path collective; the single real exchange is choosing the global best
plan: every rank contributes one (makespan, xi, instance) record per planned
instance, an all_gather (NCCL over NVLink on the GPU box, gloo on CPU tests)
collects them, and a lexicographic arg-min — smallest makespan, then the
smallest xi (planner.py:76's strict-less rule), then the lowest instance
index — picks the winner.  NCCL has no MINLOC, hence gather + arg-min.
"""

from typing import Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist


def shard(n_items: int, rank: int, world: int) -> Sequence[int]:
    """Round-robin share of instance indices for `rank`."""
    return list(range(rank, n_items, world))


def min_loc(records: np.ndarray) -> Tuple[float, int, int]:
    """Lexicographic arg-min over rows (makespan, xi, instance)."""
    r = np.asarray(records, dtype=np.float64).reshape(-1, 3)
    k = np.lexsort((r[:, 2], r[:, 1], r[:, 0]))[0]
    return float(r[k, 0]), int(r[k, 1]), int(r[k, 2])


def global_best(makespan, xi, instance, device=None) -> Tuple[float, int, int]:
    """All-gather the per-instance records of every rank and return the global min-loc.

    All ranks must pass the same number of records (weak-scaling shards)."""
    rec = np.stack([np.asarray(makespan, np.float64), np.asarray(xi, np.float64),
                    np.asarray(instance, np.float64)], axis=1)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return min_loc(rec)
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" \
            else torch.device("cpu")
    t = torch.from_numpy(rec).to(device)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return min_loc(torch.cat(out).cpu().numpy())
