"""Multi-GPU sharding of planning work (one process per GPU).

Planning instances, and the candidate plans of one instance, are independent,
so ranks split them with no data-path collective:

* ``shard(n, rank, world)`` — round-robin share of n items (C4's 4096
  instances, C5's xi = 1..256 candidate plans); shards differ in size by at
  most one and are empty when n < world.

The single real exchange is choosing the global best: every rank contributes
one (makespan, xi, instance) record per item it planned, the records are
all-gathered (NCCL over NVLink on the GPU box, gloo in the CPU tests) and a
lexicographic arg-min — smallest makespan, then smallest xi (the strict-less
rule of planner.py:76 that keeps the first, i.e. smallest, xi), then the
lowest instance index — picks the winner.  NCCL has no MINLOC, hence
gather + arg-min.  Uneven shards are handled by gathering the per-rank counts
first and padding every rank's block to the largest count with +inf rows,
which can never win the arg-min.
"""

import math
from typing import Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist

PAD = math.inf


def shard(n_items: int, rank: int, world: int) -> Sequence[int]:
    """Round-robin share of item indices for `rank` (possibly empty)."""
    return list(range(rank, n_items, world))


def min_loc(records: np.ndarray) -> Optional[Tuple[float, int, int]]:
    """Lexicographic arg-min over rows (makespan, xi, instance); None if empty."""
    r = np.asarray(records, dtype=np.float64).reshape(-1, 3)
    r = r[np.isfinite(r[:, 2])]          # drop padding rows (instance = +inf)
    if len(r) == 0:
        return None
    k = np.lexsort((r[:, 2], r[:, 1], r[:, 0]))[0]
    return float(r[k, 0]), int(r[k, 1]), int(r[k, 2])


def _device_for_backend(device):
    if device is not None:
        return device
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def global_best(makespan, xi, instance, device=None) -> Optional[Tuple[float, int, int]]:
    """All-gather every rank's (makespan, xi, instance) records and return the
    global min-loc.  Ranks may hold different numbers of records (including
    none); returns None only when no rank has any."""
    rec = np.stack([np.asarray(makespan, np.float64).reshape(-1), np.asarray(xi, np.float64).reshape(-1),
                    np.asarray(instance, np.float64).reshape(-1)], axis=1) if len(instance) else np.zeros((0, 3))
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return min_loc(rec)
    device = _device_for_backend(device)
    world = dist.get_world_size()
    cnt = torch.tensor([len(rec)], dtype=torch.int64, device=device)
    counts = [torch.empty_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt)
    cap = max(int(c.item()) for c in counts)
    if cap == 0:
        return None
    padded = np.full((cap, 3), PAD)
    padded[:len(rec)] = rec
    t = torch.from_numpy(padded).to(device)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return min_loc(torch.cat(out).cpu().numpy())
