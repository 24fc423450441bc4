"""Baseline planners on the same device pipeline (reference baselines.py:28-97;
SURVEY.md §8f item f3).

- gpipe_plan: even layer split, one ordered device per stage — host bookkeeping;
- gpipe_schedule: the flush discipline, run by the generic-queue simulation
  kernel (k_sim_plans, PP_SIM_FORWARD_BARRIER) with every resource queue
  holding its forward-side blocks for m = 1..M, then its backward-side blocks;
- dataparallel_plan: one stage over every GPU — host bookkeeping;
- noreplication_plan: ONE pp_prm run with replication disabled; the best
  stage count is the first minimum of the device-side sweep (the reference's
  strict ``best > w`` scan over xi = 1..V).
"""

import math
from itertools import accumulate
from typing import Dict, List, Optional, Tuple

import numpy as np

from .model import ClusterGraph, ModelProfile, Plan, Schedule, Stage, ValidationError
from .ordering import DeviceOrdering
from .partition import PartitionSolver
from .scheduler import build_block_list, simulate_with_order


def gpipe_plan(profile: ModelProfile, cluster: ClusterGraph, ordering: DeviceOrdering, stage_count: int,
               microbatch_count: int) -> Plan:
    """Layer counts differ by at most one, longer stages first; stage n on
    ordering.order[n] (baselines.py:28-49, same error text)."""
    hi = min(profile.num_layers, cluster.num_gpus)
    if stage_count < 1 or stage_count > hi:
        raise ValidationError(f"infeasible stage count {stage_count}: must be in 1..{hi}")
    q, rem = divmod(profile.num_layers, stage_count)
    ends = list(accumulate(q + (n < rem) for n in range(stage_count)))
    starts = [1] + [e + 1 for e in ends[:-1]]
    return Plan(stages=tuple(Stage(index=n + 1, layer_start=starts[n], layer_end=ends[n],
                                   devices=(ordering.order[n],)) for n in range(stage_count)),
                microbatch_count=microbatch_count)


def gpipe_queues(plan: Plan) -> Dict[str, Tuple[Tuple[int, int], ...]]:
    """Per-resource flush queues: blocks in block-list order, each for m = 1..M."""
    ms = range(1, plan.microbatch_count + 1)
    grouped: Dict[str, List[Tuple[int, int]]] = {}
    for blk in build_block_list(plan):
        grouped.setdefault(blk.resource, []).extend((m, blk.position) for m in ms)
    return {res: tuple(items) for res, items in grouped.items()}


def gpipe_schedule(plan: Plan, profile: ModelProfile, cluster: ClusterGraph) -> Schedule:
    """Barrier schedule of an unreplicated plan on the GPU (baselines.py:52-69)."""
    if any(s.replicated for s in plan.stages):
        raise ValidationError("barrier baseline does not support replicated stages")
    return simulate_with_order(plan, profile, cluster, gpipe_queues(plan), forward_barrier=True)


def dataparallel_plan(profile: ModelProfile, cluster: ClusterGraph, microbatch_count: int) -> Plan:
    """All layers as one stage over every GPU, ids ascending (baselines.py:72-77)."""
    return Plan(stages=(Stage(1, 1, profile.num_layers, tuple(sorted(cluster.gpu_ids))),),
                microbatch_count=microbatch_count)


def noreplication_plan(profile: ModelProfile, cluster: ClusterGraph, ordering: DeviceOrdering,
                       microbatch_count: int) -> Tuple[float, Optional[Plan]]:
    """Workload-optimal single-device-per-stage plan, or (inf, None) when no
    stage count is feasible (baselines.py:80-97)."""
    solver = PartitionSolver(profile, cluster, ordering, microbatch_count, allow_replication=False)
    solver._ensure()
    feasible = np.asarray(solver._host["sweep_r"][:cluster.num_gpus]) != 0
    w = np.where(feasible, np.asarray(solver._host["sweep_w"][:cluster.num_gpus], np.float64), math.inf)
    xi = int(np.argmin(w)) + 1  # first minimum == the strict best > w scan
    if not math.isfinite(w[xi - 1]):
        return math.inf, None
    return solver.best_partition(xi)
