"""End-to-end planner (reference planner.py:30-123) on the GPU.

spp() = validate on the host, then ONE device pipeline (pp_spp): RDO ordering,
DP tables, the wavefront DP, per-xi backtrack, a batched PE simulation of
every feasible xi plan, selection and a replay of the chosen plan with event
capture.  spp_many() runs that pipeline for a whole batch of instances in
one launch sequence (every kernel's grid carries the instance dimension).
"""

import math
import sys
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _device, _lib
from .model import (ClusterGraph, ModelProfile, Plan, Schedule, Stage, check_numeric_range, validate_cluster,
                    validate_profile)
from .partition import sum_flags
from .scheduler import _build_schedule


@dataclass(frozen=True)
class SweepEntry:
    """One stage count's outcome: workload, simulated makespan, bound."""
    stage_count: int
    feasible: bool
    workload: float
    makespan: Optional[float]
    bound: Optional[float]


@dataclass(frozen=True)
class SppResult:
    """The selected plan with its schedule and the full sweep table."""
    plan: Plan
    schedule: Schedule
    makespan: float
    sweep: Tuple[SweepEntry, ...]
    device_order: Tuple[int, ...]
    theorem_factor: float
    phi: float


def bound_factor(num_gpus: int, microbatch_count: int) -> float:
    """Approximation factor (2 + (4V-4)/M) of the end-to-end guarantee (planner.py:52-54)."""
    return 2.0 + (4.0 * num_gpus - 4.0) / microbatch_count


def _items(instances):
    """Validate and pack every instance.  Within one call the same profile /
    cluster OBJECT (e.g. one cluster planned for several models or M values)
    is validated and packed once; objects are not cached across calls (their
    bandwidth dict is mutable)."""
    items, packs = [], []
    seen_p, seen_c, seen_pc = {}, {}, {}
    flags = _lib.PP_ALLOW_REPLICATION | sum_flags()
    for profile, cluster, M in instances:
        if id(profile) not in seen_p:
            validate_profile(profile)
            seen_p[id(profile)] = profile
        if id(cluster) not in seen_c:
            validate_cluster(cluster)
            seen_c[id(cluster)] = cluster
        key = (id(profile), id(cluster))
        p = seen_pc.get(key)
        if p is None:
            check_numeric_range(profile, cluster)
            p = _device.pack(profile, cluster)
            seen_pc[key] = p
        if M < 1:
            from .model import ValidationError
            raise ValidationError("microbatch count must be positive")
        packs.append(p)
        items.append((p, int(M), flags, None))
    return items, packs


def _decode(db: _device.DeviceBatch, h, k: int, M: int, packed) -> SppResult:
    I = db.inst_host[k]
    V = I.V
    ids = packed.ids
    order = tuple(ids[int(x)] for x in h["order"][I.order_off:I.order_off + V])
    so = I.sweep_off
    sweep = []
    for xi in range(1, V + 1):
        r = int(h["sweep_r"][so + xi - 1])
        if r == 0:
            sweep.append(SweepEntry(stage_count=xi, feasible=False, workload=math.inf, makespan=None, bound=None))
        else:
            sweep.append(SweepEntry(stage_count=xi, feasible=True, workload=float(h["sweep_w"][so + xi - 1]),
                                    makespan=float(h["sweep_mk"][so + xi - 1]),
                                    bound=float(h["sweep_bound"][so + xi - 1])))
    xi = int(h["best_xi"][k])
    base = I.stage_off + xi * (xi - 1) // 2
    stages = tuple(Stage(index=n + 1, layer_start=int(h["ls"][base + n]), layer_end=int(h["le"][base + n]),
                         devices=order[int(h["dlo"][base + n]) - 1:int(h["dhi"][base + n])])
                   for n in range(xi))
    plan = Plan(stages=stages, microbatch_count=M)
    J = 4 * xi - 3
    rec = dict(makespan=float(h["best_mk"][k]),
               ev_start=h["ev_start"][I.ev_off:I.ev_off + M * J], ev_end=h["ev_end"][I.ev_off:I.ev_off + M * J],
               ar_start=h["ar_start"][I.ar_off:I.ar_off + xi], ar_end=h["ar_end"][I.ar_off:I.ar_off + xi])
    schedule = _build_schedule(plan, rec)
    p = float(h["phi"][k])
    return SppResult(plan=plan, schedule=schedule, makespan=float(h["best_mk"][k]), sweep=tuple(sweep),
                     device_order=order, theorem_factor=bound_factor(V, M) * (1.0 + p), phi=p)


def spp_many(instances: Sequence[Tuple[ModelProfile, ClusterGraph, int]]) -> List[SppResult]:
    """spp() for a batch of (profile, cluster, M) instances in one device pipeline."""
    items, packs = _items(instances)
    db = _device.DeviceBatch(items, capture_events=True)
    db.run("spp")
    h = db.fetch()
    return [_decode(db, h, k, items[k][1], packs[k]) for k in range(len(items))]


def spp(profile: ModelProfile, cluster: ClusterGraph, microbatch_count: int) -> SppResult:
    """Plan, simulate, and select over all stage counts 1..V (planner.py:57-88)."""
    return spp_many([(profile, cluster, microbatch_count)])[0]


def phi(profile: ModelProfile, cluster: ClusterGraph) -> float:
    """Bandwidth-heterogeneity penalty (cost.py:131-142), evaluated on the GPU."""
    check_numeric_range(profile, cluster)
    db = _device.DeviceBatch([(_device.pack(profile, cluster), 1, sum_flags(), None)], capture_events=False)
    db.run("phi")
    return float(db.fetch()["phi"][0])


@dataclass(frozen=True)
class BoundReport:
    """Achieved makespan against the guaranteed factor over a reference."""
    factor: float
    phi: float
    makespan: float
    reference: Optional[float]
    ratio: Optional[float]
    within_bound: Optional[bool]


def theorem1_report(profile: ModelProfile, cluster: ClusterGraph, microbatch_count: int, makespan: float,
                    reference: Optional[float] = None) -> BoundReport:
    """planner.py:102-123 (phi from the GPU; the rest is scalar bookkeeping)."""
    p = phi(profile, cluster)
    factor = bound_factor(cluster.num_gpus, microbatch_count) * (1.0 + p)
    if reference is None:
        return BoundReport(factor=factor, phi=p, makespan=makespan, reference=None, ratio=None, within_bound=None)
    if reference == 0.0:
        return BoundReport(factor=factor, phi=p, makespan=makespan, reference=reference, ratio=None,
                           within_bound=makespan == 0.0)
    ratio = makespan / reference
    return BoundReport(factor=factor, phi=p, makespan=makespan, reference=reference, ratio=ratio,
                       within_bound=ratio <= factor * (1.0 + 1e-9))
