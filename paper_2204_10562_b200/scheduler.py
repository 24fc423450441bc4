"""Microbatch scheduling and makespan simulation (reference scheduler.py:45-238).

simulate_pe / simulate_with_order / lemma1_bound run on the GPU (csrc/sim.cu):
the PE order as a closed-form pass sweep with one thread per resource, any
caller queue order as a round-based dependency sweep with forward-barrier
and stall detection.  build_block_list / compute_execution_order build the
reference's Python structures from their closed forms.
"""

import functools
from dataclasses import dataclass
from typing import Dict, List, Sequence, Tuple

import numpy as np

from . import _device, _lib
from .model import (BWD, COMM_BWD, COMM_FWD, FWD, FWDBWD, AllReduceWindow, Block, ClusterGraph, LazyEvents,
                    ModelProfile, Plan, Schedule, ValidationError, check_numeric_range)
from .partition import sum_flags


class SchedulingError(RuntimeError):
    """The simulation stalled with work left (circular waiting)."""


def build_block_list(plan: Plan) -> Tuple[Block, ...]:
    """The ordered block list J for a plan (scheduler.py:49-66)."""
    N = plan.num_stages
    if N == 1:
        return (Block(position=1, kind=FWDBWD, stage=1),)
    out: List[Block] = []
    for n in range(1, N):
        out.append(Block(position=2 * n - 1, kind=FWD, stage=n))
        out.append(Block(position=2 * n, kind=COMM_FWD, channel=n))
    out.append(Block(position=2 * N - 1, kind=FWDBWD, stage=N))
    for n in range(N - 1, 0, -1):
        out.append(Block(position=4 * N - 2 - 2 * n, kind=COMM_BWD, channel=n))
        out.append(Block(position=4 * N - 1 - 2 * n, kind=BWD, stage=n))
    return tuple(out)


@dataclass(frozen=True)
class ExecutionOrder:
    """Per-resource queues of (microbatch, block position), head first."""
    queues: Dict[str, Tuple[Tuple[int, int], ...]]


def _resources(N: int) -> List[str]:
    return [f"stage{r // 2 + 1}" if r % 2 == 0 else f"chan{r // 2 + 1}" for r in range(2 * N - 1)]


def _lane_positions(N: int):
    """Per resource lane (chain order): positions served, backward side first."""
    out = []
    for r in range(2 * N - 1):
        n = r // 2 + 1
        if r % 2 == 0:
            out.append((4 * N - 1 - 2 * n, 2 * n - 1) if n < N else (2 * N - 1,))
        else:
            out.append((4 * N - 2 - 2 * n, 2 * n))
    return out


def _pe_queue_arrays(N: int, M: int):
    """Closed form of scheduler.py:75-106: pass p serves m = p - pos + 1 at
    every position, positions descending; per lane (m, pos) in queue order."""
    J = 4 * N - 3
    res = []
    for pos_list in _lane_positions(N):
        ps = np.array(sorted(pos_list, reverse=True))
        passes = np.arange(1, M + J)
        m = passes[:, None] - ps[None, :] + 1
        pos = np.broadcast_to(ps, m.shape)
        ok = (m >= 1) & (m <= M)
        res.append(np.stack([m[ok], pos[ok]], axis=1))
    return res


def compute_execution_order(plan: Plan) -> ExecutionOrder:
    """Queue order that keeps late blocks ahead of early ones (scheduler.py:75-106)."""
    N, M = plan.num_stages, plan.microbatch_count
    names = _resources(N)
    arrs = _pe_queue_arrays(N, M)
    order = [r for r in _block_resource_order(N)]
    return ExecutionOrder(queues={names[r]: tuple(map(tuple, arrs[r].tolist())) for r in order})


def _block_resource_order(N: int) -> List[int]:
    """Resource lanes in first-appearance order of the block list (the reference's dict order)."""
    seen, out = set(), []
    for b in range(1, 4 * N - 2):
        r = _pos_lane(N, b)
        if r not in seen:
            seen.add(r)
            out.append(r)
    return out


def _pos_lane(N: int, pos: int) -> int:
    if N == 1:
        return 0
    if pos <= 2 * N - 2:
        n = (pos + 1) // 2
        return 2 * n - 2 if pos % 2 else 2 * n - 1
    if pos == 2 * N - 1:
        return 2 * N - 2
    q = pos - (2 * N - 1)
    n = N - (q + 1) // 2
    return 2 * n - 1 if q % 2 else 2 * n - 2


@functools.lru_cache(maxsize=1024)
def _labels(N: int):
    """position -> (resource, label, resource sort key) (model.py:148-158, scheduler.py:115-118)."""
    res, lab, key = [None] * (4 * N - 2), [None] * (4 * N - 2), np.zeros(4 * N - 2, dtype=np.int64)
    for b in build_block_list(Plan(stages=tuple(range(N)), microbatch_count=1)):
        res[b.position] = b.resource
        lab[b.position] = b.label
        key[b.position] = (b.stage if b.is_compute else (1 << 20) + b.channel)
    return res, lab, key


@functools.lru_cache(maxsize=256)
def _pe_tiebreak_order(N: int, M: int):
    """Permutation of the (m, pos) grid sorted by (resource key, microbatch, position): a
    stable sort by start time on top of it yields the reference's event order.
    Depends on (N, M) only: cached, arrays read-only."""
    J = 4 * N - 3
    _, _, key = _labels(N)
    m = np.repeat(np.arange(1, M + 1, dtype=np.int32), J)
    p = np.tile(np.arange(1, J + 1, dtype=np.int32), M)
    order = np.lexsort((p, m, key[p]))
    out = (order, m[order], p[order])
    for a in out:
        a.setflags(write=False)
    return out


def _check_plan(plan: Plan, profile: ModelProfile, cluster: ClusterGraph) -> None:
    """The structural errors the reference's cost functions raise (cost.py:38-41, 91-95, 112-120)."""
    L = profile.num_layers
    known = set(cluster.gpu_ids)
    if plan.microbatch_count < 1:
        raise ValidationError("microbatch_count must be >= 1")
    if not plan.stages:
        raise ValidationError("plan has no stages")
    for s in plan.stages:
        if not (1 <= s.layer_start <= s.layer_end <= L):
            raise ValidationError(f"invalid layer interval [{s.layer_start},{s.layer_end}] for L={L}")
        if not s.devices:
            raise ValidationError("empty device set")
        for d in s.devices:
            if d not in known:
                raise ValidationError(f"unknown device {d}")
    for a, b in zip(plan.stages, plan.stages[1:]):
        if not (1 <= a.layer_end <= L - 1):
            raise ValidationError(f"boundary layer {a.layer_end} out of range")
        if set(a.devices) & set(b.devices):
            raise ValidationError("overlapping device sets")
    if plan.num_stages > _lib.PP_MAX_GPUS:
        raise ValidationError(f"plans with more than {_lib.PP_MAX_GPUS} stages are outside this build")


def _sim(plan, profile, cluster, queue_lists=None, forward_barrier=False, capture=True, cycle=False):
    check_numeric_range(profile, cluster)
    _check_plan(plan, profile, cluster)
    packed = _device.pack(profile, cluster)
    pos = {g: k for k, g in enumerate(packed.ids)}
    db = _device.DeviceBatch([(packed, plan.microbatch_count, sum_flags(), None)], capture_events=False,
                             workspace=False)
    stages = [(s.layer_start, s.layer_end, [pos[d] for d in s.devices]) for s in plan.stages]
    flags = (_lib.PP_SIM_FORWARD_BARRIER if forward_barrier else 0)
    if cycle:
        flags |= _lib.PP_SIM_CYCLE
    elif queue_lists is None:
        flags |= _lib.PP_SIM_PE_ORDER
    sp = _device.SimPlan(inst=0, M=plan.microbatch_count, stages=stages, flags=flags, queues=queue_lists)
    run = _device.SimRun(db, [sp], capture_events=capture)
    return run.fetch()[0]


def _build_schedule(plan: Plan, rec, tiebreak=None) -> Schedule:
    N, M = plan.num_stages, plan.microbatch_count
    J = 4 * N - 3
    res, lab, key = _labels(N)
    start = rec["ev_start"]
    end = rec["ev_end"]
    # stable order of the reference: (start, resource key, microbatch), ties in queue order
    if tiebreak is None and rec.get("ev_order") is not None:
        # ordered on the device (k_event_order): rank k holds event (m-1)*J + pos-1
        events = LazyEvents.from_order(res, lab, J, rec["ev_order"], start, end)
    elif tiebreak is None:
        # PE queues: same-resource, same-microbatch ties are in position order
        order, mo, po = _pe_tiebreak_order(N, M)
        so = start[order]
        k = np.argsort(so, kind="stable")
        events = LazyEvents(res, lab, mo[k], po[k], so[k], end[order][k])
    else:
        m = np.repeat(np.arange(1, M + 1), J)
        p = np.tile(np.arange(1, J + 1), M)
        idx = np.lexsort((tiebreak, m, key[p], start))
        events = LazyEvents(res, lab, m[idx], p[idx], start[idx], end[idx])
    windows = tuple(AllReduceWindow(stage=s.index, start=float(rec["ar_start"][s.index - 1]),
                                    end=float(rec["ar_end"][s.index - 1]))
                    for s in plan.stages if s.replicated)
    return Schedule(events=events, allreduce=windows, makespan=rec["makespan"])


def simulate_with_order(plan: Plan, profile: ModelProfile, cluster: ClusterGraph,
                        queues: Dict[str, Tuple[Tuple[int, int], ...]],
                        forward_barrier: bool = False) -> Schedule:
    """Play out given per-resource queues (scheduler.py:121-225) on the GPU."""
    N, M = plan.num_stages, plan.microbatch_count
    J = 4 * N - 3
    names = _resources(N)
    lane_of = {nm: r for r, nm in enumerate(names)}
    for res in queues:
        if res not in lane_of:
            raise SchedulingError(f"queue given for unknown resource {res}")
    lists = [list(queues.get(nm, ())) for nm in names]
    seen = set()
    qidx = np.zeros(M * J, dtype=np.int64)
    for r, q in enumerate(lists):
        for k, item in enumerate(q):
            mm, pp = int(item[0]), int(item[1])
            # Malformed queues: the reference looks the
            # position up in its block dict (KeyError, scheduler.py:167) and
            # plays the rest out as given; here they are rejected up front
            # with the reference's simulation error class.
            if not 1 <= pp <= J:
                raise KeyError(pp)
            if not 1 <= mm <= M:
                raise SchedulingError(f"queue item {item} outside microbatches 1..{M}")
            if _pos_lane(N, pp) != r:
                raise SchedulingError(f"queue item {item} is not a block of resource {names[r]}")
            if (mm, pp) in seen:
                raise SchedulingError(f"queue item {item} appears twice")
            seen.add((mm, pp))
            qidx[(mm - 1) * J + pp - 1] = k
    rec = _sim(plan, profile, cluster, lists, forward_barrier)
    if rec["status"] != 0:
        _, lab, _ = _labels(N)
        heads = []
        for r in sorted(range(len(names)), key=lambda r: names[r]):
            h = int(rec["head"][r])
            if h >= 0:
                mm, pp = lists[r][h]
                heads.append(f"{names[r]} head ({mm},{lab[pp]})")
        raise SchedulingError(f"stalled with {M * J - rec['n_done']} executions left; " + "; ".join(heads))
    return _build_schedule(plan, rec, tiebreak=qidx)


def simulate_pe(plan: Plan, profile: ModelProfile, cluster: ClusterGraph) -> Schedule:
    """Simulate the pipeline-efficient queue order (scheduler.py:228-231)."""
    return _build_schedule(plan, _sim(plan, profile, cluster))


def simulate_pe_many(plans: Sequence[Plan], profile: ModelProfile, cluster: ClusterGraph):
    """[(makespan, lemma1_bound)] of simulate_pe for many plans of one instance in ONE launch
    (one CTA per plan; the C5 candidate sweep).  Schedules are not materialised."""
    check_numeric_range(profile, cluster)
    for p in plans:
        _check_plan(p, profile, cluster)
    packed = _device.pack(profile, cluster)
    pos = {g: k for k, g in enumerate(packed.ids)}
    db = _device.DeviceBatch([(packed, max(p.microbatch_count for p in plans), sum_flags(), None)],
                             capture_events=False, workspace=False)
    sps = [_device.SimPlan(inst=0, M=p.microbatch_count,
                           stages=[(s.layer_start, s.layer_end, [pos[d] for d in s.devices]) for s in p.stages],
                           flags=_lib.PP_SIM_PE_ORDER) for p in plans]
    run = _device.SimRun(db, sps, capture_events=False)
    return [(r["makespan"], r["bound"]) for r in run.fetch()]


def simulate_cycle_schedule(plan: Plan, profile: ModelProfile, cluster: ClusterGraph) -> Schedule:
    """Lockstep cycle schedule, M + 4N - 4 cycles (scheduler.py:241-296), on the GPU
    (k_sim_plans, PP_SIM_CYCLE).  Same-start ties sort by (resource, microbatch,
    position) — the reference's stable order, since a resource meets the same
    microbatch again only in a later cycle at a higher position."""
    rec = _sim(plan, profile, cluster, cycle=True)
    s = _build_schedule(plan, rec)
    return Schedule(events=s.events, allreduce=s.allreduce, makespan=s.makespan, cycle_count=rec["cycles"])


def lemma1_bound(plan: Plan, profile: ModelProfile, cluster: ClusterGraph) -> float:
    """(M + 4N - 4) * C + max AllReduce (scheduler.py:234-238), computed on the GPU."""
    return _sim(plan, profile, cluster, capture=False)["bound"]
