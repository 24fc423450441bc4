"""End-to-end planner (reference planner.py:30-123) on the GPU.

spp() = validate on the host, then ONE device pipeline (pp_spp): RDO ordering,
DP tables, the wavefront DP, per-xi backtrack, a batched PE simulation of
every feasible xi plan, selection and a replay of the chosen plan with event
capture.  spp_many() runs that pipeline for a whole batch of instances in
one launch sequence (every kernel's grid carries the instance dimension).
"""

import gc
import math
from collections import abc
import sys
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _device, _lib
from .model import (AllReduceWindow, ClusterGraph, LazyEvents, ModelProfile, Plan, Schedule, Stage,
                    check_cluster_range, check_numeric_range, check_profile_range, validate_cluster,
                    validate_profile)
from .partition import sum_flags
from .scheduler import _labels


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


# Validated + packed profiles across calls.  A ModelProfile is deeply immutable
# (frozen dataclasses in tuples), so the same OBJECT always packs to the same
# arrays; entries are keyed by id and held through a weak reference, so a
# recycled id can never hit a stale entry.  Clusters are NOT cached: their
# bandwidth dict is mutable.
_profile_cache = {}


def _cached_profile(profile):
    ent = _profile_cache.get(id(profile))
    if ent is not None and ent[0]() is profile:
        return ent[1]
    return None


def _cache_profile(profile, packed):
    import weakref
    key = id(profile)
    try:
        ref = weakref.ref(profile, lambda _r, k=key: _profile_cache.pop(k, None))
    except TypeError:   # not weak-referenceable: no caching
        return
    if len(_profile_cache) > 4096:
        _profile_cache.clear()
    _profile_cache[key] = (ref, packed)


def _items(instances):
    """Validate and pack every instance.  Within one call the same profile /
    cluster OBJECT (e.g. one cluster planned for several models or M values)
    is validated and packed once; profiles (immutable) are also remembered
    across calls, clusters (mutable bandwidth dict) are not."""
    gc_on = gc.isenabled()
    gc.disable()   # no reference cycles below; skip the cyclic collector's rescans
    try:
        return _items_loop(instances)
    finally:
        if gc_on:
            gc.enable()


def _items_loop(instances):
    items, packs = [], []
    seen_p, seen_c, seen_pc = {}, {}, {}
    flags = _lib.PP_ALLOW_REPLICATION | sum_flags()
    # all distinct clusters validated and packed in one vectorised pass when every
    # one of them is in the common valid form (else the per-instance path below)
    cl = list({id(c): c for _, c, _ in instances}.values())
    fast = _device.pack_clusters(cl) if len(cl) > 1 else None
    if fast is not None:
        seen_c = {id(c): (c, f) for c, f in zip(cl, fast)}
    for profile, cluster, M in instances:
        # same check order as validate_profile, validate_cluster, check_numeric_range
        pp, cc = seen_p.get(id(profile)), seen_c.get(id(cluster))
        if pp is None:
            hit = _cached_profile(profile)
            if hit is not None:
                pp = seen_p[id(profile)] = (profile, hit)
        if pp is None:
            validate_profile(profile)
        arrays = None
        if cc is None:
            arrays = _device.bandwidth_arrays(cluster) if cluster.bandwidth else None
            validate_cluster(cluster, arrays)
        if pp is None:
            check_profile_range(profile)
            pp = seen_p[id(profile)] = (profile, _device.pack_profile(profile))
            _cache_profile(profile, pp[1])
        if cc is None:
            check_cluster_range(cluster, arrays)
            cc = seen_c[id(cluster)] = (cluster, _device.pack_cluster(cluster, arrays))
        key = (id(profile), id(cluster))
        p = seen_pc.get(key)
        if p is None:
            ids, bw = cc[1]
            p = seen_pc[key] = _device.Packed(ids, *pp[1], bw)
        if M < 1:
            from .model import ValidationError
            raise ValidationError("microbatch count must be positive")
        packs.append(p)
        items.append((p, int(M), flags, None))
    return items, packs


class LazySweep(abc.Sequence):
    """SppResult.sweep backed by the fetched per-xi arrays: behaves like the
    reference's Tuple[SweepEntry, ...] (len, indexing, iteration, ==, hash)
    but builds the SweepEntry objects on first use."""

    __slots__ = ("_r", "_w", "_mk", "_bd", "_tuple")

    def __init__(self, r, w, mk, bd):
        self._r, self._w, self._mk, self._bd = r, w, mk, bd
        self._tuple = None

    def materialize(self):
        if self._tuple is None:
            self._tuple = tuple(
                _frozen(SweepEntry, stage_count=xi, feasible=False, workload=math.inf, makespan=None, bound=None)
                if r == 0 else
                _frozen(SweepEntry, stage_count=xi, feasible=True, workload=w, makespan=mk, bound=bd)
                for xi, (r, w, mk, bd) in enumerate(zip(self._r, self._w, self._mk, self._bd), start=1))
        return self._tuple

    def __len__(self):
        return len(self._r)

    def __getitem__(self, k):
        return self.materialize()[k]

    def __iter__(self):
        return iter(self.materialize())

    def __eq__(self, other):
        if isinstance(other, LazySweep):
            return self.materialize() == other.materialize()
        if isinstance(other, (tuple, list)):
            return self.materialize() == tuple(other)
        return NotImplemented

    def __ne__(self, other):
        r = self.__eq__(other)
        return r if r is NotImplemented else not r

    def __hash__(self):
        return hash(self.materialize())

    def __repr__(self):
        return repr(self.materialize())


def _frozen(cls, **fields):
    """Build a frozen dataclass instance without its per-field __setattr__
    guard (same fields, so equality / hashing / repr are unchanged)."""
    obj = object.__new__(cls)
    obj.__dict__.update(fields)
    return obj


def _decode(db: _device.DeviceBatch, h, k: int, M: int, packed) -> SppResult:
    """One instance's SppResult (see _decode_all)."""
    return _decode_all(db, h, [M if q == k else 0 for q in range(db.n)], [packed if q == k else None
                                                                        for q in range(db.n)], only=k)[0]


def _decode_all(db: _device.DeviceBatch, h, Ms, packs, only=None) -> List[SppResult]:
    """SppResult objects of a fetched batch.  Everything array-shaped is sliced
    once per batch (the chosen plans' stage rows gathered with one fancy index,
    whole columns converted to Python lists once), then each instance builds
    its frozen result objects without per-field validation."""
    n = db.n
    ks = range(n) if only is None else (only,)
    offs = db.inst_offsets()
    V = offs["V"]
    bx = h["best_xi"].tolist()
    bmk = h["best_mk"].tolist()
    phis = h["phi"].tolist()
    order_all = h["order"].tolist()
    sr, sw = h["sweep_r"].tolist(), h["sweep_w"].tolist()
    smk, sbd = h["sweep_mk"].tolist(), h["sweep_bound"].tolist()
    # the chosen plans' stage rows and allreduce windows, gathered in one pass
    xs = np.maximum(np.asarray(bx, dtype=np.int64), 0)
    cum = np.concatenate(([0], np.cumsum(xs)))
    rel = np.arange(int(cum[-1]), dtype=np.int64) - np.repeat(cum[:-1], xs)
    base = np.repeat(offs["stage"] + xs * (xs - 1) // 2, xs) + rel
    ls, le = h["ls"][base].tolist(), h["le"][base].tolist()
    dlo, dhi = h["dlo"][base].tolist(), h["dhi"][base].tolist()
    arb = np.repeat(offs["ar"], xs) + rel
    ars, are = h["ar_start"][arb].tolist(), h["ar_end"][arb].tolist()
    coff = h["ev_coff"]
    ev_s, ev_e, ev_o = h["ev_start"], h["ev_end"], h["ev_order"]
    # the objects built below hold no reference cycles: keep the cyclic collector from
    # rescanning every live object each few hundred allocations (C4: 57 k objects per call)
    gc_on = gc.isenabled()
    gc.disable()
    try:
        return _decode_loop(ks, V, Ms, packs, offs, order_all, sr, sw, smk, sbd, bx, cum, ls, le, dlo, dhi, ars, are,
                            bmk, coff, ev_s, ev_e, ev_o, phis)
    finally:
        if gc_on:
            gc.enable()


def _decode_loop(ks, V, Ms, packs, offs, order_all, sr, sw, smk, sbd, bx, cum, ls, le, dlo, dhi, ars, are, bmk,
                 coff, ev_s, ev_e, ev_o, phis):
    out = []
    for k in ks:
        Vk, M, packed = int(V[k]), Ms[k], packs[k]
        ids = packed.ids
        oo, so = int(offs["order"][k]), int(offs["sweep"][k])
        order = tuple([ids[x] for x in order_all[oo:oo + Vk]])
        sweep = LazySweep(sr[so:so + Vk], sw[so:so + Vk], smk[so:so + Vk], sbd[so:so + Vk])
        xi, c0 = bx[k], int(cum[k])
        stages = tuple([_frozen(Stage, index=q + 1, layer_start=ls[c0 + q], layer_end=le[c0 + q],
                                devices=order[dlo[c0 + q] - 1:dhi[c0 + q]]) for q in range(xi)])
        plan = _frozen(Plan, stages=stages, microbatch_count=M)
        mk = bmk[k]
        cnt = M * (4 * xi - 3)
        eo = int(coff[k])
        res, lab, _ = _labels(xi)
        events = LazyEvents.from_order(res, lab, 4 * xi - 3, ev_o[eo:eo + cnt], ev_s[eo:eo + cnt], ev_e[eo:eo + cnt])
        windows = tuple([_frozen(AllReduceWindow, stage=q + 1, start=ars[c0 + q], end=are[c0 + q])
                         for q in range(xi) if dhi[c0 + q] > dlo[c0 + q]])
        schedule = _frozen(Schedule, events=events, allreduce=windows, makespan=mk)
        p = phis[k]
        out.append(_frozen(SppResult, plan=plan, schedule=schedule, makespan=mk, sweep=sweep,
                           device_order=order, theorem_factor=bound_factor(Vk, M) * (1.0 + p), phi=p))
    return out


def spp_many(instances: Sequence[Tuple[ModelProfile, ClusterGraph, int]]) -> List[SppResult]:
    """spp() for a batch of (profile, cluster, M) instances in one device pipeline."""
    items, packs = _items(instances)
    db = _device.DeviceBatch(items, capture_events=True)
    db.run("spp")
    h = db.fetch()
    return _decode_all(db, h, [it[1] for it in items], packs)


def spp(profile: ModelProfile, cluster: ClusterGraph, microbatch_count: int) -> SppResult:
    """Plan, simulate, and select over all stage counts 1..V (planner.py:57-88)."""
    return spp_many([(profile, cluster, microbatch_count)])[0]


def phi(profile: ModelProfile, cluster: ClusterGraph) -> float:
    """Bandwidth-heterogeneity penalty (cost.py:131-142), evaluated on the GPU."""
    check_numeric_range(profile, cluster)
    db = _device.DeviceBatch([(_device.pack(profile, cluster), 1, sum_flags(), None)], capture_events=False,
                             workspace=False)
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
