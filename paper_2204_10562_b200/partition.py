"""Workload-minimizing partition and replication (reference partition.py:30-177).

PartitionSolver keeps the reference's interface and error behaviour; the
whole W(l, xi, r, i) table is computed once on the GPU by the wavefront
kernels of csrc/prm.cu (pp_prm) and every solve()/best_partition() reads it.
Realizing fragments are re-derived on device with the reference's
first-found tie rule (partition.py:126-141).
"""

import math
from dataclasses import dataclass
from typing import Dict, Optional, Sequence, Tuple

import numpy as np

from . import _device, _lib
from .model import ClusterGraph, ModelProfile, Plan, Stage, ValidationError, check_numeric_range
from .ordering import DeviceOrdering

INF = math.inf

Fragment = Tuple[int, int, Tuple[int, ...]]


@dataclass(frozen=True)
class PrmResult:
    """One DP state's value and, when feasible, its stage fragments."""
    workload: float
    stages: Optional[Tuple[Fragment, ...]]

    @property
    def feasible(self) -> bool:
        return self.stages is not None


def sum_flags() -> int:
    """CPython >= 3.12 sums floats with Neumaier compensation; earlier ones naively."""
    import sys
    return 0 if sys.version_info >= (3, 12) else _lib.PP_SUM_NAIVE


class PartitionSolver:
    """W over one profile, cluster and device order, solved on the GPU."""

    def __init__(self, profile: ModelProfile, cluster: ClusterGraph, ordering: DeviceOrdering,
                 microbatch_count: int, allow_replication: bool = True):
        if microbatch_count < 1:
            raise ValidationError("microbatch count must be positive")
        self.profile = profile
        self.cluster = cluster
        self.devices = tuple(ordering.order)
        self.microbatches = microbatch_count
        self.allow_replication = allow_replication
        self._db = None
        self._host = None
        self._memo: Dict[Tuple[int, int, int, int], PrmResult] = {}

    # -- device state ------------------------------------------------------------
    def _ensure(self):
        if self._db is not None:
            return
        check_numeric_range(self.profile, self.cluster)
        packed = _device.pack(self.profile, self.cluster)
        pos = {g: k for k, g in enumerate(packed.ids)}
        if sorted(self.devices) != list(packed.ids):
            raise ValidationError("ordering must be a permutation of the cluster's GPUs")
        order = np.array([pos[g] for g in self.devices], dtype=np.int32)
        flags = _lib.PP_GIVEN_ORDER | sum_flags() | (_lib.PP_ALLOW_REPLICATION if self.allow_replication else 0)
        self._db = _device.DeviceBatch([(packed, int(self.microbatches), flags, order)], capture_events=False)
        self._db.run("prm")
        self._host = self._db.fetch()

    def _frags(self, rows) -> Tuple[Fragment, ...]:
        return tuple((int(ls), int(le), self.devices[int(lo) - 1:int(hi)]) for ls, le, lo, hi in rows)

    # -- API ---------------------------------------------------------------------
    def solve(self, num_layers: int, num_stages: int, last_width: int, num_devices: int) -> PrmResult:
        """W(l, xi, r, i) with the realizing fragments when finite (partition.py:95-111)."""
        return self.solve_many([(num_layers, num_stages, last_width, num_devices)])[0]

    def solve_many(self, cells: Sequence[Tuple[int, int, int, int]]):
        """Batched solve(): one device query for every in-range cell."""
        out = [None] * len(cells)
        todo = []
        L, V = self.profile.num_layers, len(self.devices)
        for k, (l, xi, r, i) in enumerate(cells):
            if min(l, xi, r, i) < 1:
                raise ValidationError("all DP arguments must be positive")
            if l > L or i > V:
                raise ValidationError("DP arguments exceed the instance size")
            if not self.allow_replication and r != 1:
                out[k] = PrmResult(INF, None)
                continue
            key = (l, xi, r, i)
            got = self._memo.get(key)
            if got is not None:
                out[k] = got
                continue
            if l < xi or i < xi:
                out[k] = PrmResult(INF, None)
            elif xi != 1 and r > i:
                # the reference's stage loop calls _sync on devices[i-r:i] before
                # finding no widths (partition.py:126-129); an empty slice raises
                if not self.devices[i - r:i]:
                    raise ValidationError("empty device set")
                out[k] = PrmResult(INF, None)
            elif r > i or (xi == 1) != (r == i):
                out[k] = PrmResult(INF, None)
            else:
                todo.append(k)
        if todo:
            self._ensure()
            q = [(0,) + tuple(cells[k]) for k in todo]
            max_xi = max(cells[k][1] for k in todo)
            w, frag, feas = self._db.query(q, max_xi)
            for t, k in enumerate(todo):
                xi = cells[k][1]
                res = PrmResult(float(w[t]), self._frags(frag[t, :xi]) if feas[t] else None)
                self._memo[tuple(cells[k])] = res
                out[k] = res
        for k, res in enumerate(out):
            self._memo.setdefault(tuple(cells[k]), res)
        return out

    def best_partition(self, num_stages: int) -> Tuple[float, Optional[Plan]]:
        """Best W over last-stage widths for a fixed stage count (partition.py:144-162)."""
        V = len(self.devices)
        if not 1 <= num_stages <= V:
            raise ValidationError("stage count must be in 1..V")
        self._ensure()
        h = self._host
        xi = num_stages
        r = int(h["sweep_r"][xi - 1])
        if r == 0:
            return INF, None
        base = xi * (xi - 1) // 2
        rows = zip(h["ls"][base:base + xi], h["le"][base:base + xi], h["dlo"][base:base + xi],
                   h["dhi"][base:base + xi])
        stages = tuple(Stage(index=n + 1, layer_start=a, layer_end=b, devices=d)
                       for n, (a, b, d) in enumerate(self._frags(rows)))
        return float(h["sweep_w"][xi - 1]), Plan(stages=stages, microbatch_count=self.microbatches)


def prm(profile: ModelProfile, cluster: ClusterGraph, ordering: DeviceOrdering, microbatch_count: int,
        num_layers: int, num_stages: int, last_width: int, num_devices: int) -> PrmResult:
    """One-shot W(l, xi, r, i) evaluation (partition.py:165-170)."""
    return PartitionSolver(profile, cluster, ordering, microbatch_count).solve(
        num_layers, num_stages, last_width, num_devices)


def best_partition(profile: ModelProfile, cluster: ClusterGraph, ordering: DeviceOrdering,
                   microbatch_count: int, num_stages: int) -> Tuple[float, Optional[Plan]]:
    """partition.py:173-177."""
    return PartitionSolver(profile, cluster, ordering, microbatch_count).best_partition(num_stages)
