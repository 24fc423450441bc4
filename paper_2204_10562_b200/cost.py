"""Closed-form cost API (reference cost.py:44-230; SURVEY.md §8a a8/a9/a15/a19,
§8f f4) evaluated by the device cost pass.

Every plan-level quantity comes from ONE launch of k_sim_plans in
PP_SIM_COSTS_ONLY mode: lane r of a plan's CTA evaluates the same
``lane_cost`` the simulators use (Neumaier sums, min pairwise / cross
bandwidth, AllReduce, durations) and writes a PP_LANE_COST_FIELDS record;
the CTA also reduces cost_summary's workload and the Lemma-1 bound.  Scalar
helpers (allreduce_time, interstage_comm_time, min_*_bandwidth) are one- or
two-stage plans through the same pass.  Argument checks and their messages
stay on the host, as in the reference.
"""

from dataclasses import dataclass
from typing import Dict, List, Sequence, Tuple

from . import _device, _lib
from .model import (BWD, COMM_FWD, FWD, Block, ClusterGraph, InterLayerEdge, LayerProfile, ModelProfile, Plan,
                    ValidationError, check_numeric_range)
from .partition import sum_flags

# lane record fields (include/pipeplan_b200.h, PP_LANE_COST_FIELDS)
_DA, _DB, _CYC, _AR, _FS, _BS, _MBW = range(7)


@dataclass(frozen=True)
class CostSummary:
    """cost.py:145-159."""
    per_stage_compute: Dict[int, float]
    per_channel_comm: Dict[int, float]
    allreduce: Dict[int, float]
    cycle_time: float
    workload: float
    gamma: float
    phi: float


def _plan_costs(stage_lists, profile: ModelProfile, cluster: ClusterGraph, M: int = 1):
    """Device cost records for plans given as [(ls, le, device ids), ...] lists."""
    check_numeric_range(profile, cluster)
    packed = _device.pack(profile, cluster)
    pos = {g: k for k, g in enumerate(packed.ids)}
    db = _device.DeviceBatch([(packed, M, sum_flags(), None)], capture_events=False, workspace=False)
    sps = [_device.SimPlan(inst=0, M=M, stages=[(a, b, [pos[d] for d in devs]) for a, b, devs in st],
                           flags=_lib.PP_SIM_COSTS_ONLY) for st in stage_lists]
    return _device.SimRun(db, sps, capture_events=False, costs=True).fetch()


def _check_interval(profile: ModelProfile, a: int, b: int) -> None:
    if not (1 <= a <= b <= profile.num_layers):   # cost.py:38-41
        raise ValidationError(f"invalid layer interval [{a},{b}] for L={profile.num_layers}")


def _check_channel(profile, boundary, left, right, cluster) -> None:
    """interstage_comm_time's checks, in its order (cost.py:112-120)."""
    if not (1 <= boundary <= profile.num_layers - 1):
        raise ValidationError(f"boundary layer {boundary} out of range")
    if not left or not right:
        raise ValidationError("empty device set")
    if set(left) & set(right):
        raise ValidationError("overlapping device sets")
    known = set(cluster.gpu_ids)
    for d in list(left) + list(right):
        if d not in known:
            raise ValidationError(f"unknown device {d}")


def _check_replicas(profile, a, b, devices, cluster) -> None:
    """allreduce_time's checks (cost.py:91-95)."""
    _check_interval(profile, a, b)
    if not devices:
        raise ValidationError("empty device set")
    known = set(cluster.gpu_ids)
    for d in devices:
        if d not in known:
            raise ValidationError(f"unknown device {d}")


def _bw_probe_profile() -> ModelProfile:
    """A 2-layer all-zero chain: lets cluster-only queries ride the plan pass."""
    layers = (LayerProfile(1, 0.0, 0.0, 0.0), LayerProfile(2, 0.0, 0.0, 0.0))
    return ModelProfile("bw-probe", 1, layers, (InterLayerEdge(1, 2, 0.0, 0.0),))


def _check_pairs(cluster: ClusterGraph, pairs) -> None:
    # the reference looks each pair up in the bandwidth dict (model.py:72-73)
    for a, b in pairs:
        key = (a, b) if a < b else (b, a)
        if key not in cluster.bandwidth:
            raise KeyError(key)


def min_pairwise_bandwidth(cluster: ClusterGraph, devices: Sequence[int]) -> float:
    """Minimum bandwidth within a device set, +inf below two devices (cost.py:64-71)."""
    devs = list(devices)
    _check_pairs(cluster, ((a, b) for i, a in enumerate(devs) for b in devs[i + 1:]))
    if len(devs) < 2:
        return float("inf")
    rec = _plan_costs([[(1, 1, devs)]], _bw_probe_profile(), cluster)[0]
    return float(rec["lane_cost"][0, _MBW])


def min_cross_bandwidth(cluster: ClusterGraph, left: Sequence[int], right: Sequence[int]) -> float:
    """Minimum bandwidth between two device sets, +inf if either is empty (cost.py:74-80)."""
    left, right = list(left), list(right)
    _check_pairs(cluster, ((a, b) for a in left for b in right))
    if not left or not right:
        return float("inf")
    rec = _plan_costs([[(1, 1, left), (2, 2, right)]], _bw_probe_profile(), cluster)[0]
    return float(rec["lane_cost"][1, _MBW])


def allreduce_time(profile: ModelProfile, layer_start: int, layer_end: int, devices: Sequence[int],
                   cluster: ClusterGraph) -> float:
    """2(k-1)*sum(alpha)/(k*min pairwise bw), 0 for k = 1 (cost.py:83-99)."""
    _check_replicas(profile, layer_start, layer_end, devices, cluster)
    if len(devices) == 1:
        return 0.0
    rec = _plan_costs([[(layer_start, layer_end, list(devices))]], profile, cluster)[0]
    return float(rec["lane_cost"][0, _AR])


def interstage_comm_time(profile: ModelProfile, boundary_layer: int, devices_left: Sequence[int],
                         devices_right: Sequence[int], cluster: ClusterGraph) -> Tuple[float, float]:
    """(c_fwd, c_bwd) = bytes / (r'*r*min cross bw) (cost.py:102-123)."""
    _check_channel(profile, boundary_layer, devices_left, devices_right, cluster)
    b = boundary_layer
    rec = _plan_costs([[(b, b, list(devices_left)), (b + 1, b + 1, list(devices_right))]], profile, cluster)[0]
    lc = rec["lane_cost"][1]
    return float(lc[_DA]), float(lc[_DB])


def _channel_stage_lists(plan: Plan, profile: ModelProfile, cluster: ClusterGraph):
    """Plan stages for the kernel with every channel check done; stage layer
    intervals are pinned to valid one-layer ranges (only the boundary layer and
    the devices enter a channel's cost)."""
    st = plan.stages
    for n in range(1, plan.num_stages):
        _check_channel(profile, st[n - 1].layer_end, st[n - 1].devices, st[n].devices, cluster)
    out = [(s.layer_end, s.layer_end, list(s.devices)) for s in st[:-1]]
    last = profile.num_layers
    out.append((last, last, list(st[-1].devices)))
    return out


def channel_times(plan: Plan, profile: ModelProfile, cluster: ClusterGraph) -> Dict[int, Tuple[float, float]]:
    """(c_fwd, c_bwd) for every channel n = 1..N-1 (cost.py:162-169)."""
    if plan.num_stages < 2:
        return {}
    lc = _plan_costs([_channel_stage_lists(plan, profile, cluster)], profile, cluster)[0]["lane_cost"]
    return {n: (float(lc[2 * n - 1, _DA]), float(lc[2 * n - 1, _DB])) for n in range(1, plan.num_stages)}


def _check_costed_plan(plan: Plan, profile: ModelProfile, cluster: ClusterGraph) -> None:
    for s in plan.stages:
        if s.replication < 1:
            raise ValidationError("replication factor must be >= 1")
        _check_interval(profile, s.layer_start, s.layer_end)
        if s.replicated:
            _check_replicas(profile, s.layer_start, s.layer_end, s.devices, cluster)
    for n in range(1, plan.num_stages):
        a, b = plan.stages[n - 1], plan.stages[n]
        _check_channel(profile, a.layer_end, a.devices, b.devices, cluster)
    known = set(cluster.gpu_ids)
    for s in plan.stages:
        for d in s.devices:
            if d not in known:
                raise ValidationError(f"unknown device {d}")


def _stage_time(profile: ModelProfile, layer_start: int, layer_end: int, k, which: str) -> float:
    """sum(layer times of [layer_start, layer_end]) / k (cost.py:44-61) on the
    device cost pass: a one-stage plan on a k-GPU probe clique whose profile
    keeps only the requested time column (``cyc = sf + sb`` with the other
    sum exactly 0.0, so the record's cycle time IS ``sum / k`` bit for bit)."""
    _check_interval(profile, layer_start, layer_end)
    if k == 0:
        raise ZeroDivisionError("float division by zero")
    kk = abs(int(k))
    keep_f, keep_b = which in ("f", "fb"), which in ("b", "fb")
    layers = tuple(LayerProfile(l.id, l.fwd_time if keep_f else 0.0, l.bwd_time if keep_b else 0.0, 0.0)
                   for l in profile.layers)
    edges = tuple(InterLayerEdge(e.src, e.dst, 0.0, 0.0) for e in profile.edges)
    probe = ModelProfile(profile.name, profile.microbatch_size, layers, edges)
    ids = list(range(1, kk + 1))
    clu = ClusterGraph(gpu_ids=tuple(ids), bandwidth={(a, b): 1.0 for a in ids for b in ids if a < b})
    rec = _plan_costs([[(layer_start, layer_end, ids)]], probe, clu)[0]
    v = float(rec["lane_cost"][0, _CYC])
    return -v if k < 0 else v   # x / (-k) == -(x / k) in IEEE round-to-nearest


def stage_fwd_time(profile: ModelProfile, layer_start: int, layer_end: int, k: int) -> float:
    """Per-microbatch forward time of a stage on k replicas (cost.py:44-48), on the GPU."""
    return _stage_time(profile, layer_start, layer_end, k, "f")


def stage_bwd_time(profile: ModelProfile, layer_start: int, layer_end: int, k: int) -> float:
    """Per-microbatch backward time of a stage on k replicas (cost.py:51-54), on the GPU."""
    return _stage_time(profile, layer_start, layer_end, k, "b")


def stage_compute_time(profile: ModelProfile, layer_start: int, layer_end: int, k: int) -> float:
    """stage_fwd_time + stage_bwd_time (cost.py:56-61), on the GPU."""
    if k < 1:
        raise ValidationError("replication factor must be >= 1")
    return _stage_time(profile, layer_start, layer_end, k, "fb")


def cost_summary(plan: Plan, profile: ModelProfile, cluster: ClusterGraph) -> CostSummary:
    """Every planning-cost quantity of a plan (cost.py:172-202) from one device pass."""
    if not plan.stages:
        raise ValueError("max() arg is an empty sequence")
    _check_costed_plan(plan, profile, cluster)
    rec = _plan_costs([[(s.layer_start, s.layer_end, list(s.devices)) for s in plan.stages]], profile, cluster,
                      M=plan.microbatch_count)[0]
    lc = rec["lane_cost"]
    per_stage = {s.index: float(lc[2 * k, _CYC]) for k, s in enumerate(plan.stages)}
    ar = {s.index: float(lc[2 * k, _AR]) for k, s in enumerate(plan.stages) if s.replicated}
    per_chan = {n: float(lc[2 * n - 1, _CYC]) for n in range(1, plan.num_stages)}
    cycle = max(list(per_stage.values()) + list(per_chan.values()))
    g, p = _gamma_phi(profile, cluster)
    return CostSummary(per_stage_compute=per_stage, per_channel_comm=per_chan, allreduce=ar, cycle_time=cycle,
                       workload=rec["workload"], gamma=g, phi=p)


def block_durations(blocks: Sequence[Block], plan: Plan, profile: ModelProfile,
                    cluster: ClusterGraph) -> Dict[int, float]:
    """Duration of every block, keyed by position (cost.py:205-230)."""
    if not blocks:
        return {}
    for b in blocks:
        if b.is_compute:
            s = plan.stages[b.stage - 1]
            _check_interval(profile, s.layer_start, s.layer_end)
        else:
            a, c = plan.stages[b.channel - 1], plan.stages[b.channel]
            _check_channel(profile, a.layer_end, a.devices, c.devices, cluster)
    L = profile.num_layers
    lists = []
    for s in plan.stages:   # unreferenced stages only need in-range intervals for the pass
        a = min(max(s.layer_start, 1), L)
        lists.append((a, min(max(s.layer_end, a), L), list(s.devices)))
    lc = _plan_costs([lists], profile, cluster)[0]["lane_cost"]
    N = plan.num_stages
    out: Dict[int, float] = {}
    for b in blocks:
        if b.is_compute:
            row = lc[2 * (b.stage - 1)]
            k = plan.stages[b.stage - 1].replication
            if b.kind == FWD:   # F = (sum f / k) / k, also on the last stage
                out[b.position] = float(row[_FS])
            elif b.kind == BWD:
                out[b.position] = float(row[_BS])
            else:               # FB = stage_compute_time / k (the lane's FB on the last stage)
                out[b.position] = float(row[_DA]) if b.stage == N else float(row[_CYC]) / k
        else:
            row = lc[2 * b.channel - 1]
            out[b.position] = float(row[_DA] if b.kind == COMM_FWD else row[_DB])
    return out


def block_duration(block: Block, plan: Plan, profile: ModelProfile, cluster: ClusterGraph) -> float:
    """cost.py:205-224."""
    return block_durations([block], plan, profile, cluster)[block.position]


def _gamma_phi(profile: ModelProfile, cluster: ClusterGraph) -> Tuple[float, float]:
    check_numeric_range(profile, cluster)
    db = _device.DeviceBatch([(_device.pack(profile, cluster), 1, sum_flags(), None)], capture_events=False,
                             workspace=False)
    db.run("phi")
    h = db.fetch()
    return float(h["gamma"][0]), float(h["phi"][0])


def gamma(profile: ModelProfile, cluster: ClusterGraph) -> float:
    """sum(f + b over layers) / V (cost.py:126-128), on the GPU."""
    return _gamma_phi(profile, cluster)[0]


def phi(profile: ModelProfile, cluster: ClusterGraph) -> float:
    """cost.py:131-142 (also exported as planner.phi), evaluated on the GPU."""
    return _gamma_phi(profile, cluster)[1]
