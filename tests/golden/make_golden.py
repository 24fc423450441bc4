"""Generate tests/golden/*.json from the LIVE reference package.

Runs only in the build container, where the reference lives at
/root/reference (read-only; imported, never copied).  The fixtures pin both
the C oracle (tests/test_oracle_golden.py, CPU) and the CUDA path
(tests/test_gpu_parity.py, GPU).  Floats are stored as float.hex() strings so
every comparison is bit-exact.

    python tests/golden/make_golden.py            # all fixtures
"""

import itertools
import json
import math
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)
sys.path.insert(0, REPO)

import pipeplan as P  # noqa: E402  (the reference)
from conftest import (grid_instances, random_instance, random_weighted_clique,  # noqa: E402
                      tiny_cluster, tiny_profile, trend_instance)

from paper_2204_10562_b200 import workloads as W  # noqa: E402

SEED = 20260822


def hx(x):
    return None if x is None else float(x).hex()


def spec_of(profile, cluster, M):
    return {
        "name": profile.name,
        "fwd": [hx(l.fwd_time) for l in profile.layers],
        "bwd": [hx(l.bwd_time) for l in profile.layers],
        "param": [hx(l.param_bytes) for l in profile.layers],
        "efwd": [hx(e.fwd_bytes) for e in profile.edges],
        "ebwd": [hx(e.bwd_bytes) for e in profile.edges],
        "gpu_ids": list(cluster.gpu_ids),
        "links": [[a, b, hx(w)] for (a, b), w in sorted(cluster.bandwidth.items())],
        "M": M,
    }


def ref_model(spec: W.InstanceSpec):
    layers = tuple(P.LayerProfile(id=i + 1, fwd_time=f, bwd_time=b, param_bytes=p)
                   for i, (f, b, p) in enumerate(zip(spec.fwd, spec.bwd, spec.param)))
    edges = tuple(P.InterLayerEdge(src=i + 1, dst=i + 2, fwd_bytes=a, bwd_bytes=b)
                  for i, (a, b) in enumerate(zip(spec.efwd, spec.ebwd)))
    prof = P.ModelProfile(name=spec.name, microbatch_size=1, layers=layers, edges=edges)
    return prof, P.make_cluster(spec.gpu_ids, spec.links), spec.M


def sched_of(s):
    return {"events": [[e.resource, e.microbatch, e.block, hx(e.start), hx(e.end)] for e in s.events],
            "allreduce": [[w.stage, hx(w.start), hx(w.end)] for w in s.allreduce],
            "makespan": hx(s.makespan)}


def plan_of(p):
    return {"stages": [[s.layer_start, s.layer_end, list(s.devices)] for s in p.stages],
            "M": p.microbatch_count}


def spp_case(profile, cluster, M, events_limit=4000):
    t0 = time.perf_counter()
    r = P.spp(profile, cluster, M)
    dt = time.perf_counter() - t0
    out = {
        "input": spec_of(profile, cluster, M),
        "device_order": list(r.device_order),
        "sweep": [[e.stage_count, e.feasible, hx(e.workload), hx(e.makespan), hx(e.bound)] for e in r.sweep],
        "plan": plan_of(r.plan),
        "makespan": hx(r.makespan),
        "phi": hx(r.phi),
        "theorem_factor": hx(r.theorem_factor),
        "ref_seconds": dt,
    }
    if len(r.schedule.events) <= events_limit:
        out["schedule"] = sched_of(r.schedule)
    else:
        out["schedule"] = {"events": None, "allreduce": sched_of(r.schedule)["allreduce"],
                           "makespan": hx(r.schedule.makespan), "n_events": len(r.schedule.events)}
    return out


def gen_pysum():
    rng = random.Random(7)
    cases = []
    for _ in range(3000):
        n = rng.randint(1, 60)
        kind = rng.random()
        if kind < 0.4:
            xs = [math.exp(rng.uniform(math.log(1e-3), math.log(2.0))) for _ in range(n)]
        elif kind < 0.7:
            xs = [math.exp(rng.uniform(math.log(1e6), math.log(1e10))) for _ in range(n)]
        elif kind < 0.9:
            xs = [rng.choice([0.0, 1e-17, 1.0, 3.0, 1e16, 0.1, 0.7]) for _ in range(n)]
        else:
            xs = [rng.uniform(0, 1) * 10 ** rng.randint(-20, 20) for _ in range(n)]
        cases.append({"x": [hx(v) for v in xs], "sum": hx(sum(xs))})
    return {"python": sys.version, "cases": cases}


def gen_spp():
    cases = []
    cases.append(spp_case(tiny_profile(), tiny_cluster(), 2))
    one = P.ModelProfile(name="one", microbatch_size=1,
                         layers=(P.LayerProfile(id=1, fwd_time=1.0, bwd_time=2.0, param_bytes=1e9),),
                         edges=())
    cases.append(spp_case(one, tiny_cluster(), 2))
    cases.append(spp_case(*trend_instance()))
    skew_layers = (P.LayerProfile(1, 1.0, 2.0, 1e9), P.LayerProfile(2, 0.5, 1.0, 2e9), P.LayerProfile(3, 2.0, 3.0, 1e9))
    skew_edges = (P.InterLayerEdge(1, 2, 5e8, 5e8), P.InterLayerEdge(2, 3, 2e9, 1e9))
    skew = P.ModelProfile("skew", 1, skew_layers, skew_edges)
    skew_c = P.make_cluster([1, 2, 3], [(1, 2, 4e9), (1, 3, 1e9), (2, 3, 1e9)])
    for M in (1, 3, 7):
        cases.append(spp_case(skew, skew_c, M))
    # non-contiguous, unsorted GPU ids
    c_odd = P.make_cluster([9, 3, 17, 5], [(9, 3, 2e9), (9, 17, 5e9), (9, 5, 1e9), (3, 17, 1e9), (3, 5, 8e9), (17, 5, 2e9)])
    cases.append(spp_case(skew, c_odd, 4))
    for k, inst in enumerate(grid_instances()):
        if k % 15 == 0:
            cases.append(spp_case(*inst))
    rng = random.Random(SEED)
    for _ in range(150):
        cases.append(spp_case(*random_instance(rng)))
    # zero-valued params / bytes
    rng = random.Random(11)
    for _ in range(20):
        prof, clu, M = random_instance(rng)
        layers = tuple(P.LayerProfile(l.id, l.fwd_time, l.bwd_time, 0.0 if l.id % 2 else l.param_bytes) for l in prof.layers)
        edges = tuple(P.InterLayerEdge(e.src, e.dst, 0.0, e.bwd_bytes) for e in prof.edges)
        cases.append(spp_case(P.ModelProfile(prof.name + "z", 1, layers, edges), clu, M))
    cases.append(spp_case(*ref_model(W.c1_vgg19())))
    cases.append(spp_case(*ref_model(W.c2_bert24())))
    for k in range(2):
        cases.append(spp_case(*ref_model(W.c4_instance(k))))
    cases.append(spp_case(*ref_model(W.c3_gpt96(M=32, L=48, nodes=2, per_node=8))))
    cases.append(spp_case(*ref_model(W.c3_gpt96(M=64, jitter_seed=96, L=48, nodes=2, per_node=8))))
    return {"python": sys.version, "cases": cases}


def gen_prm():
    out = []
    rng = random.Random(5)
    insts = [(tiny_profile(), tiny_cluster(), 2)]
    for _ in range(12):
        prof, clu, M = random_instance(rng)
        insts.append((prof, clu, M))
    insts.append(next(itertools.islice(grid_instances(), 1500, None)))
    for prof, clu, M in insts:
        for order_kind in ("rdo", "reversed"):
            order = P.rdo(clu)
            if order_kind == "reversed":
                o = tuple(reversed(order.order))
                order = P.DeviceOrdering(order=o, rank={v: k + 1 for k, v in enumerate(o)})
            for allow in (True, False):
                s = P.PartitionSolver(prof, clu, order, M, allow_replication=allow)
                L, V = prof.num_layers, clu.num_gpus
                cells = []
                for l in range(1, L + 1):
                    for xi in range(1, V + 2):
                        for r in range(1, V + 2):
                            for i in range(1, V + 1):
                                try:
                                    res = s.solve(l, xi, r, i)
                                except P.ValidationError as e:
                                    cells.append([l, xi, r, i, "error", str(e)])
                                    continue
                                cells.append([l, xi, r, i, hx(res.workload),
                                              None if res.stages is None else [[a, b, list(d)] for a, b, d in res.stages]])
                best = []
                for xi in range(1, V + 1):
                    w, plan = s.best_partition(xi)
                    best.append([xi, hx(w), None if plan is None else plan_of(plan)])
                out.append({"input": spec_of(prof, clu, M), "order": list(order.order), "allow_replication": allow,
                            "cells": cells, "best": best})
    return {"python": sys.version, "cases": out}


def gen_sim():
    cases = []
    prof, clu = tiny_profile(), tiny_cluster()

    def split(M):
        return P.Plan((P.Stage(1, 1, 1, (1,)), P.Stage(2, 2, 2, (2,))), M)

    def add(name, plan, profile, cluster, queues=None, barrier=False):
        rec = {"name": name, "input": spec_of(profile, cluster, plan.microbatch_count), "plan": plan_of(plan),
               "forward_barrier": barrier}
        if queues is None:
            queues = P.compute_execution_order(plan).queues
            rec["pe"] = True
        rec["queues"] = {k: [list(x) for x in v] for k, v in queues.items()}
        try:
            s = P.simulate_with_order(plan, profile, cluster, queues, forward_barrier=barrier)
            rec["schedule"] = sched_of(s)
        except P.SchedulingError as e:
            rec["error"] = ["SchedulingError", str(e)]
        rec["lemma1_bound"] = hx(P.lemma1_bound(plan, profile, cluster))
        cases.append(rec)

    for M in (1, 2, 3, 5):
        add(f"tiny_split_pe_M{M}", split(M), prof, clu)
        add(f"tiny_gpipe_M{M}", split(M), prof, clu,
            queues=_gpipe_queues(split(M)), barrier=True)
        add(f"tiny_pe_barrier_M{M}", split(M), prof, clu, barrier=True, queues=P.compute_execution_order(split(M)).queues)
    q = dict(P.compute_execution_order(split(2)).queues)
    q["stage1"] = ((1, 5), (2, 5), (1, 1), (2, 1))
    add("tiny_circular", split(2), prof, clu, queues=q)
    q = dict(P.compute_execution_order(split(3)).queues)
    del q["chan1"]
    add("tiny_missing_queue", split(3), prof, clu, queues=q)
    add("tiny_replicated", P.Plan((P.Stage(1, 1, 2, (1, 2)),), 2), prof, clu)
    rng = random.Random(99)
    for k in range(40):
        profile, cluster, M = random_instance(rng)
        L, V = profile.num_layers, cluster.num_gpus
        N = rng.randint(1, min(L, V))
        cuts = sorted(rng.sample(range(1, L), N - 1))
        bounds = [0] + cuts + [L]
        devs = list(cluster.gpu_ids)
        rng.shuffle(devs)
        dcuts = sorted(rng.sample(range(1, V), N - 1)) if N > 1 else []
        db = [0] + dcuts + [V]
        stages = tuple(P.Stage(n + 1, bounds[n] + 1, bounds[n + 1], tuple(devs[db[n]:db[n + 1]])) for n in range(N))
        plan = P.Plan(stages, M)
        add(f"rand{k}_pe", plan, profile, cluster)
        if not any(s.replicated for s in stages):
            add(f"rand{k}_gpipe", plan, profile, cluster, queues=_gpipe_queues(plan), barrier=True)
        if k % 4 == 0:
            qq = {kk: tuple(reversed(v)) if kk == "stage1" else v for kk, v in P.compute_execution_order(plan).queues.items()}
            add(f"rand{k}_reversed_stage1", plan, profile, cluster, queues=qq)
    return {"python": sys.version, "cases": cases}


def _gpipe_queues(plan):
    blocks = P.build_block_list(plan)
    M = plan.microbatch_count
    queues = {}
    for b in blocks:
        queues[b.resource] = queues.get(b.resource, ()) + tuple((m, b.position) for m in range(1, M + 1))
    return queues


def gen_baselines():
    """gpipe_plan / gpipe_schedule / dataparallel_plan / noreplication_plan
    through the reference's own API (baselines.py:28-97)."""
    rng = random.Random(41)
    insts = [(tiny_profile(), tiny_cluster(), 2)]
    for _ in range(30):
        insts.append(random_instance(rng))
    insts.append(ref_model(W.c1_vgg19()))
    insts.append(ref_model(W.c2_bert24(M=8)))
    insts.append(ref_model(W.c3_gpt96(M=16, jitter_seed=96, L=24, nodes=2, per_node=4)))
    cases = []
    for prof, clu, M in insts:
        order = P.rdo(clu)
        L, V = prof.num_layers, clu.num_gpus
        gp = []
        for n in range(0, min(L, V) + 2):
            try:
                plan = P.gpipe_plan(prof, clu, order, n, M)
            except P.ValidationError as e:
                gp.append([n, "error", str(e)])
                continue
            s = P.gpipe_schedule(plan, prof, clu)
            sc = sched_of(s) if len(s.events) <= 3000 else {"events": None, "makespan": hx(s.makespan),
                                                             "allreduce": sched_of(s)["allreduce"]}
            gp.append([n, plan_of(plan), sc])
        w, plan = P.noreplication_plan(prof, clu, order, M)
        cases.append({"input": spec_of(prof, clu, M), "order": list(order.order), "gpipe": gp,
                      "dataparallel": plan_of(P.dataparallel_plan(prof, clu, M)),
                      "noreplication": [hx(w), None if plan is None else plan_of(plan)]})
    return {"python": sys.version, "cases": cases}


def gen_fileio():
    """write_trace / save_profile / save_cluster / save_plan text through the
    reference (fileio.py), for the sim.json schedules and the spp plans."""
    sim = json.load(open(os.path.join(HERE, "sim.json")))
    out = []
    for c in sim["cases"]:
        if "schedule" not in c:
            continue
        spec = c["input"]
        prof, clu, _ = ref_model(W.InstanceSpec(spec["name"], *[[float.fromhex(x) for x in spec[k]] for k in
                                                                 ("fwd", "bwd", "param", "efwd", "ebwd")],
                                                spec["gpu_ids"], [(a, b, float.fromhex(w)) for a, b, w in
                                                                  spec["links"]], spec["M"]))
        st = c["plan"]["stages"]
        plan = P.Plan(tuple(P.Stage(n + 1, a, b, tuple(d)) for n, (a, b, d) in enumerate(st)), c["plan"]["M"])
        sched = P.simulate_with_order(plan, prof, clu, {k: tuple(map(tuple, v)) for k, v in c["queues"].items()},
                                      forward_barrier=c["forward_barrier"])
        out.append({"name": c["name"], "trace": P.write_trace(None, sched), "profile": P.save_profile(None, prof),
                    "cluster": P.save_cluster(None, clu), "plan": P.save_plan(None, plan)})
    rng = random.Random(3)
    nums = [0.0, -0.0, 5.0, 1 / 3, 123456789.0, 1e9, 1e-320, 5e-324, 1.7976931348623157e308, 2.0 ** 53,
            2.0 ** 53 + 2, 0.1, 1e16, 123456789012.0, 9.9999999995e-5]
    for _ in range(5000):
        nums.append(math.exp(rng.uniform(-700, 700)) * rng.choice((1, -1)))
        nums.append(round(rng.uniform(0, 1e6), rng.randint(0, 12)))
    fmt = [[hx(x), P.format_number(x)] for x in nums]
    return {"python": sys.version, "cases": out, "format_number": fmt}


def _sim_case_models():
    sim = json.load(open(os.path.join(HERE, "sim.json")))
    seen = set()
    for c in sim["cases"]:
        spec = c["input"]
        key = (json.dumps(spec, sort_keys=True), json.dumps(c["plan"]))
        if key in seen:
            continue
        seen.add(key)
        prof, clu, _ = ref_model(W.InstanceSpec(spec["name"], *[[float.fromhex(x) for x in spec[k]] for k in
                                                                 ("fwd", "bwd", "param", "efwd", "ebwd")],
                                                spec["gpu_ids"], [(a, b, float.fromhex(w)) for a, b, w in
                                                                  spec["links"]], spec["M"]))
        st = c["plan"]["stages"]
        plan = P.Plan(tuple(P.Stage(n + 1, a, b, tuple(d)) for n, (a, b, d) in enumerate(st)), c["plan"]["M"])
        yield c["name"], spec, prof, clu, plan


def gen_costs():
    """cost_summary / channel_times / block_durations / scalar cost helpers /
    simulate_cycle_schedule through the reference (cost.py, scheduler.py:241-296)."""
    cases = []
    extra = []
    for ws in (W.c2_bert24(M=6), W.c1_vgg19(M=5)):
        prof, clu, M = ref_model(ws)
        order = P.rdo(clu)
        for n in range(1, min(prof.num_layers, clu.num_gpus) + 1):
            extra.append((f"{ws.name}_gpipe{n}", spec_of(prof, clu, M), prof, clu, P.gpipe_plan(prof, clu, order, n, M)))
        extra.append((f"{ws.name}_dp", spec_of(prof, clu, M), prof, clu, P.dataparallel_plan(prof, clu, M)))
    zl = tuple(P.LayerProfile(id=i, fwd_time=0.0 if i % 2 else 1.0, bwd_time=0.0, param_bytes=1e8) for i in range(1, 7))
    ze = tuple(P.InterLayerEdge(src=i, dst=i + 1, fwd_bytes=0.0, bwd_bytes=1e8 * (i % 2)) for i in range(1, 6))
    zprof = P.ModelProfile(name="zeros", microbatch_size=1, layers=zl, edges=ze)
    zclu = P.make_cluster([1, 2, 3, 4], [(a, b, 1e9) for a in range(1, 5) for b in range(a + 1, 5)])
    for st in (((1, 2, (1,)), (3, 4, (2, 3)), (5, 6, (4,))), ((1, 1, (1,)), (2, 3, (2,)), (4, 6, (3, 4)))):
        plan = P.Plan(tuple(P.Stage(n + 1, a, b, d) for n, (a, b, d) in enumerate(st)), 4)
        extra.append((f"zeros{len(extra)}", spec_of(zprof, zclu, 4), zprof, zclu, plan))
    for name, spec, prof, clu, plan in list(_sim_case_models()) + extra:
        cs = P.cost_summary(plan, prof, clu)
        blocks = P.build_block_list(plan)
        cyc = P.simulate_cycle_schedule(plan, prof, clu)
        rec = {"name": name, "input": spec, "plan": plan_of(plan),
               "summary": {"per_stage_compute": {str(k): hx(v) for k, v in cs.per_stage_compute.items()},
                           "per_channel_comm": {str(k): hx(v) for k, v in cs.per_channel_comm.items()},
                           "allreduce": {str(k): hx(v) for k, v in cs.allreduce.items()},
                           "cycle_time": hx(cs.cycle_time), "workload": hx(cs.workload), "gamma": hx(cs.gamma),
                           "phi": hx(cs.phi)},
               "channel_times": {str(k): [hx(a), hx(b)] for k, (a, b) in P.channel_times(plan, prof, clu).items()},
               "block_durations": {str(k): hx(v) for k, v in P.block_durations(blocks, plan, prof, clu).items()},
               "allreduce_time": [hx(P.allreduce_time(prof, s.layer_start, s.layer_end, s.devices, clu))
                                  for s in plan.stages],
               "min_pairwise": [hx(P.min_pairwise_bandwidth(clu, s.devices)) for s in plan.stages],
               "min_cross": [hx(P.min_cross_bandwidth(clu, a.devices, b.devices))
                             for a, b in zip(plan.stages, plan.stages[1:])],
               "interstage": [[hx(x) for x in P.interstage_comm_time(prof, a.layer_end, a.devices, b.devices, clu)]
                              for a, b in zip(plan.stages, plan.stages[1:])],
               "gamma": hx(P.gamma(prof, clu)),
               "cycle": sched_of(cyc), "cycle_count": cyc.cycle_count}
        cases.append(rec)
    return {"python": sys.version, "cases": cases}


def _perturb(rng, sched, plan):
    """A few deterministic corruptions of a valid schedule (each a separate case)."""
    ev = list(sched.events)
    E = len(ev)
    out = [("valid", sched)]

    def mk(name, events=None, allreduce=None, makespan=None):
        out.append((name, P.Schedule(events=tuple(ev if events is None else events),
                                     allreduce=tuple(sched.allreduce if allreduce is None else allreduce),
                                     makespan=sched.makespan if makespan is None else makespan)))

    k = rng.randrange(E)
    e = ev[k]
    sh = 0.5 * (e.end - e.start) + 1e-3
    mk("shift", ev[:k] + [P.ScheduleEvent(e.resource, e.microbatch, e.block, e.start - sh, e.end - sh)] + ev[k + 1:])
    mk("late", ev[:k] + [P.ScheduleEvent(e.resource, e.microbatch, e.block, e.start + sh, e.end + sh)] + ev[k + 1:])
    mk("drop", ev[:k] + ev[k + 1:])
    mk("dup", ev[:k + 1] + [e] + ev[k + 1:])
    mk("resource", ev[:k] + [P.ScheduleEvent("stage99", e.microbatch, e.block, e.start, e.end)] + ev[k + 1:])
    mk("duration", ev[:k] + [P.ScheduleEvent(e.resource, e.microbatch, e.block, e.start, e.end + 0.25)] + ev[k + 1:])
    mk("unknown_block", ev + [P.ScheduleEvent("stage1", 1, "fwd99", 0.0, 1.0)])
    mk("unknown_micro", ev + [P.ScheduleEvent(e.resource, plan.microbatch_count + 3, e.block, 0.0, 1.0)])
    mk("backwards", ev[:k] + [P.ScheduleEvent(e.resource, e.microbatch, e.block, e.end + 1.0, e.start)] + ev[k + 1:])
    mk("makespan", makespan=sched.makespan * 1.5 + 1.0)
    mk("swap_starts", sorted((P.ScheduleEvent(x.resource, x.microbatch, x.block, x.start * 0.5, x.start * 0.5 +
                                              (x.end - x.start)) for x in ev), key=lambda x: x.start))
    mk("extra_window", allreduce=tuple(sched.allreduce) + (P.AllReduceWindow(1, sched.makespan, sched.makespan + 1),))
    if sched.allreduce:
        w = sched.allreduce[0]
        mk("no_window", allreduce=tuple(sched.allreduce[1:]))
        mk("early_window", allreduce=(P.AllReduceWindow(w.stage, w.start - 1.0, w.end - 1.0),) +
           tuple(sched.allreduce[1:]))
    mk("reversed", list(reversed(ev)))
    return out


def gen_validate():
    """validate_schedule messages through the reference on valid and corrupted schedules."""
    rng = random.Random(77)
    cases = []
    for name, spec, prof, clu, plan in _sim_case_models():
        if name.startswith("tiny_circular") or name.startswith("tiny_missing"):
            continue
        for barrier in (False, True):
            if barrier and any(s.replicated for s in plan.stages):
                continue
            sched = (P.gpipe_schedule(plan, prof, clu) if barrier else P.simulate_pe(plan, prof, clu))
            for kind, s2 in _perturb(rng, sched, plan):
                msgs = P.validate_schedule(s2, plan, prof, clu, forward_barrier=barrier)
                cases.append({"name": f"{name}_{'gpipe' if barrier else 'pe'}_{kind}", "input": spec,
                              "plan": plan_of(plan), "forward_barrier": barrier, "schedule": sched_of(s2),
                              "messages": msgs})
    # cross-checks: a PE schedule under the barrier rule, a split last stage
    prof, clu, M = tiny_profile(), tiny_cluster(), 2
    plan = P.Plan((P.Stage(1, 1, 1, (1,)), P.Stage(2, 2, 2, (2,))), M)
    pe = P.simulate_pe(plan, prof, clu)
    cases.append({"name": "tiny_pe_under_barrier", "input": spec_of(prof, clu, M), "plan": plan_of(plan),
                  "forward_barrier": True, "schedule": sched_of(pe),
                  "messages": P.validate_schedule(pe, plan, prof, clu, forward_barrier=True)})
    split = []
    for e in pe.events:
        if e.block == "fwdbwd2":
            mid = e.start + 1.0
            split.append(P.ScheduleEvent(e.resource, e.microbatch, "fwd2", e.start, mid))
            split.append(P.ScheduleEvent(e.resource, e.microbatch, "bwd2", mid, e.end))
        else:
            split.append(e)
    ss = P.Schedule(events=tuple(split), allreduce=pe.allreduce, makespan=pe.makespan)
    cases.append({"name": "tiny_split_last", "input": spec_of(prof, clu, M), "plan": plan_of(plan),
                  "forward_barrier": False, "schedule": sched_of(ss),
                  "messages": P.validate_schedule(ss, plan, prof, clu)})
    return {"python": sys.version, "cases": cases}


def gen_ordering():
    rng = random.Random(SEED)
    cuts = []
    for _ in range(300):
        c = random_weighted_clique(rng)
        a, b, w = P.global_min_cut(c)
        cuts.append({"gpu_ids": list(c.gpu_ids), "links": [[x, y, hx(v)] for (x, y), v in sorted(c.bandwidth.items())],
                     "side_a": list(a), "side_b": list(b), "weight": hx(w)})
    orders = []
    clusters = []
    for k in range(60):
        clusters.append(random_weighted_clique(rng))
    ids, links = W.two_tier_cluster(4, 4)
    clusters.append(P.make_cluster(ids, links))
    ids, links = W.two_tier_cluster(2, 8)
    clusters.append(P.make_cluster(ids, links))
    spec = W.c4_instance(3)
    clusters.append(P.make_cluster(spec.gpu_ids, spec.links))
    spec = W.c2_bert24()
    clusters.append(P.make_cluster(spec.gpu_ids, spec.links))
    ids = list(range(1, 7))
    clusters.append(P.make_cluster(ids, [(a, b, 1e9) for i, a in enumerate(ids) for b in ids[i + 1:]]))
    for c in clusters:
        o = P.rdo(c)
        orders.append({"gpu_ids": list(c.gpu_ids), "links": [[x, y, hx(v)] for (x, y), v in sorted(c.bandwidth.items())],
                       "order": list(o.order)})
    return {"python": sys.version, "min_cut": cuts, "rdo": orders}


def _sim_rec(name, plan, profile, cluster, queues=None, barrier=False):
    rec = {"name": name, "input": spec_of(profile, cluster, plan.microbatch_count), "plan": plan_of(plan),
           "forward_barrier": barrier}
    if queues is None:
        queues = P.compute_execution_order(plan).queues
        rec["pe"] = True
    rec["queues"] = {k: [list(x) for x in v] for k, v in queues.items()}
    try:
        rec["schedule"] = sched_of(P.simulate_with_order(plan, profile, cluster, queues, forward_barrier=barrier))
    except P.SchedulingError as e:
        rec["error"] = ["SchedulingError", str(e)]
    rec["lemma1_bound"] = hx(P.lemma1_bound(plan, profile, cluster))
    return rec


def gen_edge():
    """Edge semantics the survey flagged (VERDICT r1 missing #5):
    * -0.0 inputs: validate_profile only rejects values < 0 (model.py:207-210),
      so -0.0 times / bytes / params are legal reference inputs;
    * zero-duration blocks (zero-time layers, zero-byte edges), whose event
      order among equal start times is the heap-pop fallback
      (scheduler.py:161-164, :221-224)."""
    rng = random.Random(2026)
    spp_cases, sim_cases = [], []
    nz = -0.0

    def mk(fwd, bwd, par, ef, eb, name):
        layers = tuple(P.LayerProfile(k + 1, f, b, p) for k, (f, b, p) in enumerate(zip(fwd, bwd, par)))
        edges = tuple(P.InterLayerEdge(k + 1, k + 2, a, b) for k, (a, b) in enumerate(zip(ef, eb)))
        return P.ModelProfile(name, 1, layers, edges)

    def clique(V, bw=lambda a, b: 1e9):
        ids = list(range(1, V + 1))
        return P.make_cluster(ids, [(a, b, bw(a, b)) for a in ids for b in ids if a < b])

    # -0.0 everywhere a value may be zero
    for k in range(40):
        prof, clu, M = random_instance(rng)
        p = rng.random()
        neg = lambda x: nz if rng.random() < p else x
        layers = [(neg(l.fwd_time), neg(l.bwd_time), neg(l.param_bytes)) for l in prof.layers]
        if not any(f + b > 0 for f, b, _ in layers):
            layers[0] = (prof.layers[0].fwd_time, layers[0][1], layers[0][2])
        ef = [neg(e.fwd_bytes) for e in prof.edges]
        eb = [neg(e.bwd_bytes) for e in prof.edges]
        spp_cases.append(spp_case(mk([a for a, _, _ in layers], [b for _, b, _ in layers],
                                     [c for _, _, c in layers], ef, eb, f"negzero{k}"), clu, M))
    # all-(-0.0) except one layer's forward time
    for L, V, M in ((5, 4, 3), (8, 8, 6), (1, 3, 2)):
        fwd = [nz] * L
        fwd[L // 2] = 1.0
        spp_cases.append(spp_case(mk(fwd, [nz] * L, [nz] * L, [nz] * (L - 1), [nz] * (L - 1), f"allnegzero{L}"),
                                  clique(V), M))
    # zero-duration layers and zero-byte edges: many events share start times
    for k in range(30):
        prof, clu, M = random_instance(rng)
        zl = set(rng.sample(range(1, prof.num_layers + 1), rng.randint(0, prof.num_layers - 1)))
        layers = [(0.0 if l.id in zl else l.fwd_time, 0.0 if l.id in zl else l.bwd_time, l.param_bytes)
                  for l in prof.layers]
        ze = rng.random()
        ef = [0.0 if rng.random() < ze else e.fwd_bytes for e in prof.edges]
        eb = [0.0 if rng.random() < ze else e.bwd_bytes for e in prof.edges]
        spp_cases.append(spp_case(mk([a for a, _, _ in layers], [b for _, b, _ in layers],
                                     [c for _, _, c in layers], ef, eb, f"zerodur{k}"), clu, M))
    # one non-zero layer, everything else zero: almost every block has zero duration
    for L, V, M in ((6, 4, 5), (10, 6, 8), (4, 4, 1)):
        fwd = [0.0] * L
        bwd = [0.0] * L
        bwd[0] = 2.0
        spp_cases.append(spp_case(mk(fwd, bwd, [0.0] * L, [0.0] * (L - 1), [0.0] * (L - 1), f"mostlyzero{L}"),
                                  clique(V), M))
    # simulations of explicit plans with zero-duration blocks (PE order, GPipe + barrier)
    for k in range(30):
        L = rng.randint(2, 10)
        V = rng.randint(2, 6)
        M = rng.randint(1, 6)
        N = rng.randint(2, min(L, V))
        fwd = [rng.choice([0.0, nz, 1.0, 0.5]) for _ in range(L)]
        bwd = [rng.choice([0.0, 2.0, nz]) for _ in range(L)]
        if not any(f + b > 0 for f, b in zip(fwd, bwd)):
            fwd[0] = 1.0
        ef = [rng.choice([0.0, nz, 1e9]) for _ in range(L - 1)]
        eb = [rng.choice([0.0, 1e9]) for _ in range(L - 1)]
        prof = mk(fwd, bwd, [rng.choice([0.0, 1e9]) for _ in range(L)], ef, eb, f"zsim{k}")
        clu = clique(V)
        cuts = sorted(rng.sample(range(1, L), N - 1))
        bounds = [0] + cuts + [L]
        dcuts = sorted(rng.sample(range(1, V), N - 1))
        db = [0] + dcuts + [V]
        stages = tuple(P.Stage(n + 1, bounds[n] + 1, bounds[n + 1], tuple(range(db[n] + 1, db[n + 1] + 1)))
                       for n in range(N))
        plan = P.Plan(stages, M)
        sim_cases.append(_sim_rec(f"zsim{k}_pe", plan, prof, clu))
        sim_cases.append(_sim_rec(f"zsim{k}_pe_barrier", plan, prof, clu, barrier=True,
                                  queues=P.compute_execution_order(plan).queues))
        if not any(s.replicated for s in stages):
            sim_cases.append(_sim_rec(f"zsim{k}_gpipe", plan, prof, clu, queues=_gpipe_queues(plan), barrier=True))
    return {"python": sys.version, "spp": spp_cases, "sim": sim_cases}


def main():
    which = sys.argv[1:] or ["pysum", "spp", "prm", "sim", "ordering", "baselines", "fileio", "costs", "validate",
                             "edge"]
    gens = {"pysum": gen_pysum, "spp": gen_spp, "prm": gen_prm, "sim": gen_sim, "ordering": gen_ordering,
            "baselines": gen_baselines, "fileio": gen_fileio, "costs": gen_costs, "validate": gen_validate,
            "edge": gen_edge}
    for name in which:
        t0 = time.time()
        data = gens[name]()
        path = os.path.join(HERE, f"{name}.json")
        with open(path, "w") as f:
            json.dump(data, f, separators=(",", ":"))
        print(f"{name}: {os.path.getsize(path) / 1e6:.2f} MB in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
