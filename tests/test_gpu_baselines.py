"""Baseline planners (reference baselines.py) on the CUDA path vs the reference
goldens (tests/golden/baselines.json) and the C oracle: bit-exact."""

import math

import pytest

import oracle as O
from helpers import load, model_of

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2204_10562_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2204_10562_b200 import _lib
    _lib.load()


def h(x):
    return None if x is None else float(x).hex()


def plan_fx(p):
    return {"stages": [[s.layer_start, s.layer_end, list(s.devices)] for s in p.stages], "M": p.microbatch_count}


def sched_fx(s):
    return {"events": [[e.resource, e.microbatch, e.block, h(e.start), h(e.end)] for e in s.events],
            "allreduce": [[w.stage, h(w.start), h(w.end)] for w in s.allreduce], "makespan": h(s.makespan)}


def test_baselines_match_reference_goldens():
    for case in load("baselines")["cases"]:
        prof, clu, M = model_of(case["input"])
        order = P.rdo(clu)
        assert list(order.order) == case["order"]
        for n, *rest in case["gpipe"]:
            if rest[0] == "error":
                with pytest.raises(P.ValidationError, match="infeasible stage count"):
                    P.gpipe_plan(prof, clu, order, n, M)
                continue
            want_plan, want_sched = rest
            plan = P.gpipe_plan(prof, clu, order, n, M)
            assert plan_fx(plan) == want_plan
            got = sched_fx(P.gpipe_schedule(plan, prof, clu))
            if want_sched["events"] is None:
                assert got["makespan"] == want_sched["makespan"] and got["allreduce"] == want_sched["allreduce"]
            else:
                assert got == want_sched
        assert plan_fx(P.dataparallel_plan(prof, clu, M)) == case["dataparallel"]
        w, plan = P.noreplication_plan(prof, clu, order, M)
        assert [h(w), None if plan is None else plan_fx(plan)] == case["noreplication"]


def test_pinned_barrier_timeline_and_replicated_rejection():
    prof, clu, M = model_of(load("baselines")["cases"][0]["input"])
    order = P.rdo(clu)
    s = P.gpipe_schedule(P.gpipe_plan(prof, clu, order, 2, M), prof, clu)
    assert s.makespan == 12.0
    with pytest.raises(P.ValidationError, match="replicated"):
        P.gpipe_schedule(P.dataparallel_plan(prof, clu, M), prof, clu)


def test_gpipe_never_beats_pe_and_matches_oracle_on_c2():
    from paper_2204_10562_b200 import workloads as W
    spec = W.c2_bert24(M=32)
    prof, clu, M = spec.to_model()
    order = P.rdo(clu)
    inst = O.Instance(spec.fwd, spec.bwd, spec.param, spec.efwd, spec.ebwd, _bw(spec), M)
    ids = sorted(spec.gpu_ids)
    for n in range(1, 9):
        plan = P.gpipe_plan(prof, clu, order, n, M)
        barrier = P.gpipe_schedule(plan, prof, clu)
        assert P.simulate_pe(plan, prof, clu).makespan <= barrier.makespan
        op = O.Plan([(s.layer_start, s.layer_end, [ids.index(d) for d in s.devices]) for s in plan.stages], M)
        q = P.baselines.gpipe_queues(plan)
        ref = O.simulate(inst, op, *_oracle_queues(q, n), forward_barrier=True)
        assert barrier.makespan.hex() == float(ref["makespan"]).hex()


def _bw(spec):
    import numpy as np
    ids = sorted(spec.gpu_ids)
    bw = np.zeros((len(ids), len(ids)))
    for a, b, w in spec.links:
        bw[ids.index(a), ids.index(b)] = bw[ids.index(b), ids.index(a)] = w
    return bw


def _oracle_queues(queues, N):
    import numpy as np
    names = [f"stage{r // 2 + 1}" if r % 2 == 0 else f"chan{r // 2 + 1}" for r in range(2 * N - 1)]
    off, items = [0], []
    for nm in names:
        items.extend(queues.get(nm, ()))
        off.append(len(items))
    return np.array(off, np.int32), np.array(items, np.int32).reshape(-1, 2)


def test_noreplication_infeasible_when_fewer_layers_than_gpus():
    case = next(c for c in load("baselines")["cases"] if len(c["input"]["fwd"]) < len(c["input"]["gpu_ids"]))
    prof, clu, M = model_of(case["input"])
    w, plan = P.noreplication_plan(prof, clu, P.rdo(clu), M)
    assert math.isinf(w) and plan is None


def test_trace_of_device_schedule_matches_object_path():
    """write_trace on the LazyEvents of a device schedule (arrays straight to
    pp_format_trace) == write_trace on the materialized ScheduleEvent tuple."""
    from paper_2204_10562_b200 import workloads as W
    prof, clu, M = W.c3_gpt96(M=64, nodes=2, per_node=8, L=48).to_model()
    r = P.spp(prof, clu, M)
    lazy = P.write_trace(None, r.schedule)
    objs = P.Schedule(events=tuple(r.schedule.events), allreduce=r.schedule.allreduce, makespan=r.makespan)
    assert lazy == P.write_trace(None, objs)
    assert len(lazy.splitlines()) == 2 + len(r.schedule.events) + len(r.schedule.allreduce)
