"""validate_schedule (scheduler.py:303-452) on the device checker vs messages
the reference produced for valid and corrupted schedules
(tests/golden/validate.json), plus the acceptance property at scale: every
schedule the device planners emit validates clean."""

import pytest

from helpers import fx, load, model_of

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2204_10562_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2204_10562_b200 import _lib
    _lib.load()


def plan_of(d):
    return P.Plan(tuple(P.Stage(n + 1, a, b, tuple(dv)) for n, (a, b, dv) in enumerate(d["stages"])), d["M"])


def sched_of(d):
    return P.Schedule(events=tuple(P.ScheduleEvent(r, m, b, fx(s), fx(e)) for r, m, b, s, e in d["events"]),
                      allreduce=tuple(P.AllReduceWindow(k, fx(s), fx(e)) for k, s, e in d["allreduce"]),
                      makespan=fx(d["makespan"]))


def test_messages_match_reference():
    for c in load("validate")["cases"]:
        prof, clu, _ = model_of(c["input"])
        got = P.validate_schedule(sched_of(c["schedule"]), plan_of(c["plan"]), prof, clu,
                                  forward_barrier=c["forward_barrier"])
        assert got == c["messages"], c["name"]


def test_device_schedules_validate_clean():
    """LazyEvents path: simulate_pe / gpipe_schedule / cycle schedules of the golden plans."""
    seen = set()
    for c in load("validate")["cases"]:
        if not c["name"].endswith("_valid") or c["name"] in seen:
            continue
        seen.add(c["name"])
        prof, clu, _ = model_of(c["input"])
        plan = plan_of(c["plan"])
        if c["forward_barrier"]:
            s = P.gpipe_schedule(plan, prof, clu)
        else:
            s = P.simulate_pe(plan, prof, clu)
            assert P.validate_schedule(P.simulate_cycle_schedule(plan, prof, clu), plan, prof, clu) == []
        assert P.validate_schedule(s, plan, prof, clu, forward_barrier=c["forward_barrier"]) == [], c["name"]


def test_spp_schedules_validate_at_scale():
    """Acceptance property (test_acceptance.py) at C2/C3 sizes: the selected
    plan's schedule has no violations, and its makespan is within Lemma 1."""
    from paper_2204_10562_b200 import workloads as W
    insts = [W.c2_bert24(M=32).to_model(), W.c3_gpt96(M=128).to_model(), W.c3_gpt96(M=32, jitter_seed=96).to_model()]
    for prof, clu, M in insts:
        r = P.spp(prof, clu, M)
        assert P.validate_schedule(r.schedule, r.plan, prof, clu) == []
        assert r.makespan <= P.lemma1_bound(r.plan, prof, clu) * (1 + 1e-12)


def test_large_m_overlap_check_uses_global_sort():
    """2M > 8192 events per resource: the overlap check sorts in global
    scratch (k_val_ov_*).  Clean PE schedule -> []; the same schedule with one
    stage-1 forward moved onto its predecessor's interval -> the overlap (and
    the dependency messages it causes) are reported, exactly as for a
    shared-memory-sized M with the same corruption."""
    import dataclasses

    def corrupt(sched, M):
        evs = list(sched.events)
        k1 = next(k for k, e in enumerate(evs) if e.resource == "stage1" and e.block == "fwd1" and e.microbatch == 3)
        k0 = next(k for k, e in enumerate(evs) if e.resource == "stage1" and e.block == "fwd1" and e.microbatch == 2)
        d = evs[k1].end - evs[k1].start
        evs[k1] = dataclasses.replace(evs[k1], start=evs[k0].start, end=evs[k0].start + d)
        return P.Schedule(events=tuple(evs), allreduce=sched.allreduce, makespan=sched.makespan)

    layers = tuple(P.LayerProfile(k, 1.0, 2.0, 1e8) for k in (1, 2, 3))
    edges = (P.InterLayerEdge(1, 2, 1e8, 1e8), P.InterLayerEdge(2, 3, 1e8, 1e8))
    prof = P.ModelProfile("bigM", 1, layers, edges)
    clu = P.make_cluster([1, 2, 3], [(1, 2, 1e9), (1, 3, 1e9), (2, 3, 1e9)])
    msgs = {}
    for M in (64, 5000):
        plan = P.Plan((P.Stage(1, 1, 1, (1,)), P.Stage(2, 2, 3, (2, 3))), M)
        s = P.simulate_pe(plan, prof, clu)
        assert P.validate_schedule(s, plan, prof, clu) == []
        msgs[M] = P.validate_schedule(corrupt(s, M), plan, prof, clu)
        assert any(m.startswith("overlap on stage1: (2,fwd1) and (3,fwd1)") or
                   m.startswith("overlap on stage1: (3,fwd1) and (2,fwd1)") for m in msgs[M]), msgs[M]
    assert msgs[64] == msgs[5000]
