"""Cost API (cost.py) and the lockstep cycle schedule (scheduler.py:241-296) on
the CUDA cost pass / PP_SIM_CYCLE vs reference goldens: bit-exact."""

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


def h(x):
    return None if x is None else float(x).hex()


def plan_of(d):
    return P.Plan(tuple(P.Stage(n + 1, a, b, tuple(dv)) for n, (a, b, dv) in enumerate(d["stages"])), d["M"])


def test_costs_match_reference():
    for c in load("costs")["cases"]:
        prof, clu, _ = model_of(c["input"])
        plan = plan_of(c["plan"])
        cs = P.cost_summary(plan, prof, clu)
        got = {"per_stage_compute": {str(k): h(v) for k, v in cs.per_stage_compute.items()},
               "per_channel_comm": {str(k): h(v) for k, v in cs.per_channel_comm.items()},
               "allreduce": {str(k): h(v) for k, v in cs.allreduce.items()},
               "cycle_time": h(cs.cycle_time), "workload": h(cs.workload), "gamma": h(cs.gamma), "phi": h(cs.phi)}
        assert got == c["summary"], c["name"]
        ct = {str(k): [h(a), h(b)] for k, (a, b) in P.channel_times(plan, prof, clu).items()}
        assert ct == c["channel_times"], c["name"]
        bd = P.block_durations(P.build_block_list(plan), plan, prof, clu)
        assert {str(k): h(v) for k, v in bd.items()} == c["block_durations"], c["name"]
        assert [h(P.allreduce_time(prof, s.layer_start, s.layer_end, s.devices, clu))
                for s in plan.stages] == c["allreduce_time"]
        assert [h(P.min_pairwise_bandwidth(clu, s.devices)) for s in plan.stages] == c["min_pairwise"]
        pairs = list(zip(plan.stages, plan.stages[1:]))
        assert [h(P.min_cross_bandwidth(clu, a.devices, b.devices)) for a, b in pairs] == c["min_cross"]
        assert [[h(x) for x in P.interstage_comm_time(prof, a.layer_end, a.devices, b.devices, clu)]
                for a, b in pairs] == c["interstage"]
        assert h(P.gamma(prof, clu)) == c["gamma"]


def test_cycle_schedule_matches_reference():
    for c in load("costs")["cases"]:
        prof, clu, _ = model_of(c["input"])
        plan = plan_of(c["plan"])
        got = P.simulate_cycle_schedule(plan, prof, clu)
        assert got.cycle_count == c["cycle_count"] == plan.microbatch_count + 4 * plan.num_stages - 4
        s = {"events": [[e.resource, e.microbatch, e.block, h(e.start), h(e.end)] for e in got.events],
             "allreduce": [[w.stage, h(w.start), h(w.end)] for w in got.allreduce], "makespan": h(got.makespan)}
        assert s == c["cycle"], c["name"]
        # Lemma 1 covers the cycle schedule; the event schedule never loses to it
        assert got.makespan <= P.lemma1_bound(plan, prof, clu) * (1 + 1e-12)
        assert P.simulate_pe(plan, prof, clu).makespan <= got.makespan * (1 + 1e-12)


def test_cost_argument_errors():
    c = load("costs")["cases"][0]
    prof, clu, _ = model_of(c["input"])
    L = prof.num_layers
    with pytest.raises(P.ValidationError, match="invalid layer interval"):
        P.allreduce_time(prof, 0, 1, (clu.gpu_ids[0],), clu)
    with pytest.raises(P.ValidationError, match="empty device set"):
        P.allreduce_time(prof, 1, 1, (), clu)
    with pytest.raises(P.ValidationError, match="unknown device"):
        P.allreduce_time(prof, 1, 1, (999,), clu)
    with pytest.raises(P.ValidationError, match="out of range"):
        P.interstage_comm_time(prof, L, (clu.gpu_ids[0],), (clu.gpu_ids[-1],), clu)
    if clu.num_gpus > 1 and L > 1:
        with pytest.raises(P.ValidationError, match="overlapping"):
            P.interstage_comm_time(prof, 1, (clu.gpu_ids[0],), (clu.gpu_ids[0],), clu)
    assert P.min_pairwise_bandwidth(clu, (clu.gpu_ids[0],)) == float("inf")
    assert P.min_cross_bandwidth(clu, (), clu.gpu_ids) == float("inf")
