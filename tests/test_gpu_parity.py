"""CUDA path vs the reference goldens and the C oracle: bit-exact.

Every float is compared by its bits (float.hex) — plans, workloads,
makespans, Lemma-1 bounds, event start/end times, AllReduce windows, phi.
Needs a GPU (run on the B200 box); fixtures come from the live reference
(tests/golden/make_golden.py), the oracle covers everything beyond them.
"""

import math
import random

import numpy as np
import pytest

import oracle as O
from helpers import fx, load, model_of, oracle_instance

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2204_10562_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2204_10562_b200 import _lib
    _lib.load()   # fail loudly if the native library is missing


def h(x):
    return None if x is None else float(x).hex()


def result_as_fixture(r):
    return {
        "device_order": list(r.device_order),
        "sweep": [[e.stage_count, e.feasible, h(e.workload), h(e.makespan), h(e.bound)] for e in r.sweep],
        "plan": {"stages": [[s.layer_start, s.layer_end, list(s.devices)] for s in r.plan.stages],
                 "M": r.plan.microbatch_count},
        "makespan": h(r.makespan), "phi": h(r.phi), "theorem_factor": h(r.theorem_factor),
    }


def sched_as_fixture(s):
    return {"events": [[e.resource, e.microbatch, e.block, h(e.start), h(e.end)] for e in s.events],
            "allreduce": [[w.stage, h(w.start), h(w.end)] for w in s.allreduce], "makespan": h(s.makespan)}


# ------------------------------------------------------------------ goldens
def test_spp_matches_reference_goldens_batched():
    cases = load("spp")["cases"]
    insts = [model_of(c["input"]) for c in cases]
    got = P.spp_many(insts)
    for c, r in zip(cases, got):
        name = c["input"]["name"]
        want = {k: c[k] for k in ("device_order", "sweep", "plan", "makespan", "phi", "theorem_factor")}
        assert result_as_fixture(r) == want, name
        s = sched_as_fixture(r.schedule)
        if c["schedule"]["events"] is not None:
            assert s == c["schedule"], name
        else:
            assert len(r.schedule.events) == c["schedule"]["n_events"]
            assert s["allreduce"] == c["schedule"]["allreduce"] and s["makespan"] == c["schedule"]["makespan"]


def test_spp_single_calls_match_goldens():
    for c in load("spp")["cases"][:12]:
        r = P.spp(*model_of(c["input"]))
        assert result_as_fixture(r)["sweep"] == c["sweep"]
        assert sched_as_fixture(r.schedule) == c["schedule"]


def test_partition_solver_cells_match_reference():
    for case in load("prm")["cases"]:
        prof, clu, M = model_of(case["input"])
        order = tuple(case["order"])
        ordering = P.DeviceOrdering(order=order, rank={v: k + 1 for k, v in enumerate(order)})
        solver = P.PartitionSolver(prof, clu, ordering, M, allow_replication=case["allow_replication"])
        ok_cells = [c for c in case["cells"] if c[4] != "error"]
        got = solver.solve_many([tuple(c[:4]) for c in ok_cells])
        for c, g in zip(ok_cells, got):
            assert h(g.workload) == c[4], c[:4]
            want = None if c[5] is None else tuple((a, b, tuple(d)) for a, b, d in c[5])
            assert g.stages == want, c[:4]
        for c in case["cells"]:
            if c[4] == "error":
                with pytest.raises(P.ValidationError, match=c[5]):
                    solver.solve(*c[:4])
        for xi, w, plan in case["best"]:
            gw, gp = solver.best_partition(xi)
            assert h(gw) == w
            if plan is None:
                assert gp is None
            else:
                assert [[s.layer_start, s.layer_end, list(s.devices)] for s in gp.stages] == plan["stages"]


def _plan_of(d):
    return P.Plan(stages=tuple(P.Stage(index=n + 1, layer_start=a, layer_end=b, devices=tuple(devs))
                               for n, (a, b, devs) in enumerate(d["stages"])), microbatch_count=d["M"])


def test_simulation_matches_reference_goldens():
    for case in load("sim")["cases"]:
        prof, clu, _ = model_of(case["input"])
        plan = _plan_of(case["plan"])
        assert h(P.lemma1_bound(plan, prof, clu)) == case["lemma1_bound"], case["name"]
        queues = {k: tuple(tuple(x) for x in v) for k, v in case["queues"].items()}
        if "error" in case:
            with pytest.raises(P.SchedulingError) as ei:
                P.simulate_with_order(plan, prof, clu, queues, forward_barrier=case["forward_barrier"])
            assert str(ei.value) == case["error"][1], case["name"]
            continue
        got = P.simulate_with_order(plan, prof, clu, queues, forward_barrier=case["forward_barrier"])
        assert sched_as_fixture(got) == case["schedule"], case["name"]
        if case.get("pe") and not case["forward_barrier"]:
            assert sched_as_fixture(P.simulate_pe(plan, prof, clu)) == case["schedule"], case["name"]


def test_execution_order_closed_form():
    for case in load("sim")["cases"]:
        if case.get("pe"):
            plan = _plan_of(case["plan"])
            got = P.compute_execution_order(plan).queues
            assert {k: [list(x) for x in v] for k, v in got.items()} == case["queues"]


def test_ordering_matches_reference_goldens():
    data = load("ordering")
    for case in data["min_cut"]:
        clu = P.make_cluster(case["gpu_ids"], [(a, b, fx(w)) for a, b, w in case["links"]])
        a, b, w = P.global_min_cut(clu)
        assert (list(a), list(b), h(w)) == (case["side_a"], case["side_b"], case["weight"])
    for case in data["rdo"]:
        clu = P.make_cluster(case["gpu_ids"], [(a, b, fx(w)) for a, b, w in case["links"]])
        assert list(P.rdo(clu).order) == case["order"]


# ------------------------------------------------------------------ oracle differential
def _random_instance(rng, Lmax=10, Vmax=6, Mmax=16):
    L = rng.randint(1, Lmax)
    V = rng.randint(1, Vmax)
    M = rng.randint(1, Mmax)
    lu = lambda lo, hi: math.exp(rng.uniform(math.log(lo), math.log(hi)))
    fwd = [lu(1e-3, 1.0) for _ in range(L)]
    bwd = [lu(1e-3, 2.0) for _ in range(L)]
    par = [lu(1e6, 1e10) for _ in range(L)]
    ef = [lu(1e5, 1e9) for _ in range(L - 1)]
    eb = [lu(1e5, 1e9) for _ in range(L - 1)]
    ids = rng.sample(range(1, 1000), V)
    links = [(a, b, lu(1e8, 1e11)) for i, a in enumerate(ids) for b in ids[i + 1:]]
    return fwd, bwd, par, ef, eb, ids, links, M


def _spec(fwd, bwd, par, ef, eb, ids, links, M):
    return {"name": "r", "fwd": [x.hex() for x in fwd], "bwd": [x.hex() for x in bwd],
            "param": [x.hex() for x in par], "efwd": [x.hex() for x in ef], "ebwd": [x.hex() for x in eb],
            "gpu_ids": ids, "links": [[a, b, w.hex()] for a, b, w in links], "M": M}


def _check_vs_oracle(specs, results):
    for spec, r in zip(specs, results):
        inst, ids = oracle_instance(spec)
        want = O.spp(inst)
        assert list(r.device_order) == [ids[k] for k in want["order"]]
        sweep = [[xi, f, h(w), h(mk), h(bd)] for xi, f, w, mk, bd in want["sweep"]]
        assert result_as_fixture(r)["sweep"] == sweep
        assert [[s.layer_start, s.layer_end, list(s.devices)] for s in r.plan.stages] == \
            [[a, b, [ids[d] for d in devs]] for a, b, devs in want["frags"]]
        assert h(r.makespan) == h(want["makespan"])
        assert h(r.phi) == h(want["phi"]) and h(r.theorem_factor) == h(want["theorem_factor"])
        lab = {}
        got_ev = [(e.microbatch, e.block, h(e.start), h(e.end)) for e in r.schedule.events]
        from helpers import block_labels
        bl = block_labels(r.plan.num_stages)
        assert got_ev == [(m, bl[p][1], h(s), h(e)) for m, p, s, e in want["events"]]


def test_random_instances_vs_oracle():
    rng = random.Random(424242)
    specs = [_spec(*_random_instance(rng)) for _ in range(400)]
    res = P.spp_many([model_of(s) for s in specs])
    _check_vs_oracle(specs, res)


def test_wider_random_instances_vs_oracle():
    rng = random.Random(77)
    specs = [_spec(*_random_instance(rng, Lmax=40, Vmax=24, Mmax=64)) for _ in range(40)]
    res = P.spp_many([model_of(s) for s in specs])
    _check_vs_oracle(specs, res)


def test_event_order_ties_vs_oracle():
    """Equal costs and zero-byte edges: many events share a start time, so the
    device event order (k_event_order) is decided by the (resource key,
    microbatch, position) tie rule."""
    rng = random.Random(5)
    specs = []
    for L, V, M in ((6, 4, 5), (12, 8, 16), (9, 6, 7), (24, 16, 32), (1, 3, 4), (5, 1, 9)):
        ids = rng.sample(range(1, 1000), V)
        e = [0.0] * (L - 1) if L % 2 == 0 else [1e6] * (L - 1)
        specs.append(_spec([1.0] * L, [2.0] * L, [1e6] * L, e, list(e), ids,
                           [(a, b, 1e9) for k, a in enumerate(ids) for b in ids[k + 1:]], M))
    res = P.spp_many([model_of(s) for s in specs])
    _check_vs_oracle(specs, res)
    starts = [ev.start for r in res for ev in r.schedule.events]
    assert len(starts) > len(set(starts))   # the cases do tie


def test_event_order_large_schedules_vs_oracle():
    """Schedules beyond the shared-memory merge (M (4N-3) > 18432 events) are
    ordered by the per-event rank kernel."""
    rng = random.Random(11)
    fwd, bwd, par, ef, eb, ids, links, _ = _random_instance(rng, Lmax=20, Vmax=12, Mmax=2)
    specs = [_spec(fwd, bwd, par, ef, eb, ids, links, 700)]
    ids = rng.sample(range(1, 1000), 12)
    # heavy parameters on slow links: replication loses, the plan pipelines deep
    specs.append(_spec([1.0] * 24, [2.0] * 24, [1e12] * 24, [1e3] * 23, [1e3] * 23, ids,
                       [(a, b, 1e9) for k, a in enumerate(ids) for b in ids[k + 1:]], 1500))
    res = P.spp_many([model_of(s) for s in specs])
    _check_vs_oracle(specs, res)
    assert max(len(r.schedule.events) for r in res) > 18432


def _spec_from_workload(w):
    return _spec(w.fwd, w.bwd, w.param, w.efwd, w.ebwd, list(w.gpu_ids), w.links, w.M)


def test_named_configs_vs_oracle():
    from paper_2204_10562_b200 import workloads as W
    specs = [_spec_from_workload(w) for w in
             [W.c1_vgg19(), W.c2_bert24()] + [W.c4_instance(k) for k in range(16)]
             + [W.c3_gpt96(M=M, L=96, nodes=2, per_node=8) for M in (8, 64)]
             + [W.c3_gpt96(M=32, jitter_seed=96, L=96, nodes=2, per_node=8)]]
    res = P.spp_many([model_of(s) for s in specs])
    _check_vs_oracle(specs, res)


def test_large_shapes_use_the_chunked_dp_path():
    """L or V above the shared-memory-resident limit (128) run the chunked kernels."""
    rng = random.Random(9)
    specs = []
    lu = lambda lo, hi: math.exp(rng.uniform(math.log(lo), math.log(hi)))
    for L, V, M in ((150, 5, 4), (140, 9, 8), (3, 136, 2)):
        ids = rng.sample(range(1, 1000), V)
        specs.append(_spec([lu(1e-3, 1.0) for _ in range(L)], [lu(1e-3, 2.0) for _ in range(L)],
                           [lu(1e6, 1e10) for _ in range(L)], [lu(1e5, 1e9) for _ in range(L - 1)],
                           [lu(1e5, 1e9) for _ in range(L - 1)], ids,
                           [(a, b, lu(1e8, 1e11)) for k, a in enumerate(ids) for b in ids[k + 1:]], M))
    res = P.spp_many([model_of(s) for s in specs])
    _check_vs_oracle(specs, res)


def test_c3_full_size_vs_oracle():
    """GPT-96 on the 64-GPU 8x8 two-tier topology, M = 8 and jittered M = 256."""
    from paper_2204_10562_b200 import workloads as W
    specs = [_spec_from_workload(W.c3_gpt96(M=8)), _spec_from_workload(W.c3_gpt96(M=256, jitter_seed=96))]
    res = P.spp_many([model_of(s) for s in specs])
    _check_vs_oracle(specs, res)


# ------------------------------------------------------------------ properties at scale
def test_batched_equals_single():
    from paper_2204_10562_b200 import workloads as W
    specs = [W.c4_instance(k) for k in range(8)] + [W.c2_bert24()]
    many = P.spp_many([s.to_model() for s in specs])
    for s, r in zip(specs, many):
        assert P.spp(*s.to_model()) == r


def test_edge_cases():
    # single layer, single GPU, single microbatch
    prof = P.ModelProfile("one", 1, (P.LayerProfile(1, 1.0, 2.0, 0.0),), ())
    r = P.spp(prof, P.make_cluster([7], []), 1)
    assert r.makespan == 3.0 and r.plan.num_stages == 1 and r.sweep[0].bound == 3.0
    # numeric guard
    bad = P.ModelProfile("bad", 1, (P.LayerProfile(1, math.inf, 2.0, 0.0),), ())
    with pytest.raises(P.ValidationError):
        P.spp(bad, P.make_cluster([1], []), 1)


def test_workspace_bounds_check():
    """pp_batch.ws_doubles > 0: pp_rdo / pp_prm / pp_spp validate every
    instance's workspace range first (C callers); too small -> PP_EINVAL."""
    from paper_2204_10562_b200 import _device, _lib, workloads as W
    from paper_2204_10562_b200.partition import sum_flags
    specs = [W.c2_bert24(), W.c4_instance(0)]
    items = [(_device.pack(*s.to_model()[:2]), s.M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for s in specs]
    db = _device.DeviceBatch(items, capture_events=True)
    db.batch.ws_doubles = db.sizes["ws"]
    db.run("spp")   # exact size: accepted
    h = db.fetch()
    assert list(h["best_xi"]) == [len(r.plan.stages) for r in P.spp_many([s.to_model() for s in specs])]
    db.batch.ws_doubles = db.sizes["ws"] - 1
    with pytest.raises(RuntimeError, match="exceeds ws_doubles"):
        db.run("spp")
    db.batch.ws_doubles = 0
