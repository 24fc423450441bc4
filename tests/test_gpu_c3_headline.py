"""Parity of the exact headline workload (bench.py, BASELINE.json configs[2]).

Every C3 instance the bench times — the 12-instance batch of
``workloads.c3_sweep()`` (96 layers x 64 GPUs, 8x8 two-tier, M = 8..256,
uniform + jitter seed 96) and the jitter seeds 97..103 that ranks 1..7 plan
under ``--gpus N`` — is planned through the same batched device path as the
bench and compared bit-for-bit with the C oracle: device order, the whole
xi sweep (feasibility, workload, makespan, Lemma-1 bound), the chosen plan,
makespan, phi, theorem factor, and every schedule event (start, end, order).
The oracle itself is pinned at this shape by the Python-reference goldens
``tests/golden/c3_full_*.json`` (test_oracle_golden.py); the CUDA path is
checked against those goldens directly too.

Also: the -0.0 / zero-duration-block goldens (tests/golden/edge.json).
"""

import glob
import os

import pytest

from helpers import GOLDEN, block_labels, load, model_of, oracle_spp_parallel, spec_from_workload

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


def check(results, wants):
    for r, (want, ids) in zip(results, wants):
        assert list(r.device_order) == [ids[k] for k in want["order"]]
        sweep = [[e.stage_count, e.feasible, h(e.workload), h(e.makespan), h(e.bound)] for e in r.sweep]
        assert sweep == [[xi, f, h(w), h(mk), h(bd)] for xi, f, w, mk, bd in want["sweep"]]
        assert [[s.layer_start, s.layer_end, list(s.devices)] for s in r.plan.stages] == \
            [[a, b, [ids[d] for d in devs]] for a, b, devs in want["frags"]]
        assert h(r.makespan) == h(want["makespan"])
        assert h(r.phi) == h(want["phi"]) and h(r.theorem_factor) == h(want["theorem_factor"])
        bl = block_labels(r.plan.num_stages)
        got_ev = [(e.microbatch, e.block, h(e.start), h(e.end)) for e in r.schedule.events]
        assert got_ev == [(m, bl[p][1], h(s), h(e)) for m, p, s, e in want["events"]]
        assert [(w.stage, h(w.start), h(w.end)) for w in r.schedule.allreduce] == \
            [(s, h(a), h(b)) for s, a, b in want["ar"]]


def _bench_batch(seed):
    from paper_2204_10562_b200 import workloads as W
    return W.c3_sweep(jitter_seeds=(None, seed))


def test_bench_batch_all_12_instances_vs_oracle():
    """The rank-0 bench batch, planned as ONE batch through spp_many (the
    bench's device path: one graph replay over the 12 instances)."""
    from paper_2204_10562_b200 import workloads as W
    specs = _bench_batch(96)
    assert len(specs) == 12
    res = P.spp_many(W.models_of(specs))
    check(res, oracle_spp_parallel([spec_from_workload(s) for s in specs]))


@pytest.mark.parametrize("seed", [97, 98, 99, 100, 101, 102, 103])
def test_rank_jitter_seeds_vs_oracle(seed):
    """The jittered half of the batch ranks 1..7 plan under --gpus N."""
    from paper_2204_10562_b200 import workloads as W
    specs = [W.c3_gpt96(M, seed) for M in W.C3_MICROBATCHES]
    res = P.spp_many(W.models_of(specs))
    check(res, oracle_spp_parallel([spec_from_workload(s) for s in specs]))


def test_single_instance_path_matches_batch():
    """One C3 instance alone (the p50-latency path: split critical-path DP
    chain) gives the same result as inside the 12-instance batch."""
    from paper_2204_10562_b200 import workloads as W
    specs = _bench_batch(96)
    many = P.spp_many(W.models_of(specs))
    for k in (0, 2, 11):
        assert P.spp(*specs[k].to_model()) == many[k]


def _full_goldens():
    return sorted(glob.glob(os.path.join(GOLDEN, "c3_full_*.json")))


@pytest.mark.parametrize("path", _full_goldens() or [None])
def test_c3_full_python_reference_golden(path):
    """96 x 64 results produced by the Python reference itself (pipeplan.spp,
    hours of CPU per case; tests/golden/make_c3_full.py)."""
    if path is None:
        pytest.skip("no c3_full_*.json golden generated yet")
    case = load(os.path.basename(path)[:-5])
    r = P.spp(*model_of(case["input"]))
    assert list(r.device_order) == case["device_order"]
    assert [[e.stage_count, e.feasible, h(e.workload), h(e.makespan), h(e.bound)] for e in r.sweep] == case["sweep"]
    assert [[s.layer_start, s.layer_end, list(s.devices)] for s in r.plan.stages] == case["plan"]["stages"]
    assert (h(r.makespan), h(r.phi), h(r.theorem_factor)) == (case["makespan"], case["phi"], case["theorem_factor"])
    s = case["schedule"]
    assert [[w.stage, h(w.start), h(w.end)] for w in r.schedule.allreduce] == s["allreduce"]
    if s["events"] is not None:
        assert [[e.resource, e.microbatch, e.block, h(e.start), h(e.end)] for e in r.schedule.events] == s["events"]
    else:
        assert len(r.schedule.events) == s["n_events"]


def test_edge_semantics_goldens():
    """-0.0 inputs and zero-duration blocks, against the reference goldens."""
    data = load("edge")
    res = P.spp_many([model_of(c["input"]) for c in data["spp"]])
    for c, r in zip(data["spp"], res):
        name = c["input"]["name"]
        assert list(r.device_order) == c["device_order"], name
        assert [[e.stage_count, e.feasible, h(e.workload), h(e.makespan), h(e.bound)] for e in r.sweep] == \
            c["sweep"], name
        assert [[s.layer_start, s.layer_end, list(s.devices)] for s in r.plan.stages] == c["plan"]["stages"], name
        assert (h(r.makespan), h(r.phi), h(r.theorem_factor)) == (c["makespan"], c["phi"], c["theorem_factor"])
        ev = [[e.resource, e.microbatch, e.block, h(e.start), h(e.end)] for e in r.schedule.events]
        assert ev == c["schedule"]["events"], name
        assert [[w.stage, h(w.start), h(w.end)] for w in r.schedule.allreduce] == c["schedule"]["allreduce"]
    for c in data["sim"]:
        prof, clu, _ = model_of(c["input"])
        plan = P.Plan(stages=tuple(P.Stage(index=n + 1, layer_start=a, layer_end=b, devices=tuple(d))
                                   for n, (a, b, d) in enumerate(c["plan"]["stages"])),
                      microbatch_count=c["plan"]["M"])
        queues = {k: tuple(tuple(x) for x in v) for k, v in c["queues"].items()}
        assert h(P.lemma1_bound(plan, prof, clu)) == c["lemma1_bound"], c["name"]
        if "error" in c:
            with pytest.raises(P.SchedulingError) as ei:
                P.simulate_with_order(plan, prof, clu, queues, forward_barrier=c["forward_barrier"])
            assert str(ei.value) == c["error"][1], c["name"]
            continue
        got = P.simulate_with_order(plan, prof, clu, queues, forward_barrier=c["forward_barrier"])
        assert [[e.resource, e.microbatch, e.block, h(e.start), h(e.end)] for e in got.events] == \
            c["schedule"]["events"], c["name"]
        assert [[w.stage, h(w.start), h(w.end)] for w in got.allreduce] == c["schedule"]["allreduce"], c["name"]
        assert h(got.makespan) == c["schedule"]["makespan"], c["name"]
