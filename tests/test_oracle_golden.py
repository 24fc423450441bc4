"""Pin the C oracle (oracle/pipeplan_oracle.c) to the reference's own outputs.

CPU-only.  Every fixture under tests/golden/ was produced by the live
reference (tests/golden/make_golden.py); the oracle must reproduce every
float bit-for-bit before it is trusted as the checker of the CUDA path.
"""

import numpy as np
import pytest

import oracle as O
from helpers import arrays, block_labels, fx, load, oracle_instance


def test_pysum_matches_cpython():
    data = load("pysum")
    assert data["python"].startswith("3.12")
    for case in data["cases"]:
        x = np.array([fx(v) for v in case["x"]])
        assert O.pysum(x).hex() == case["sum"]


def test_pysum_matches_this_interpreter():
    rng = np.random.default_rng(3)
    for _ in range(2000):
        x = np.exp(rng.uniform(-8, 25, size=rng.integers(1, 40)))
        assert O.pysum(x) == sum(x.tolist())


def _ord_inst(case):
    spec = {"fwd": ["0x1p+0"], "bwd": ["0x1p+0"], "param": ["0x0p+0"], "efwd": [], "ebwd": [],
            "gpu_ids": case["gpu_ids"], "links": case["links"], "M": 1}
    return oracle_instance(spec)


def test_min_cut_golden():
    for case in load("ordering")["min_cut"]:
        inst, ids = _ord_inst(case)
        a, b, w = O.min_cut(inst, range(len(ids)))
        assert [ids[k] for k in a] == case["side_a"]
        assert [ids[k] for k in b] == case["side_b"]
        assert w.hex() == case["weight"]


def test_rdo_golden():
    for case in load("ordering")["rdo"]:
        inst, ids = _ord_inst(case)
        assert [ids[k] for k in O.rdo(inst)] == case["order"]


def test_prm_cells_golden():
    for case in load("prm")["cases"]:
        inst, ids = oracle_instance(case["input"])
        pos = {g: k for k, g in enumerate(ids)}
        order = [pos[g] for g in case["order"]]
        prm = O.Prm(inst, order, case["allow_replication"])
        for l, xi, r, i, w, frags in case["cells"]:
            if w == "error":
                continue  # argument-handling error raised by the host API, not the DP
            st, got_w, got_f = prm.solve(l, xi, r, i)
            assert got_w.hex() == w, (l, xi, r, i)
            if frags is None:
                assert st == 0
            else:
                assert st == 1
                assert [[a, b, [ids[d] for d in devs]] for a, b, devs in got_f] == frags
        for xi, w, plan in case["best"]:
            st, got_w, got_f = prm.best(xi)
            assert got_w.hex() == w
            if plan is None:
                assert st == 0
            else:
                assert [[a, b, [ids[d] for d in devs]] for a, b, devs in got_f] == plan["stages"]


def queues_to_arrays(queues, N):
    """Fixture queue dict -> (q_off, items) in chain resource order."""
    R = 2 * N - 1
    names = [f"stage{r // 2 + 1}" if r % 2 == 0 else f"chan{r // 2 + 1}" for r in range(R)]
    off, items = [0], []
    for nm in names:
        q = queues.get(nm, [])
        items.extend(q)
        off.append(len(items))
    return np.array(off, np.int32), np.array(items if items else [[0, 0]], np.int32), names


def stall_message(res, names, M, N):
    J = 4 * N - 3
    lab = block_labels(N)
    heads = []
    for r in sorted(range(len(names)), key=lambda r: names[r]):
        m, p = res["heads"][r]
        if p:
            heads.append(f"{names[r]} head ({m},{lab[p][1]})")
    return f"stalled with {M * J - res['n_done']} executions left; " + "; ".join(heads)


def test_sim_golden():
    check_sim_cases(load("sim")["cases"])


def check_sim_cases(cases):
    for case in cases:
        inst, ids = oracle_instance(case["input"])
        pos = {g: k for k, g in enumerate(ids)}
        stages = [(a, b, tuple(pos[d] for d in devs)) for a, b, devs in case["plan"]["stages"]]
        plan = O.Plan(stages, case["plan"]["M"])
        q_off, items, names = queues_to_arrays(case["queues"], plan.N)
        res = O.simulate(inst, plan, q_off, items, case["forward_barrier"])
        assert O.lemma1_bound(inst, plan).hex() == case["lemma1_bound"], case["name"]
        if "error" in case:
            assert res["status"] == 1, case["name"]
            assert stall_message(res, names, plan.M, plan.N) == case["error"][1], case["name"]
            continue
        assert res["status"] == 0, case["name"]
        lab = block_labels(plan.N)
        got = [[lab[p][0], m, lab[p][1], s.hex(), e.hex()] for m, p, s, e in res["events"]]
        assert got == case["schedule"]["events"], case["name"]
        assert [[s, a.hex(), b.hex()] for s, a, b in res["ar"]] == case["schedule"]["allreduce"]
        assert res["makespan"].hex() == case["schedule"]["makespan"]


def check_spp(res, case, ids):
    assert [ids[k] for k in res["order"]] == case["device_order"]
    sweep = [[xi, f, w.hex(), None if mk is None else mk.hex(), None if bd is None else bd.hex()]
             for xi, f, w, mk, bd in res["sweep"]]
    assert sweep == case["sweep"]
    assert [[a, b, [ids[d] for d in devs]] for a, b, devs in res["frags"]] == case["plan"]["stages"]
    assert res["makespan"].hex() == case["makespan"]
    assert res["phi"].hex() == case["phi"]
    assert res["theorem_factor"].hex() == case["theorem_factor"]


def test_spp_golden():
    check_spp_cases(load("spp")["cases"])


def test_edge_semantics_golden():
    """-0.0 inputs and zero-duration blocks (tests/golden/edge.json)."""
    data = load("edge")
    check_spp_cases(data["spp"])
    check_sim_cases(data["sim"])


def check_spp_cases(cases):
    for case in cases:
        inst, ids = oracle_instance(case["input"])
        res = O.spp(inst)
        check_spp(res, case, ids)
        sched = case["schedule"]
        if sched["events"] is not None:
            lab = block_labels(res["best_xi"])
            got = [[lab[p][0], m, lab[p][1], s.hex(), e.hex()] for m, p, s, e in res["events"]]
            assert got == sched["events"], case["input"]["name"]
        assert [[s, a.hex(), b.hex()] for s, a, b in res["ar"]] == sched["allreduce"]


def test_spp_batch_matches_single():
    cases = load("spp")["cases"][:24]
    insts = [oracle_instance(c["input"])[0] for c in cases]
    mk, bx = O.spp_batch(insts, 4)
    for k, c in enumerate(cases):
        assert mk[k].hex() == c["makespan"]
        assert bx[k] == len(c["plan"]["stages"])


def test_c3_full_size_python_reference_goldens():
    """The headline shape (96 layers x 64 GPUs, 8x8 two-tier) pinned by the
    Python reference itself (tests/golden/make_c3_full.py: ~2.3 h of
    pipeplan.spp per case): uniform M = 8, jittered M = 8 and M = 256."""
    import glob
    import os
    from helpers import GOLDEN
    paths = sorted(glob.glob(os.path.join(GOLDEN, "c3_full_*.json")))
    assert paths, "no c3_full golden"
    cases = [load(os.path.basename(p)[:-5]) for p in paths]
    from concurrent.futures import ThreadPoolExecutor   # the oracle call releases the GIL
    with ThreadPoolExecutor(len(cases)) as ex:
        list(ex.map(lambda c: check_spp_cases([c]), cases))
