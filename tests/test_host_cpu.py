"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
host-side layout/ordering logic, validators, and the loud no-GPU failure."""

import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
from helpers import block_labels

import paper_2204_10562_b200 as P
from paper_2204_10562_b200 import _lib
from paper_2204_10562_b200 import workloads as W

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(REPO, "include", "pipeplan_b200.h")).read()
    return sorted(set(re.findall(r"\b(pp_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    return _lib.load(require_device=False)


def test_library_exports_every_declared_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert b"sm_100a" in lib.pp_version()


def test_layout_offsets(lib):
    L = np.array([3, 96, 1], np.int32)
    V = np.array([2, 64, 5], np.int32)
    M = np.array([2, 8, 1], np.int32)
    f = np.zeros(3, np.int32)
    inst = (_lib.PPInstance * 3)()
    tot = [C.c_int64() for _ in range(8)]
    rc = lib.pp_layout(3, L.ctypes.data, V.ctypes.data, M.ctypes.data, f.ctypes.data, C.cast(inst, C.c_void_p),
                       *[C.byref(t) for t in tot])
    assert rc == 0
    assert [inst[k].layer_off for k in range(3)] == [0, 3, 99]
    assert [inst[k].bw_off for k in range(3)] == [0, 4, 4 + 64 * 64]
    assert [inst[k].stage_off for k in range(3)] == [0, 3, 3 + 64 * 65 // 2]
    assert tot[0].value == 100 and tot[4].value == 3 + 2080 + 15
    assert inst[1].ws_off > inst[0].ws_off and tot[7].value > inst[2].ws_off
    bad = np.array([0], np.int32)
    assert lib.pp_layout(1, bad.ctypes.data, V.ctypes.data, M.ctypes.data, f.ctypes.data,
                         C.cast(inst, C.c_void_p), *[C.byref(t) for t in tot]) == -1
    assert b"outside" in lib.pp_last_error()


def test_block_list_matches_reference_layout():
    for N in range(1, 12):
        plan = P.Plan(stages=tuple(P.Stage(n + 1, n + 1, n + 1, (n + 1,)) for n in range(N)), microbatch_count=1)
        got = {b.position: (b.resource, b.label) for b in P.build_block_list(plan)}
        assert got == block_labels(N)


def test_execution_order_closed_form_matches_pass_loop():
    for N in range(1, 9):
        for M in (1, 2, 3, 7, 16):
            plan = P.Plan(stages=tuple(P.Stage(n + 1, n + 1, n + 1, (n + 1,)) for n in range(N)),
                          microbatch_count=M)
            got = P.compute_execution_order(plan).queues
            q_off, items = O.pe_queues(N, M)
            names = [f"stage{r // 2 + 1}" if r % 2 == 0 else f"chan{r // 2 + 1}" for r in range(2 * N - 1)]
            want = {names[r]: tuple(map(tuple, items[q_off[r]:q_off[r + 1]].tolist())) for r in range(2 * N - 1)}
            assert got == want


def test_validators_and_numeric_guard():
    with pytest.raises(P.ValidationError, match="no layers"):
        P.validate_profile(P.ModelProfile("x", 1, (), ()))
    with pytest.raises(P.ValidationError, match="missing pair"):
        P.validate_cluster(P.ClusterGraph((1, 2, 3), {(1, 2): 1.0}))
    with pytest.raises(P.ValidationError, match="asymmetric"):
        P.make_cluster([1, 2], [(1, 2, 1.0), (2, 1, 2.0)])
    prof = P.ModelProfile("x", 1, (P.LayerProfile(1, 1e101, 1.0, 0.0),), ())
    with pytest.raises(P.ValidationError, match="supported range"):
        P.check_numeric_range(prof, P.make_cluster([1], []))


def test_workload_generators_are_deterministic():
    a, b = W.c4_instance(5), W.c4_instance(5)
    assert a.fwd == b.fwd and a.links == b.links
    assert W.c1_vgg19().L == 19 and W.c2_bert24().V == 8
    c3 = W.c3_gpt96()
    assert (c3.L, c3.V) == (96, 64)
    assert len(W.c3_sweep()) == 12
    c5 = W.c5_instance()
    assert (c5.L, c5.V, c5.M) == (1024, 256, 512)
    plan = W.even_split_plan(10, list(range(7)), 3)
    assert plan == [(1, 4, (0, 1, 2)), (5, 7, (3, 4)), (8, 10, (5, 6))]


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    prof, clu, M = W.c2_bert24().to_model()
    with pytest.raises(_lib.BackendUnavailable):
        P.spp(prof, clu, M)


def test_cluster_validation_fast_and_slow_paths_agree():
    good = P.make_cluster([3, 1, 2], [(1, 2, 1.0), (1, 3, 2.0), (2, 3, 3.0)])
    assert P.validate_cluster(good) is good
    # both orientations of a pair with equal values: legal in the reference (slow path)
    both = P.ClusterGraph((1, 2), {(1, 2): 1.0, (2, 1): 1.0})
    assert P.validate_cluster(both) is both
    cases = [
        (P.ClusterGraph((1, 2, 3), {(1, 2): 1.0, (1, 3): 1.0}), "missing pair"),
        (P.ClusterGraph((1, 2), {(1, 2): 0.0}), "non-positive"),
        (P.ClusterGraph((1, 2), {(1, 5): 1.0}), "unknown GPU"),
        (P.ClusterGraph((1, 2), {(1, 1): 1.0}), "self-link"),
        (P.ClusterGraph((1, 1), {}), "duplicate GPU id"),
        (P.ClusterGraph((1, 2), {(1, 2): 1.0, (2, 1): 2.0}), "asymmetric"),
    ]
    for clu, msg in cases:
        with pytest.raises(P.ValidationError, match=msg):
            P.validate_cluster(clu)


def test_batched_cluster_packing_matches_per_cluster_and_defers_errors():
    """_device.pack_clusters (spp_many's one-pass validation + packing of all
    distinct clusters) gives the per-cluster pack_cluster results, and returns
    None — so the per-instance path raises the reference's first error — when
    any cluster is outside the common valid form."""
    import random
    from paper_2204_10562_b200 import _device, planner
    rng = random.Random(5)
    cls = [c for _, c, _ in W.models_of(W.c4_batch(40))]
    for k in range(20):   # sparse / negative ids take the searchsorted branch
        ids = rng.sample(range(-10 ** 7, 10 ** 7), rng.randrange(2, 12))
        cls.append(P.ClusterGraph(tuple(ids), {(a, b) if a < b else (b, a): rng.uniform(1e9, 1e11)
                                               for i, a in enumerate(ids) for b in ids[i + 1:]}))
    cls.append(P.make_cluster([7], []))
    fast = _device.pack_clusters(cls)
    for (fi, fb), c in zip(fast, cls):
        si, sb = _device.pack_cluster(c)
        assert fi == si and np.array_equal(fb, sb)
    bad = [P.ClusterGraph((1, 2), {(2, 1): 1.0}),          # reversed key: slow path (legal)
           P.ClusterGraph((1, 2), {(1, 2): 0.0}),          # non-positive
           P.ClusterGraph((1, 2), {(1, 5): 1.0}),          # unknown GPU
           P.ClusterGraph((1, 2), {(1, 2): 1e101}),        # outside the numeric domain
           P.ClusterGraph((1, 2, 3), {(1, 2): 1.0, (1, 3): 1.0})]   # missing pair
    for b in bad:
        assert _device.pack_clusters(cls[:3] + [b]) is None
    # spp_many's packing: a bad cluster in the middle raises the per-instance error
    prof, _, M = W.c4_batch(1)[0].to_model()
    with pytest.raises(P.ValidationError, match="non-positive"):
        planner._items([(prof, cls[0], M), (prof, bad[1], M), (prof, cls[1], M)])


def test_lazy_events_behave_like_tuples():
    from paper_2204_10562_b200.model import LazyEvents, ScheduleEvent
    res = [None, "stage1", "chan1", "stage2"]
    lab = [None, "fwd1", "comm_fwd1", "fwdbwd2"]
    ev = LazyEvents(res, lab, np.array([1, 1, 2]), np.array([1, 2, 1]), np.array([0.0, 1.0, 1.0]),
                    np.array([1.0, 2.0, 2.0]))
    want = (ScheduleEvent("stage1", 1, "fwd1", 0.0, 1.0), ScheduleEvent("chan1", 1, "comm_fwd1", 1.0, 2.0),
            ScheduleEvent("stage1", 2, "fwd1", 1.0, 2.0))
    assert len(ev) == 3 and ev[1] == want[1] and ev[-1] == want[2] and ev[0:2] == want[0:2]
    assert ev == want and want == ev and tuple(ev) == want and list(ev) == list(want)
    assert hash(ev) == hash(want)
    s1 = P.Schedule(events=ev, allreduce=(), makespan=2.0)
    s2 = P.Schedule(events=want, allreduce=(), makespan=2.0)
    assert s1 == s2
    other = LazyEvents(res, lab, np.array([1, 1, 2]), np.array([1, 2, 1]), np.array([0.0, 1.0, 1.0]),
                       np.array([1.0, 2.0, 2.5]))
    assert other != ev


def test_baseline_host_planners_match_goldens():
    """gpipe_plan / dataparallel_plan / the flush queues are host bookkeeping:
    checked here against the reference goldens without a GPU."""
    from helpers import load, model_of
    from paper_2204_10562_b200.baselines import gpipe_queues
    for case in load("baselines")["cases"]:
        prof, clu, M = model_of(case["input"])
        o = tuple(case["order"])
        ordering = P.DeviceOrdering(order=o, rank={v: k + 1 for k, v in enumerate(o)})
        for n, *rest in case["gpipe"]:
            if rest[0] == "error":
                with pytest.raises(P.ValidationError, match="infeasible stage count"):
                    P.gpipe_plan(prof, clu, ordering, n, M)
                continue
            plan = P.gpipe_plan(prof, clu, ordering, n, M)
            assert [[s.layer_start, s.layer_end, list(s.devices)] for s in plan.stages] == rest[0]["stages"]
        dp = P.dataparallel_plan(prof, clu, M)
        assert [[s.layer_start, s.layer_end, list(s.devices)] for s in dp.stages] == case["dataparallel"]["stages"]
    for case in load("sim")["cases"]:
        if "gpipe" not in case["name"]:
            continue
        st = case["plan"]["stages"]
        plan = P.Plan(tuple(P.Stage(n + 1, a, b, tuple(d)) for n, (a, b, d) in enumerate(st)), case["plan"]["M"])
        want = {k: tuple(map(tuple, v)) for k, v in case["queues"].items()}
        assert gpipe_queues(plan) == want


def test_lazy_sweep_behaves_like_the_reference_tuple():
    import math
    from paper_2204_10562_b200.planner import LazySweep, SweepEntry
    lz = LazySweep([1, 0, 2], [1.5, 0.0, 2.5], [3.0, 0.0, 4.0], [5.0, 0.0, 6.0])
    want = (SweepEntry(1, True, 1.5, 3.0, 5.0), SweepEntry(2, False, math.inf, None, None),
            SweepEntry(3, True, 2.5, 4.0, 6.0))
    assert len(lz) == 3 and lz == want and want == tuple(lz) and lz[1] == want[1] and lz[-1] == want[-1]
    assert lz[:2] == want[:2] and list(lz) == list(want) and hash(lz) == hash(want)
    assert lz == LazySweep([1, 0, 2], [1.5, 0.0, 2.5], [3.0, 0.0, 4.0], [5.0, 0.0, 6.0])
    assert lz != LazySweep([1, 0, 2], [1.5, 0.0, 2.5], [3.0, 0.0, 4.5], [5.0, 0.0, 6.0])


def test_pipeplan_alias_exposes_the_reference_names():
    """dropin/pipeplan: `import pipeplan` gives the drop-in with every public
    name of the reference package (reference __init__.py:96-174)."""
    import ast
    import subprocess
    import sys
    ref_init = os.path.join(REPO, "baseline", "_ref", "pipeplan", "__init__.py")
    if not os.path.isfile(ref_init):
        pytest.skip("reference not staged under baseline/_ref")
    tree = ast.parse(open(ref_init).read())
    names = next(ast.literal_eval(n.value) for n in tree.body
                 if isinstance(n, ast.Assign) and getattr(n.targets[0], "id", "") == "__all__")
    env = dict(os.environ, PYTHONPATH=os.path.join(REPO, "dropin"))
    code = ("import pipeplan, json, sys; from pipeplan.model import FWD; from pipeplan.cli import main; "
            "import pipeplan.oracle as o; assert o.Plan is pipeplan.Plan; "
            "print(json.dumps([n for n in sys.argv[1:] if not hasattr(pipeplan, n)]), pipeplan.IMPLEMENTATION)")
    r = subprocess.run([sys.executable, "-c", code] + names, env=env, capture_output=True, text=True, cwd="/tmp")
    assert r.returncode == 0, r.stderr
    assert r.stdout.split() == ["[]", "paper_2204_10562_b200"]
