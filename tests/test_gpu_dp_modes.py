"""Persistent dependency-driven DP (dp_persist.cu) vs the launch-per-step wavefront.

Both schedules evaluate the same fp64 expressions over the same min/max sets,
so every SppResult (plans, workloads, makespans, events) and every
PartitionSolver cell must be identical; the oracle pins both.
"""

import math
import random

import pytest

import oracle as O
from helpers import model_of, oracle_instance

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2204_10562_b200")
from paper_2204_10562_b200 import _lib, workloads as W  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    _lib.load()


@pytest.fixture
def persistent():
    prev = _lib.dp_persistent(0)
    yield _lib.dp_persistent
    _lib.dp_persistent(prev)


def test_default_mode_is_auto():
    prev = _lib.dp_persistent(2)
    assert prev == 2
    _lib.dp_persistent(prev)


@pytest.fixture
def early_exit():
    prev = _lib.dp_early_exit(True)
    yield _lib.dp_early_exit
    _lib.dp_early_exit(prev)


@pytest.mark.parametrize("mode", [(True, 0), (True, 3), (False, 3), (True, 2)])
def test_early_exit_identical(persistent, early_exit, mode):
    """Per-step schedule with every candidate folded (no early exit) vs early
    exit on / off in each schedule: identical results."""
    rng = random.Random(99)
    specs = _rand_specs(rng, 30, 60, 20) + [W.c3_gpt96(M=64, jitter_seed=3), W.c2_bert24()] + W.c4_batch(4)
    models = [s.to_model() for s in specs]
    persistent(0); early_exit(False)
    ref = P.spp_many(models)
    persistent(mode[1]); early_exit(mode[0])
    got = P.spp_many(models)
    for s, x, y in zip(specs, ref, got):
        assert x == y, (s.name, mode)


def _rand_specs(rng, n, Lmax, Vmax, Mmax=32):
    out = []
    lu = lambda lo, hi: math.exp(rng.uniform(math.log(lo), math.log(hi)))
    for k in range(n):
        L, V, M = rng.randint(1, Lmax), rng.randint(1, Vmax), rng.randint(1, Mmax)
        ids = rng.sample(range(1, 1000), V)
        out.append(W.InstanceSpec(f"r{k}", [lu(1e-3, 1.0) for _ in range(L)], [lu(1e-3, 2.0) for _ in range(L)],
                                  [lu(1e6, 1e10) for _ in range(L)], [lu(1e5, 1e9) for _ in range(L - 1)],
                                  [lu(1e5, 1e9) for _ in range(L - 1)], ids,
                                  [(a, b, lu(1e8, 1e11)) for i, a in enumerate(ids) for b in ids[i + 1:]], M))
    return out


def _both(persistent, specs, modes=(3, 0)):
    models = [s.to_model() for s in specs]
    out = []
    for m in modes:
        persistent(m)
        out.append(P.spp_many(models))
    return out


def test_instance_per_cta_identical(persistent):
    """One CTA per instance (mode 3, auto for >= 2 x SMs instances) vs per-step."""
    rng = random.Random(4242)
    specs = _rand_specs(rng, 40, 50, 20) + W.c4_batch(12) + [W.c2_bert24(), W.c1_vgg19()]
    specs += [W.c3_gpt96(M=16, nodes=2, per_node=8), W.c3_gpt96(M=8)]
    a, b = _both(persistent, specs, modes=(3, 0))
    for s, x, y in zip(specs, a, b):
        assert x == y, s.name


def test_c4_auto_batch_matches_oracle():
    """A C4-size batch (auto picks instance-per-CTA): every 64th instance vs the oracle."""
    specs = W.c4_batch(512)
    res = P.spp_many(W.models_of(specs))
    for k in range(0, 512, 64):
        s = specs[k]
        want = O.spp(O.Instance(s.fwd, s.bwd, s.param, s.efwd, s.ebwd, _bw(s), s.M), with_events=False)
        assert res[k].makespan == want["makespan"], k
        assert [(e.stage_count, e.feasible, e.workload, e.makespan, e.bound) for e in res[k].sweep] == \
            [tuple(x) for x in want["sweep"]], k


def test_mode_values_checked():
    with pytest.raises(Exception, match="DP schedule 1"):
        _lib.dp_persistent(1)
    assert _lib.dp_persistent(2) == 2


def test_mixed_batch_modes_identical(persistent):
    """Ragged batch: instances far below the batch maxima exercise the skipped tasks."""
    rng = random.Random(31337)
    specs = _rand_specs(rng, 60, 40, 24) + [W.c2_bert24(), W.c1_vgg19()] + W.c4_batch(6)
    specs += [W.c3_gpt96(M=16, nodes=3, per_node=8)]
    a, b = _both(persistent, specs)
    for s, x, y in zip(specs, a, b):
        assert x == y, s.name


def test_c3_modes_identical_and_match_oracle(persistent):
    specs = [W.c3_gpt96(M=32), W.c3_gpt96(M=128, jitter_seed=5)]
    a, b = _both(persistent, specs)
    for s, x, y in zip(specs, a, b):
        assert x == y, s.name
        inst = O.Instance(s.fwd, s.bwd, s.param, s.efwd, s.ebwd, _bw(s), s.M)
        want = O.spp(inst, with_events=False)
        assert x.makespan == want["makespan"]
        assert [e.workload for e in x.sweep] == [w for _, _, w, _, _ in want["sweep"]]


def _bw(s):
    import numpy as np
    ids = sorted(s.gpu_ids)
    pos = {g: k for k, g in enumerate(ids)}
    bw = np.zeros((len(ids), len(ids)))
    for a, b, w in s.links:
        bw[pos[a], pos[b]] = bw[pos[b], pos[a]] = w
    return bw


@pytest.mark.parametrize("allow", [True, False])
def test_partition_solver_cells_modes_identical(persistent, allow):
    rng = random.Random(5 + allow)
    for s in _rand_specs(rng, 6, 30, 20):
        prof, clu, M = s.to_model()
        order = P.rdo(clu)
        cells = [(l, x, r, i) for i in range(1, s.V + 1) for r in range(1, i + 1)
                 for x in range(1, i + 1) for l in range(1, s.L + 1) if (l + x + r + i) % 3 == 0]
        got = {}
        for mode in (3, 0):
            persistent(mode)
            solver = P.PartitionSolver(prof, clu, order, M, allow_replication=allow)
            got[mode] = [(g.workload, g.stages) for g in solver.solve_many(cells)]
        assert got[3] == got[0], s.name


def test_graph_replay_across_batches(persistent):
    """The per-step DP is replayed from a CUDA graph cached per batch shape (its
    descriptors rewritten before each replay); batches of one shape with
    different data and buffers (and repeated runs) must each give their own,
    exact results."""
    from paper_2204_10562_b200 import _device, planner
    specs_a = [W.c3_gpt96(M=m, nodes=2, per_node=8) for m in (8, 32, 128)]
    specs_b = [W.c3_gpt96(M=m, jitter_seed=11, nodes=2, per_node=8) for m in (8, 32, 128)]
    persistent(3)
    want_a = P.spp_many([s.to_model() for s in specs_a])
    want_b = P.spp_many([s.to_model() for s in specs_b])
    persistent(0)
    for specs, want in ((specs_a, want_a), (specs_b, want_b), (specs_a, want_a)):
        models = [s.to_model() for s in specs]
        items, packs = planner._items(models)
        db = _device.DeviceBatch(items, capture_events=True)
        for _ in range(2):   # first run may capture, second replays
            db.run("spp")
            h = db.fetch()
            got = [planner._decode(db, h, k, items[k][1], packs[k]) for k in range(len(items))]
            assert got == want
        del db


@pytest.mark.parametrize("early", [True, False])
def test_crossing_search_combine_identical(early_exit, early):
    """Per-step combine: crossing search (default) vs the exhaustive register
    tiles, with and without the monotonicity certificates in use: identical
    results on random, C2, C3 (full 96 x 64, uniform and jittered) and C4."""
    rng = random.Random(1234)
    specs = (_rand_specs(rng, 40, 60, 24) + [W.c2_bert24(), W.c3_gpt96(M=8), W.c3_gpt96(M=256, jitter_seed=7)]
             + W.c4_batch(6))
    models = [s.to_model() for s in specs]
    prev = _lib.dp_combine(0)
    assert prev == 2
    try:
        early_exit(True)
        ref = P.spp_many(models)
        _lib.dp_combine(1)
        early_exit(early)
        got = P.spp_many(models)
        one = [P.spp(*m) for m in models[-8:]]   # single-instance path (split critical chain)
    finally:
        _lib.dp_combine(prev)
    for s, x, y in zip(specs, ref, got):
        assert x == y, s.name
    assert one == ref[-8:]
