"""Speculative RDO (rdo.cu) vs the reference goldens and the C oracle.

The speculative rounds only decide which exact cuts are computed in
parallel, so the order must equal the reference's for every round count —
including clusters whose recursion tree is not a chain (prediction misses),
ties everywhere (uniform bandwidths) and V > 128 (global-memory cut scratch).
"""

import random

import numpy as np
import pytest

import oracle as O
from helpers import fx, load

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2204_10562_b200")
from paper_2204_10562_b200 import _lib, spp_many, workloads as W  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    _lib.load()


@pytest.fixture
def rounds():
    prev = _lib.rdo_rounds(3)
    yield _lib.rdo_rounds
    _lib.rdo_rounds(prev)


def oracle_order(ids, links):
    ids = sorted(ids)
    pos = {g: k for k, g in enumerate(ids)}
    V = len(ids)
    bw = np.zeros((V, V))
    for a, b, w in links:
        bw[pos[a], pos[b]] = bw[pos[b], pos[a]] = w
    one = np.ones(1)
    inst = O.Instance(one, one, one, np.zeros(0), np.zeros(0), bw, 1)
    return tuple(ids[k] for k in O.rdo(inst))


def clique(ids, fn):
    return [(a, b, fn(a, b)) for i, a in enumerate(ids) for b in ids[i + 1:]]


def clusters():
    rng = random.Random(2204)
    out = []
    for nodes, per in ((8, 8), (4, 4), (3, 5), (2, 2), (5, 3), (16, 8), (6, 7)):
        ids, links = W.two_tier_cluster(nodes, per)
        out.append((f"tier{nodes}x{per}", ids, links))
    spec = W.c2_bert24()
    out.append(("dgx1", spec.gpu_ids, spec.links))
    for V in (2, 3, 5, 8, 13, 16, 31, 32, 33, 47, 64, 65, 100):
        ids = list(range(1, V + 1))
        out.append((f"rand{V}", ids, clique(ids, lambda a, b: W._logu(rng, 1e8, 1e11))))
    for V in (7, 24, 64):   # every cut ties: the first-found rules decide everything
        ids = list(range(1, V + 1))
        out.append((f"uniform{V}", ids, clique(ids, lambda a, b: 25e9)))
    # two dense blocks joined weakly: balanced splits, so chain predictions miss
    ids = list(range(1, 41))
    out.append(("blocks", ids, clique(ids, lambda a, b: 100e9 if (a <= 17) == (b <= 17) else rng.uniform(1e9, 2e9))))
    # tree prediction (rdo.cu): three tiers, uneven nodes, a block cut that ties a
    # singleton peel exactly, maximum-bandwidth links forming a path
    ids = list(range(1, 33))
    out.append(("tier3", ids, clique(ids, lambda a, b: 450e9 if (a - 1) // 4 == (b - 1) // 4 else
                                      (50e9 if (a - 1) // 16 == (b - 1) // 16 else 12.5e9))))
    sizes = (2, 3, 5, 8, 1, 4)
    node = [k for k, n in enumerate(sizes) for _ in range(n)]
    ids = list(range(1, len(node) + 1))
    out.append(("uneven-nodes", ids, clique(ids, lambda a, b: 300e9 if node[a - 1] == node[b - 1] else 10e9)))
    ids = list(range(1, 7))   # pairs: a GPU's degree 40 + 4 x 10 equals a pair's cut 2 x 4 x 10
    out.append(("tie-pairs", ids, clique(ids, lambda a, b: 40e9 if (a - 1) // 2 == (b - 1) // 2 else 10e9)))
    ids = list(range(1, 13))
    out.append(("max-path", ids, clique(ids, lambda a, b: 100e9 if abs(a - b) == 1 and a <= 8 and b <= 8 else 5e9)))
    # non-contiguous ids, shuffled per-node structure
    ids = [3 * k + 7 for k in range(30)]
    grp = {g: rng.randrange(4) for g in ids}
    out.append(("sparse-ids", ids, clique(ids, lambda a, b: 300e9 if grp[a] == grp[b] else rng.choice((10e9, 12e9)))))
    return out


@pytest.mark.parametrize("n_rounds", [0, 1, 2, 3, 8])
def test_rdo_every_round_count_matches_oracle(rounds, n_rounds):
    rounds(n_rounds)
    for name, ids, links in clusters():
        got = P.rdo(P.make_cluster(ids, links)).order
        assert got == oracle_order(ids, links), (name, n_rounds)


def test_rdo_goldens_with_speculation(rounds):
    for n_rounds in (1, 3):
        rounds(n_rounds)
        for case in load("ordering")["rdo"]:
            clu = P.make_cluster(case["gpu_ids"], [(a, b, fx(w)) for a, b, w in case["links"]])
            assert list(P.rdo(clu).order) == case["order"]


def test_rdo_global_scratch_path(rounds):
    """V > 128: contracted weights per chain item live in the workspace."""
    rng = random.Random(7)
    ids, links = W.two_tier_cluster(18, 8)   # V = 144
    rand = list(range(1, 161))
    cases = [("tier18x8", ids, links),
             ("rand160", rand, clique(rand, lambda a, b: W._logu(rng, 1e8, 1e11)))]
    for n_rounds in (0, 3):
        rounds(n_rounds)
        for name, i, l in cases:
            assert P.rdo(P.make_cluster(i, l)).order == oracle_order(i, l), (name, n_rounds)


def test_spp_batch_orders_with_speculation(rounds):
    """spp_many over mixed clusters (C3, C4 random, C2): orders equal the oracle's."""
    specs = [W.c3_gpt96(8), W.c2_bert24()] + W.c4_batch(24)
    for n_rounds in (0, 3):
        rounds(n_rounds)
        res = spp_many(W.models_of(specs))
        for s, r in zip(specs, res):
            assert r.device_order == oracle_order(s.gpu_ids, s.links), (s.name, n_rounds)


def test_batch_dedup_of_identical_clusters():
    """A batch that plans one cluster many times (the C3 shape) runs RDO once
    per distinct bandwidth matrix (k_rdo_hash / k_rdo_rep / k_rdo_copy).
    Duplicates with different GPU ids, a near-duplicate differing in one
    bandwidth by one ulp, and a different V of the same data must all get
    their own correct order."""
    import math
    rng = random.Random(7)
    ids, links = W.two_tier_cluster(4, 4)
    base = W.c3_gpt96(M=8, L=6, nodes=4, per_node=4)
    specs = []
    for k in range(5):
        s = base.with_m(8 + k)
        specs.append(s)
    # same matrix, other (sorted-equivalent) ids: positions, not ids, decide the order
    shifted = [g + 100 for g in ids]
    specs.append(W.InstanceSpec("shift", base.fwd, base.bwd, base.param, base.efwd, base.ebwd, shifted,
                                [(a + 100, b + 100, w) for a, b, w in links], 8))
    # one ulp off on one pair
    near = list(links)
    a, b, w = near[3]
    near[3] = (a, b, math.nextafter(w, math.inf))
    specs.append(W.InstanceSpec("near", base.fwd, base.bwd, base.param, base.efwd, base.ebwd, ids, near, 8))
    # random clusters interleaved
    for k in range(4):
        rids = rng.sample(range(1, 500), 16)
        specs.append(W.InstanceSpec(f"rand{k}", base.fwd, base.bwd, base.param, base.efwd, base.ebwd, rids,
                                    clique(rids, lambda x, y: math.exp(rng.uniform(20, 25))), 8))
    specs.append(base.with_m(99))
    prev = _lib.rdo_dedup(2)
    try:
        res = spp_many([s.to_model() for s in specs])
    finally:
        _lib.rdo_dedup(prev)
    for s, r in zip(specs, res):
        assert r.device_order == oracle_order(s.gpu_ids, s.links), s.name


def test_batch_dedup_hash_table_many_instances():
    """Hundreds of instances drawn from a few clusters in shuffled order: the
    open-addressing table (one slot per instance, k_rdo_insert) must map every
    duplicate to a representative with the same matrix."""
    import math
    rng = random.Random(11)
    base = W.c3_gpt96(M=8, L=6, nodes=2, per_node=4)
    pool = []
    for k in range(6):
        rids = list(range(1, 9))
        pool.append((rids, clique(rids, lambda x, y: math.exp(rng.uniform(20, 25)))))
    pool.append(W.two_tier_cluster(2, 4))
    specs = []
    for k in range(400):
        ids, links = pool[rng.randrange(len(pool))]
        specs.append(W.InstanceSpec(f"i{k}", base.fwd, base.bwd, base.param, base.efwd, base.ebwd, ids, links, 8))
    prev = _lib.rdo_dedup(2)
    try:
        res = spp_many([s.to_model() for s in specs])
    finally:
        _lib.rdo_dedup(prev)
    want = {id(l): oracle_order(i, l) for i, l in pool}
    for s, r in zip(specs, res):
        assert r.device_order == want[id(s.links)], s.name
