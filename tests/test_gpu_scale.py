"""GPU parity at the BASELINE.json config sizes beyond C3 (C4 batch, C5 simulation).

Bit-exact against the C oracle on samples, plus size-independent properties
on the full batches.
"""

import numpy as np
import pytest

import oracle as O
from helpers import block_labels

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2204_10562_b200")
from paper_2204_10562_b200 import workloads as W  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _oinst(spec):
    ids = sorted(spec.gpu_ids)
    pos = {g: k for k, g in enumerate(ids)}
    bw = np.zeros((len(ids), len(ids)))
    for a, b, w in spec.links:
        bw[pos[a], pos[b]] = bw[pos[b], pos[a]] = w
    return O.Instance(spec.fwd, spec.bwd, spec.param, spec.efwd, spec.ebwd, bw, spec.M), ids


def test_c4_full_batch_sampled_vs_oracle():
    specs = W.c4_batch(4096)
    res = P.spp_many([s.to_model() for s in specs])
    assert len(res) == 4096
    for r in res:   # properties on every instance
        feas = [e for e in r.sweep if e.feasible]
        assert r.makespan == min(e.makespan for e in feas)
        assert all(e.makespan <= e.bound * (1 + 1e-9) for e in feas)
        assert sorted(r.device_order) == list(range(1, 17))
        assert len(r.schedule.events) == r.plan.microbatch_count * (4 * r.plan.num_stages - 3)
    for k in range(0, 4096, 64):   # 64 instances bit-exact vs the oracle
        inst, ids = _oinst(specs[k])
        want = O.spp(inst)
        r = res[k]
        assert list(r.device_order) == [ids[x] for x in want["order"]]
        assert [(e.stage_count, e.feasible, e.workload, e.makespan, e.bound) for e in r.sweep] == want["sweep"]
        assert r.makespan == want["makespan"]
        bl = block_labels(r.plan.num_stages)
        assert [(e.microbatch, e.block, e.start, e.end) for e in r.schedule.events] == \
            [(m, bl[p][1], s, e) for m, p, s, e in want["events"]]


def test_c5_candidate_simulation_vs_oracle():
    spec = W.c5_instance()
    profile, cluster, M = spec.to_model()
    order = P.rdo(cluster).order
    inst, ids = _oinst(spec)
    assert [ids[x] for x in O.rdo(inst)] == list(order)
    plans, oplans = [], []
    pos = {g: k for k, g in enumerate(ids)}
    for xi in range(1, 257):
        st = W.even_split_plan(spec.L, order, xi)
        plans.append(P.Plan(tuple(P.Stage(n + 1, a, b, d) for n, (a, b, d) in enumerate(st)), M))
        oplans.append(O.Plan([(a, b, tuple(pos[g] for g in d)) for a, b, d in st], M))
    import torch
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    got = P.simulate_pe_many(plans, profile, cluster)
    # caller-plan simulation allocates no DP workspace (68 GB at 1024 x 256)
    assert torch.cuda.max_memory_allocated() - base < 1 << 30
    want = O.simulate_pe_batch(inst, oplans, 16)
    assert [m for m, _ in got] == list(want)
    best = min(range(256), key=lambda k: (got[k][0], k))
    assert best + 1 == min(range(256), key=lambda k: (want[k], k)) + 1
    for k in (0, 59, 255):
        assert got[k][1] == O.lemma1_bound(inst, oplans[k])


def test_c5_scaled_chunked_dp_vs_oracle_golden():
    """The C5 generator at 256 layers x 64 GPUs (L > 128: the chunked DP kernels
    that also run the full 1024 x 256 C5 DP) against the oracle's result
    (tests/golden/make_c5_scaled.py; 237 s of the C oracle)."""
    import glob
    import os
    from helpers import GOLDEN, load, model_of
    paths = sorted(glob.glob(os.path.join(GOLDEN, "c5_scaled_*.json")))
    assert paths
    h = lambda x: None if x is None else float(x).hex()
    for path in paths:
        c = load(os.path.basename(path)[:-5])
        r = P.spp(*model_of(c["input"]))
        assert list(r.device_order) == c["device_order"]
        assert [[e.stage_count, e.feasible, h(e.workload), h(e.makespan), h(e.bound)] for e in r.sweep] == c["sweep"]
        assert [[s.layer_start, s.layer_end, list(s.devices)] for s in r.plan.stages] == c["plan"]["stages"]
        assert (h(r.makespan), h(r.phi), h(r.theorem_factor)) == (c["makespan"], c["phi"], c["theorem_factor"])


def test_batch_without_workspace_serves_simulation_only():
    """DeviceBatch(workspace=False) (pp_batch.ws = NULL): pp_phi and pp_simulate
    run; RDO, the DP, the sweep and the select+replay refuse instead of touching
    a NULL workspace."""
    from paper_2204_10562_b200 import _device
    from paper_2204_10562_b200.partition import sum_flags
    spec = W.c4_batch(1)[0]
    profile, cluster, M = spec.to_model()
    db = _device.DeviceBatch([(_device.pack(profile, cluster), M, sum_flags(), None)], capture_events=True,
                             workspace=False)
    assert db.d_ws is None
    db.run("phi")
    assert db.fetch()["phi"][0] == P.phi(profile, cluster)
    for what in ("rdo", "prm", "sweep", "select", "spp"):
        with pytest.raises(RuntimeError, match="ws is NULL"):
            db.run(what)
