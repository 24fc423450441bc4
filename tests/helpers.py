"""Shared test helpers: fixture loading and conversions (tests only)."""

import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")


def load(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as f:
        return json.load(f)


def fx(h):
    return None if h is None else float.fromhex(h)


def arrays(spec):
    """Raw arrays from a fixture input dict: (fwd, bwd, param, efwd, ebwd, bw[V,V], sorted ids, M)."""
    ids = sorted(spec["gpu_ids"])
    pos = {g: k for k, g in enumerate(ids)}
    V = len(ids)
    bw = np.zeros((V, V))
    for a, b, w in spec["links"]:
        bw[pos[a], pos[b]] = bw[pos[b], pos[a]] = fx(w)
    f = lambda key: np.array([fx(v) for v in spec[key]], dtype=np.float64)
    return f("fwd"), f("bwd"), f("param"), f("efwd"), f("ebwd"), bw, ids, spec["M"]


def oracle_instance(spec, M=None):
    import oracle as O
    fwd, bwd, param, efwd, ebwd, bw, ids, m = arrays(spec)
    return O.Instance(fwd, bwd, param, efwd, ebwd, bw, m if M is None else M), ids


def model_of(spec, M=None):
    """(ModelProfile, ClusterGraph, M) of the product package from a fixture input."""
    from paper_2204_10562_b200.model import InterLayerEdge, LayerProfile, ModelProfile, make_cluster
    layers = tuple(LayerProfile(id=k + 1, fwd_time=fx(a), bwd_time=fx(b), param_bytes=fx(c))
                   for k, (a, b, c) in enumerate(zip(spec["fwd"], spec["bwd"], spec["param"])))
    edges = tuple(InterLayerEdge(src=k + 1, dst=k + 2, fwd_bytes=fx(a), bwd_bytes=fx(b))
                  for k, (a, b) in enumerate(zip(spec["efwd"], spec["ebwd"])))
    prof = ModelProfile(name=spec["name"], microbatch_size=1, layers=layers, edges=edges)
    clu = make_cluster(spec["gpu_ids"], [(a, b, fx(w)) for a, b, w in spec["links"]])
    return prof, clu, spec["M"] if M is None else M


def block_labels(N):
    """position -> (resource, label) following the reference block list J."""
    out = {}
    if N == 1:
        return {1: ("stage1", "fwdbwd1")}
    pos = 1
    for n in range(1, N):
        out[pos] = (f"stage{n}", f"fwd{n}")
        out[pos + 1] = (f"chan{n}", f"comm_fwd{n}")
        pos += 2
    out[pos] = (f"stage{N}", f"fwdbwd{N}")
    pos += 1
    for n in range(N - 1, 0, -1):
        out[pos] = (f"chan{n}", f"comm_bwd{n}")
        out[pos + 1] = (f"stage{n}", f"bwd{n}")
        pos += 2
    return out


def oracle_spp_parallel(specs, threads=None):
    """O.spp over fixture-style specs on a thread pool (the ctypes call
    releases the GIL; the oracle has no global state).  Returns [(want, ids)]."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    import oracle as O
    insts = [oracle_instance(s) for s in specs]
    n = threads or max(1, min(len(insts), len(os.sched_getaffinity(0)), 32))
    # the oracle's dense DP table is ~V^3 L * 13 bytes per instance (0.33 GB at
    # 96 x 64): keep the concurrent ones within half the host's free memory
    per = max(13 * max(t[0].V for t in insts) ** 3 * max(t[0].L for t in insts), 1)
    try:
        free = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
        n = max(1, min(n, int(0.5 * free // per)))
    except (ValueError, OSError):
        pass
    with ThreadPoolExecutor(n) as ex:
        outs = list(ex.map(lambda t: O.spp(t[0]), insts))
    return [(w, ids) for w, (_, ids) in zip(outs, insts)]


def spec_from_workload(w):
    """Fixture-style input dict (floats as hex) from a workloads.InstanceSpec."""
    h = lambda xs: [float(x).hex() for x in xs]
    return {"name": w.name, "fwd": h(w.fwd), "bwd": h(w.bwd), "param": h(w.param), "efwd": h(w.efwd),
            "ebwd": h(w.ebwd), "gpu_ids": list(w.gpu_ids), "links": [[a, b, float(x).hex()] for a, b, x in w.links],
            "M": w.M}
