"""Process start-up: CUDA context, library load and first launch of every kernel.

The reference is pure Python and has no start-up cost; this package's first
planning call in a process pays for CUDA context creation, loading
libpipeplan_b200.so and lazy module loading of each kernel (~1 s on a fresh
B200 box).  Latency-sensitive callers (a planning service, a test-suite with
per-test deadlines) call :func:`warmup` once at start-up.
"""


def warmup() -> None:
    from .baselines import gpipe_plan, gpipe_schedule
    from .checker import validate_schedule
    from .cost import cost_summary
    from .model import InterLayerEdge, LayerProfile, ModelProfile, make_cluster
    from .ordering import rdo
    from .planner import spp
    from .scheduler import lemma1_bound, simulate_cycle_schedule, simulate_pe

    layers = tuple(LayerProfile(k, 1.0, 2.0, 1e8) for k in (1, 2, 3))
    edges = (InterLayerEdge(1, 2, 1e8, 1e8), InterLayerEdge(2, 3, 1e8, 1e8))
    profile = ModelProfile("warmup", 1, layers, edges)
    cluster = make_cluster([1, 2, 3], [(1, 2, 1e9), (1, 3, 2e9), (2, 3, 1e9)])
    r = spp(profile, cluster, 3)
    validate_schedule(r.schedule, r.plan, profile, cluster)
    simulate_pe(r.plan, profile, cluster)
    simulate_cycle_schedule(r.plan, profile, cluster)
    lemma1_bound(r.plan, profile, cluster)
    cost_summary(r.plan, profile, cluster)
    gp = gpipe_plan(profile, cluster, rdo(cluster), 2, 3)
    validate_schedule(gpipe_schedule(gp, profile, cluster), gp, profile, cluster, forward_barrier=True)
