"""Per-call latency of the drop-in's small-instance entry points (the calls the
reference test-suite makes thousands of times), plus a cProfile of a batch of
them.  Run on the GPU box:  python tools/small_call_latency.py"""
import cProfile
import os
import pstats
import random
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "dropin"))
sys.path.insert(0, os.path.join(REPO, "baseline", "_ref", "pipeplan_tests"))
import pipeplan as P  # noqa: E402
from conftest import random_instance  # noqa: E402

P.warmup()
rng = random.Random(5)
insts = [random_instance(rng) for _ in range(200)]


def timeit(name, fn, n=200):
    fn(0)
    t0 = time.perf_counter()
    for k in range(n):
        fn(k)
    dt = (time.perf_counter() - t0) / n
    print(f"{name:28s} {dt * 1e6:9.1f} us/call")


res = [P.spp(*i) for i in insts]
timeit("spp", lambda k: P.spp(*insts[k]))
timeit("simulate_pe", lambda k: P.simulate_pe(res[k].plan, insts[k][0], insts[k][1]))
timeit("simulate_cycle_schedule", lambda k: P.simulate_cycle_schedule(res[k].plan, insts[k][0], insts[k][1]))
timeit("lemma1_bound", lambda k: P.lemma1_bound(res[k].plan, insts[k][0], insts[k][1]))
timeit("validate_schedule", lambda k: P.validate_schedule(res[k].schedule, res[k].plan, insts[k][0], insts[k][1]))
timeit("rdo", lambda k: P.rdo(insts[k][1]))
timeit("phi", lambda k: P.phi(insts[k][0], insts[k][1]))
timeit("PartitionSolver+best(all)", lambda k: [P.PartitionSolver(insts[k][0], insts[k][1], P.rdo(insts[k][1]),
                                                                  insts[k][2]).best_partition(x)
                                               for x in range(1, insts[k][1].num_gpus + 1)])
pr = cProfile.Profile()
pr.enable()
for k in range(100):
    P.simulate_pe(res[k].plan, insts[k][0], insts[k][1])
    P.spp(*insts[k])
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
