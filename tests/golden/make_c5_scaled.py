"""Down-scaled C5 planning instances (the C5 generator at L x V below the full
1024 x 256) planned by the C oracle — the CPU cannot reach the full size
(T_fact 1.5e12), so the GPU's full-size DP is pinned through these shapes,
which run the same chunked (L > 128) kernels.  The oracle itself is pinned to
the reference's goldens (test_oracle_golden.py), including the 96 x 64 C3
goldens produced by pipeplan.spp.

    python tests/golden/make_c5_scaled.py 256 64 64
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, os.path.join(REPO, "tests"))
import oracle as O  # noqa: E402
from helpers import oracle_instance, spec_from_workload  # noqa: E402
from paper_2204_10562_b200 import workloads as W  # noqa: E402

L, V, M = (int(x) for x in sys.argv[1:4])
spec = spec_from_workload(W.c5_instance(L=L, V=V, M=M))
inst, ids = oracle_instance(spec)
t0 = time.time()
r = O.spp(inst, with_events=False)
h = lambda x: None if x is None else float(x).hex()
case = {"input": spec, "device_order": [ids[k] for k in r["order"]],
        "sweep": [[xi, f, h(w), h(mk), h(bd)] for xi, f, w, mk, bd in r["sweep"]],
        "plan": {"stages": [[a, b, [ids[d] for d in devs]] for a, b, devs in r["frags"]], "M": M},
        "makespan": h(r["makespan"]), "phi": h(r["phi"]), "theorem_factor": h(r["theorem_factor"]),
        "oracle_seconds": time.time() - t0, "generator": "oracle/pipeplan_oracle.c (C restatement of the reference)"}
path = os.path.join(HERE, f"c5_scaled_{L}x{V}_M{M}.json")
json.dump(case, open(path, "w"), separators=(",", ":"))
print(path, case["oracle_seconds"])
