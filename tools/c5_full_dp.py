"""C5 full planning DP on the GPU (SURVEY.md §7 stretch):
spp over a 1024-layer chain on a 256-GPU clique, M = 512 — the whole PRM DP
(T_fact = 1.47e12 factored candidates), RDO, the 256-plan sweep and selection.
Workspace ~74 GB of HBM.  Prints per-phase device times and the result.

    python tools/c5_full_dp.py [L V M]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_10562_b200 import _device, _lib, workloads as W  # noqa: E402
from paper_2204_10562_b200.partition import sum_flags  # noqa: E402

L, V, M = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (1024, 256, 512)


def t_fact(L, V):
    tot = 0
    for xi in range(2, min(L, V) + 1):
        A, K = L - xi + 1, V - xi + 1
        tot += A * K * (K + 1) * (K + 2) // 6 + A * (A + 1) // 2 * K * (K + 1) // 2
    return tot


spec = W.c5_instance(L=L, V=V, M=M)
profile, cluster, _ = spec.to_model()
t0 = time.time()
db = _device.DeviceBatch([(_device.pack(profile, cluster), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None)],
                         capture_events=False)
print(f"workspace {db.sizes['ws'] * 8 / 1e9:.1f} GB, setup {time.time() - t0:.1f} s", flush=True)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
ev[0].record(); db.run("phi"); ev[1].record(); db.run("rdo"); ev[2].record(); db.run("prm"); ev[3].record()
db.run("sweep"); ev[4].record(); db.run("select"); ev[5].record()
torch.cuda.synchronize()
ms = {nm: ev[k].elapsed_time(ev[k + 1]) for k, nm in enumerate(("phi", "rdo", "dp", "sweep", "select"))}
h = db.fetch()
tf = t_fact(L, V)
out = {"L": L, "V": V, "M": M, "phase_ms": ms, "t_fact": tf, "dp_minmax_ops_per_s": 2 * tf / (ms["dp"] / 1e3),
       "best_xi": int(h["best_xi"][0]), "best_makespan": float(h["best_mk"][0]),
       "feasible_xi": int((h["sweep_r"][:V] > 0).sum())}
print(json.dumps(out), flush=True)
