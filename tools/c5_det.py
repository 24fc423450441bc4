"""Determinism / uninitialised-read probe of the chunked DP: plan the same
instance with the workspace pre-filled by different garbage and compare."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_10562_b200 import _device, _lib, workloads as W  # noqa: E402
from paper_2204_10562_b200.partition import sum_flags  # noqa: E402
L, V, M = (int(x) for x in sys.argv[1:4])
spec = W.c5_instance(L=L, V=V, M=M)
profile, cluster, _ = spec.to_model()
outs = []
for fill in (0.0, float("nan"), -1.0, float("inf")):
    db = _device.DeviceBatch([(_device.pack(profile, cluster), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None)],
                             capture_events=False)
    db.d_ws.fill_(fill)
    db.run("spp"); torch.cuda.synchronize()
    h = db.fetch()
    outs.append((fill, h["sweep_r"][:V].copy(), h["sweep_w"][:V].copy(), int(h["best_xi"][0]), float(h["best_mk"][0])))
    del db; torch.cuda.empty_cache()
for f, r, w, bx, mk in outs:
    bad = np.nonzero(r == 0)[0]
    print(f"fill {f}: best xi {bx} mk {mk!r} infeasible xi {list(bad + 1)[:10]} "
          f"same_r {np.array_equal(r, outs[0][1])} same_w {np.array_equal(w, outs[0][2], equal_nan=True)}")
