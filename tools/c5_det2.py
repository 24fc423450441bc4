"""Which workspace region carries the uninitialised read: fill one region at a time with NaN."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_10562_b200 import _device, _lib, workloads as W  # noqa: E402
from paper_2204_10562_b200.partition import sum_flags  # noqa: E402
L, V, M = (int(x) for x in sys.argv[1:4])


def a16(x):
    return (x + 15) & ~15


def sum_sq(n):
    return n * (n + 1) * (2 * n + 1) // 6


def tet(n):
    return (n + 1) * n * (n - 1) // 6


def layout(L, V):
    o, d = 0, {}
    def reg(name, n):
        nonlocal o
        d[name] = (o, n); o += a16(n)
    reg("prefix", L + 1); reg("psum", L * L); reg("minpair", V * V); reg("cross", V * V * V)
    reg("W", L * sum_sq(V) + 16 * V); reg("X", L * tet(V) + 16 * V * V); reg("rdo_w", V * V)
    reg("rdo_st", (4 * (8 * V + 4) + V * V + 7) // 8)
    reg("rdo_iw", (V - 1) * V * V if V > 128 else 0); reg("rdo_key", 2); reg("dpc", (3 * V + 8 + 1) // 2)
    reg("T1", V * L * L); reg("S", V * L * L)
    return d, o


spec = W.c5_instance(L=L, V=V, M=M)
profile, cluster, _ = spec.to_model()
d, tot = layout(L, V)
ref = None
for region in [None] + list(d):
    db = _device.DeviceBatch([(_device.pack(profile, cluster), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None)],
                             capture_events=False)
    assert db.sizes["ws"] >= tot, (db.sizes["ws"], tot)
    db.d_ws.fill_(0.0)
    if region is not None:
        o, n = d[region]
        if n:
            db.d_ws[o:o + n].fill_(float("nan"))
    db.run("spp"); torch.cuda.synchronize()
    h = db.fetch()
    cur = (h["order"][:V].copy(), h["sweep_r"][:V].copy(), h["sweep_w"][:V].copy())
    if ref is None:
        ref = cur
        print("reference (zero fill) infeasible xi:", list(np.nonzero(cur[1] == 0)[0] + 1)[:8], flush=True)
    else:
        print(f"NaN in {region:8s}: same order {np.array_equal(cur[0], ref[0])} same r {np.array_equal(cur[1], ref[1])} "
              f"same w {np.array_equal(cur[2], ref[2], equal_nan=True)}", flush=True)
    del db; torch.cuda.empty_cache()
