"""Timeline of the persistent DP kernel on the C3 batch (debug tool, GPU only).

    python tools/dp_trace.py [n_instances]

Prints, per task kind, the count, mean wait (fetch -> inputs ready) and mean
compute (ready -> end), the CTA-time split, and the critical chain's step times.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_10562_b200 import _device, _lib  # noqa: E402
from paper_2204_10562_b200 import workloads as W  # noqa: E402
from paper_2204_10562_b200.partition import sum_flags  # noqa: E402

KINDS = {1: "E1", 2: "Eb", 3: "C1", 4: "Cb"}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    specs = (W.c3_sweep() * 4)[:n]
    models = W.models_of(specs)
    items = [(_device.pack(p, c), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for p, c, M in models]
    db = _device.DeviceBatch(items, capture_events=True)
    lib = _lib.load()
    cap = 1 << 20
    buf = torch.zeros(4 * cap, dtype=torch.int64, device="cuda")
    db.run("spp")
    torch.cuda.synchronize()
    db.run("phi"); db.run("rdo")
    torch.cuda.synchronize()
    _lib.check(lib.pp_dp_trace(buf.data_ptr(), cap))
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); db.run("prm"); b.record()
    torch.cuda.synchronize()
    _lib.check(lib.pp_dp_trace(None, 0))
    print(f"prm phase {a.elapsed_time(b):.3f} ms for {n} instances")
    tr = buf.view(-1, 4).cpu().numpy().astype(np.uint64)
    used = tr[:, 3] != 0
    ids = np.nonzero(used)[0]
    tr = tr[used].astype(np.int64)
    kind = (tr[:, 0] & 0xffffffff).astype(int)
    sm = (tr[:, 0] >> 32).astype(int)
    t0 = tr[:, 1].min()
    fetch = (tr[:, 1] - t0) / 1e3
    ready = np.where(tr[:, 2] > 0, (tr[:, 2] - t0) / 1e3, fetch)
    end = (tr[:, 3] - t0) / 1e3
    span = end.max()
    print(f"kernel span {span:.1f} us, {len(ids)} tasks with work, {len(np.unique(sm))} SMs")
    for k, nm in KINDS.items():
        m = kind == k
        if m.any():
            w, c = ready[m] - fetch[m], end[m] - ready[m]
            print(f"  {nm}: {m.sum():6d} tasks  wait mean {w.mean():7.2f} us (sum {w.sum() / 1e3:8.2f} ms)  "
                  f"compute mean {c.mean():7.2f} us (sum {c.sum() / 1e3:8.2f} ms)  max {c.max():7.1f}")
    busy = (end - ready).sum()
    wait = (ready - fetch).sum()
    print(f"CTA-time: compute {busy / 1e3:.2f} ms, waiting {wait / 1e3:.2f} ms; "
          f"CTA-slots x span = {len(np.unique(sm)) * 2 * span / 1e3:.2f} ms")
    # progress over time: fraction of compute in 10 bins
    bins = np.linspace(0, span, 11)
    for lo, hi in zip(bins[:-1], bins[1:]):
        c = np.clip(np.minimum(end, hi) - np.maximum(ready, lo), 0, None).sum()
        w = np.clip(np.minimum(ready, hi) - np.maximum(fetch, lo), 0, None).sum()
        print(f"  [{lo:7.1f},{hi:7.1f}) us: compute CTAs {c / (hi - lo):6.1f}  waiting CTAs {w / (hi - lo):6.1f}")


if __name__ == "__main__":
    main()
