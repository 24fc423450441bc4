"""A/B timing of the DP schedules on the C3 batch (GPU only; results are identical).

    python tools/dp_ab.py [n_instances ...]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_10562_b200 import _device, _lib  # noqa: E402
from paper_2204_10562_b200 import workloads as W  # noqa: E402
from paper_2204_10562_b200.partition import sum_flags  # noqa: E402


def prm_ms(db, reps=5):
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    best = []
    for _ in range(reps):
        db.run("phi"); db.run("rdo")
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); db.run("prm"); b.record()
        torch.cuda.synchronize()
        best.append(a.elapsed_time(b))
    return min(best), sorted(best)[len(best) // 2]


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [12, 1]
    for n in sizes:
        specs = (W.c3_sweep() * 64)[:n] if n > 0 else W.c4_batch(-n)
        items = [(_device.pack(p, c), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None)
                 for p, c, M in W.models_of(specs)]
        db = _device.DeviceBatch(items, capture_events=True)
        for mode in [int(m) for m in os.environ.get('MODES', '0,3').split(',')]:
            for ee in (True, False):
                _lib.dp_persistent(mode); _lib.dp_early_exit(ee)
                db.run("spp"); torch.cuda.synchronize()
                mn, med = prm_ms(db)
                print(f"n={n:4d} mode={mode} early_exit={ee!s:5}: prm {mn:7.3f} ms (median {med:7.3f})")
        _lib.dp_persistent(2); _lib.dp_early_exit(True)


if __name__ == "__main__":
    main()
