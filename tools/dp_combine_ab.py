"""DP time (pp_prm) per combine kernel kind and batch size, one process (GPU only):
    python tools/dp_combine_ab.py [n ...]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_10562_b200 import _device, _lib  # noqa: E402
from paper_2204_10562_b200 import workloads as W  # noqa: E402
from paper_2204_10562_b200.partition import sum_flags  # noqa: E402

ns = [int(x) for x in sys.argv[1:]] or [1, 12]
for n in ns:
    specs = (W.c3_sweep() * 64)[:n] if n > 2 else [W.c3_gpt96(M=32), W.c3_gpt96(M=64, jitter_seed=96)][:n]
    items = [(_device.pack(p, c), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for p, c, M in W.models_of(specs)]
    db = _device.DeviceBatch(items, capture_events=True)
    for kind in (0, 1, 0, 1):
        _lib.dp_combine(kind)
        db.run("phi"); db.run("rdo"); db.run("prm"); torch.cuda.synchronize()
        ts = []
        for _ in range(7):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); db.run("prm"); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"n={n:3d} combine={'bis' if kind else 'tiles'} dp min {min(ts):.3f} ms median {sorted(ts)[3]:.3f}",
              flush=True)
    _lib.dp_combine(2)
