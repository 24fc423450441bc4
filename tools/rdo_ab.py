"""RDO phase time vs speculative rounds (GPU only): python tools/rdo_ab.py [n ...]."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_10562_b200 import _device, _lib, workloads as W  # noqa: E402
from paper_2204_10562_b200.partition import sum_flags  # noqa: E402

for n in [int(x) for x in sys.argv[1:]] or [12, 1]:
    specs = (W.c3_sweep() * 8)[:n] if n > 0 else W.c4_batch(-n)
    items = [(_device.pack(p, c), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for p, c, M in W.models_of(specs)]
    db = _device.DeviceBatch(items, capture_events=True)
    for rounds in (0, 1, 2, 3, 4):
        _lib.rdo_rounds(rounds)
        db.run("rdo"); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); db.run("rdo"); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"n={n:3d} rounds={rounds}: rdo {min(ts):.3f} ms")
    _lib.rdo_rounds(1)
