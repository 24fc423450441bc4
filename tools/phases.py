"""Per-phase device time of one spp batch (GPU only): python tools/phases.py c3|c4 [n]."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_10562_b200 import _device, _lib  # noqa: E402
from paper_2204_10562_b200 import workloads as W  # noqa: E402
from paper_2204_10562_b200.partition import sum_flags  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else (12 if wl == "c3" else 4096)
specs = (W.c3_sweep() * 64)[:n] if wl == "c3" else W.c4_batch(n)
items = [(_device.pack(p, c), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for p, c, M in W.models_of(specs)]
db = _device.DeviceBatch(items, capture_events=True)
db.run("spp"); torch.cuda.synchronize()
for rep in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    ev[0].record(); db.run("phi"); ev[1].record(); db.run("rdo"); ev[2].record(); db.run("prm"); ev[3].record()
    db.run("sweep"); ev[4].record(); db.run("select"); ev[5].record(); db.run("spp"); ev[6].record()
    torch.cuda.synchronize()
    names = ("phi", "rdo", "prm", "sweep", "select", "spp(all)")
    print(wl, n, " ".join(f"{nm} {ev[k].elapsed_time(ev[k + 1]):.3f}" for k, nm in enumerate(names)))
