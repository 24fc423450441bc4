"""RDO passes (speculative rounds = argv[2], default 1) on C3 (n = argv[1]) or a
C4 batch (n < 0), for a launch-list capture of the LAST pass with warm caches:
ncu --cache-control none --metrics gpu__time_duration.sum -k regex:rdo -s <skip>
python tools/rdo_probe.py 1."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_10562_b200 import _device, _lib, workloads as W  # noqa: E402
from paper_2204_10562_b200.partition import sum_flags  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
specs = (W.c3_sweep() * 8)[:n] if n > 0 else W.c4_batch(-n)
items = [(_device.pack(p, c), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for p, c, M in W.models_of(specs)]
db = _device.DeviceBatch(items, capture_events=True)
_lib.rdo_rounds(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
for _ in range(3):
    db.run("rdo")
torch.cuda.synchronize()
