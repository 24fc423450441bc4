"""One spp pass over n C3 instances (for ncu launch filtering): python tools/prm_once.py [n]."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_10562_b200 import _device, _lib, workloads as W  # noqa: E402
from paper_2204_10562_b200.partition import sum_flags  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
specs = (W.c3_sweep() * 16)[:n]
items = [(_device.pack(p, c), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for p, c, M in W.models_of(specs)]
db = _device.DeviceBatch(items)
db.run("spp"); torch.cuda.synchronize()
