"""RDO alone on the C5 cluster (256 GPUs) and a C4 / C3 batch, warm: device ms per call.
    python tools/c5_rdo.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_10562_b200 import _device, _lib, workloads as W  # noqa: E402
from paper_2204_10562_b200.partition import sum_flags  # noqa: E402


def timed(db, reps=4):
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); db.run("rdo"); b.record(); torch.cuda.synchronize()
        out.append(round(a.elapsed_time(b), 3))
    return out


spec = W.c5_instance(L=8, V=256, M=512)   # RDO depends on the cluster only: a short chain keeps the workspace small
p, c, _ = spec.to_model()
db = _device.DeviceBatch([(_device.pack(p, c), 512, _lib.PP_ALLOW_REPLICATION | sum_flags(), None)], capture_events=False)
print("c5 cluster (V 256) rdo ms", timed(db))
