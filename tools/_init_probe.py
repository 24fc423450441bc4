import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_10562_b200 import _device, _lib, workloads as W  # noqa: E402
from paper_2204_10562_b200.partition import sum_flags  # noqa: E402
L, V, M = (int(x) for x in sys.argv[1:4])
spec = W.c5_instance(L=L, V=V, M=M)
profile, cluster, _ = spec.to_model()
db = _device.DeviceBatch([(_device.pack(profile, cluster), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None)],
                         capture_events=False)
db.run("phi"); db.run("rdo"); torch.cuda.synchronize()
print("rdo done", flush=True)
db.run("prm"); torch.cuda.synchronize()
print("prm done", flush=True)
h = db.fetch()
print("order", list(h["order"][:V]))
