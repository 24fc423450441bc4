"""Small batches through every DP schedule and the large-schedule event path (for compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_10562_b200 import _lib, planner, workloads as W
ms = [W.c2_bert24().to_model()] + [W.c4_instance(k).to_model() for k in range(3)]
for mode in (0, 3):
    _lib.dp_persistent(mode)
    planner.spp_many(ms)
_lib.dp_persistent(2)
p, c, _ = W.c4_instance(0).to_model()
planner.spp(p, c, 1500)          # M (4N - 3) > 18432 events: k_event_rank
torch.cuda.synchronize()
print("ok")
