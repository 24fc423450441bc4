"""A batch large enough for the multi-row expand (> 4 rows per SM) but small per instance (for compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_10562_b200 import _lib, planner, workloads as W
_lib.dp_persistent(0)   # per-step schedule (auto would pick instance-per-CTA for many small instances)
planner.spp_many([W.c4_instance(k).to_model() for k in range(24)])   # rows without a payload class
planner.spp_many([W.c3_gpt96(M=8 * (k + 1), nodes=2, per_node=8).to_model() for k in range(8)])   # one class
torch.cuda.synchronize()
_lib.dp_persistent(2)
print("ok")
