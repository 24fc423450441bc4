"""A few small spp instances through the default path (for compute-sanitizer runs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_10562_b200 import planner, workloads as W
ms = [W.c2_bert24().to_model()] + [W.c4_instance(k).to_model() for k in range(3)]
planner.spp_many(ms)                                 # batch of 4 (per-step graph, bulk combine)
planner.spp(*W.c3_gpt96(M=8, nodes=2, per_node=8).to_model())   # single instance (split chain)
torch.cuda.synchronize()
print("ok")
