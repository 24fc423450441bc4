"""cProfile of the host side of spp_many on the C3 batch (GPU box): python tools/host_prof.py."""
import cProfile, pstats, sys
sys.path.insert(0, ".")
import torch
from paper_2204_10562_b200 import planner, workloads as W

models = W.models_of(W.c3_sweep())
for _ in range(3):
    planner.spp_many(models)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    planner.spp_many(models)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
