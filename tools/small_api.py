"""The other device entry points on small inputs (for compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2204_10562_b200 as P
from paper_2204_10562_b200 import workloads as W
prof, cl, M = W.c2_bert24().to_model()
r = P.spp(prof, cl, M)
P.simulate_pe(r.plan, prof, cl)
P.simulate_pe_many([r.plan, r.plan], prof, cl)
P.simulate_with_order(r.plan, prof, cl, P.compute_execution_order(r.plan).queues)
P.simulate_cycle_schedule(r.plan, prof, cl)
P.validate_schedule(r.schedule, r.plan, prof, cl)
P.cost_summary(r.plan, prof, cl)
P.write_trace(None, r.schedule)
P.global_min_cut(cl)
o = P.rdo(cl)
P.prm(prof, cl, o, M, prof.num_layers, 2, 1, len(cl.gpu_ids))
s = P.PartitionSolver(prof, cl, o, M)
s.solve(prof.num_layers, 2, 1, len(cl.gpu_ids))
P.gpipe_schedule(P.gpipe_plan(prof, cl, o, 4, M), prof, cl)
torch.cuda.synchronize()
print("ok")
