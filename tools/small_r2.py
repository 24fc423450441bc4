"""Round-2 device paths on small inputs (for compute-sanitizer): the crossing-search
combine (single instance), k_dp_inst2 (mode 3), the chunked DP with two xi planes and
the multi-warp PE sweep (V > 64), RDO deduplication, large-M validation."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2204_10562_b200 as P
from paper_2204_10562_b200 import _lib, planner, workloads as W
P.spp(*W.c3_gpt96(M=8, L=24, nodes=2, per_node=8).to_model())                 # k_combine_bis_p
P.spp(*W.c3_gpt96(M=64, jitter_seed=3, L=30, nodes=2, per_node=8).to_model())
_lib.dp_persistent(3)
planner.spp_many([W.c4_instance(k).to_model() for k in range(4)])            # k_dp_inst2
_lib.dp_persistent(2)
P.spp(*W.c5_instance(L=140, V=72, M=4).to_model())                           # chunked, mw sweep
prev = _lib.rdo_dedup(2)
m = W.models_of([W.c3_gpt96(M=mm, L=12, nodes=2, per_node=4) for mm in (4, 8, 16)])
planner.spp_many(m)                                                          # RDO dedup
_lib.rdo_dedup(prev)
prof, cl, _ = W.c2_bert24().to_model()
r = P.spp(prof, cl, 4200)
P.validate_schedule(r.schedule, r.plan, prof, cl)                            # global-sort overlap check
torch.cuda.synchronize()
print("ok")
