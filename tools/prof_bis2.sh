cd $GRAFT_REPO_ROOT
cat > /tmp/run_n.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_2204_10562_b200 import _device, _lib, workloads as W
from paper_2204_10562_b200.partition import sum_flags
n = int(sys.argv[1])
specs = (W.c3_sweep() * 8)[:n] if n > 1 else [W.c3_gpt96(M=32)]
items = [(_device.pack(p, c), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for p, c, M in W.models_of(specs)]
db = _device.DeviceBatch(items, capture_events=True)
db.run("spp"); torch.cuda.synchronize()
PY
PP_DP_GROUPS=1 PP_BIS_WAVES=1 PP_BIS_RB=1 ncu --set full --clock-control none --import-source on -k regex:k_combine_bis -s 31 -c 1 -o gpurun_out/bis2_n12 python /tmp/run_n.py 12 > /dev/null 2>&1
PP_DP_GROUPS=1 PP_COMBINE_BIS=0 ncu --set full --clock-control none --import-source on -k regex:k_combine_s -s 31 -c 1 -o gpurun_out/tiles_n12 python /tmp/run_n.py 12 > /dev/null 2>&1
PP_DP_GROUPS=1 ncu --set full --clock-control none --import-source on -k regex:k_expand -s 31 -c 1 -o gpurun_out/exp_n12 python /tmp/run_n.py 12 > /dev/null 2>&1
ls gpurun_out/*_n12*
