cd $GRAFT_REPO_ROOT
cat > /tmp/run48.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_2204_10562_b200 import _device, _lib, workloads as W
from paper_2204_10562_b200.partition import sum_flags
specs = (W.c3_sweep() * 8)[:48]
items = [(_device.pack(p, c), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for p, c, M in W.models_of(specs)]
db = _device.DeviceBatch(items, capture_events=True)
db.run("spp"); torch.cuda.synchronize()
PY
PP_DP_GROUPS=1 ncu --set full --clock-control none --import-source on -k regex:k_combine_s -s 31 -c 1 -o gpurun_out/comb48 python /tmp/run48.py > /dev/null 2>&1
PP_DP_GROUPS=1 ncu --set full --clock-control none --import-source on -k regex:k_expand_s -s 31 -c 1 -o gpurun_out/exp48 python /tmp/run48.py > /dev/null 2>&1
ls gpurun_out/*48*
