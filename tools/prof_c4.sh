cd $GRAFT_REPO_ROOT
cat > /tmp/run_c4.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_2204_10562_b200 import _device, _lib, workloads as W
from paper_2204_10562_b200.partition import sum_flags
specs = W.c4_batch(4096)
items = [(_device.pack(*s.to_model()[:2]), s.M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for s in specs]
db = _device.DeviceBatch(items, capture_events=True)
db.run("spp"); torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:k_dp_inst -c 1 -o gpurun_out/dpinst_c4 python /tmp/run_c4.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python /tmp/run_c4.py > /dev/null 2>&1
