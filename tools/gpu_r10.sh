cat > /tmp/run_c4.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_2204_10562_b200 import _device, _lib, workloads as W
from paper_2204_10562_b200.partition import sum_flags
specs = W.c4_batch(4096)
items = [(_device.pack(*s.to_model()[:2]), s.M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for s in specs]
db = _device.DeviceBatch(items, capture_events=True)
for _ in range(3): db.run("spp")
torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r10_c4_warm.csv python /tmp/run_c4.py > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/r10_c4_warm.csv 3 > gpurun_out/r10_c4_warm.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r10_c3n1_warm.csv python tools/phases.py c3 1 > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/r10_c3n1_warm.csv 7 > gpurun_out/r10_c3n1_warm.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r10_c3n12_warm.csv python tools/phases.py c3 12 > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/r10_c3n12_warm.csv 7 > gpurun_out/r10_c3n12_warm.txt 2>&1
