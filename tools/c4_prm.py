"""pp_prm time for C4 batches of n instances (GPU only): python tools/c4_prm.py n ..."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_10562_b200 import _device, _lib, workloads as W  # noqa: E402
from paper_2204_10562_b200.partition import sum_flags  # noqa: E402
for n in [int(x) for x in sys.argv[1:]] or [4096]:
    specs = W.c4_batch(n)
    items = [(_device.pack(*s.to_model()[:2]), s.M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for s in specs]
    db = _device.DeviceBatch(items, capture_events=True)
    db.run("phi"); db.run("rdo"); db.run("prm"); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); db.run("prm"); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"PP_DP_INST={os.environ.get('PP_DP_INST', '2')} n={n} prm min {min(ts):.3f} ms  per-instance {1e3 * min(ts) / n:.2f} us",
          flush=True)
    del db
    torch.cuda.empty_cache()
