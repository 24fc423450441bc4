"""Device time of one global_min_cut (k_min_cut, one warp) on the C3 cluster's
full 64-GPU set and on a C4 cluster (PP_LIB_OVERRIDE selects the library)."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_10562_b200 import _device, _lib, workloads as W  # noqa: E402

for name, spec in (("C3", W.c3_sweep()[0]), ("C4", W.c4_batch(1)[0])):
    profile, cluster, M = spec.to_model()
    db = _device.DeviceBatch([(_device.pack(profile, cluster), 1, 0, None)], capture_events=False)
    V = db.max_V
    v = torch.arange(V, dtype=torch.int32, device="cuda")
    in_a = torch.zeros(V, dtype=torch.uint8, device="cuda")
    w = torch.empty(1, dtype=torch.float64, device="cuda")
    call = lambda: _lib.check(db.lib.pp_min_cut(C.byref(db.batch), 0, v.data_ptr(), V, in_a.data_ptr(), w.data_ptr(),
                                                 _device._stream()))
    call(); torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); call(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print(f"{name} V={V}: min cut {min(ts):.1f} us (median {sorted(ts)[10]:.1f}), weight {w.item():.6g}")
