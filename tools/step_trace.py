"""Per-CTA timeline of the per-step DP kernels (GPU only): python tools/step_trace.py [n]."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_10562_b200 import _device, _lib, workloads as W  # noqa: E402
from paper_2204_10562_b200.partition import sum_flags  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
specs = (W.c3_sweep() * 16)[:n]
items = [(_device.pack(p, c), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for p, c, M in W.models_of(specs)]
db = _device.DeviceBatch(items, capture_events=True)
lib = _lib.load()
db.run("spp"); torch.cuda.synchronize()
cap = 1 << 20
buf = torch.zeros(4 * cap, dtype=torch.int64, device="cuda")
db.run("phi"); db.run("rdo"); torch.cuda.synchronize()
_lib.check(lib.pp_step_trace(buf.data_ptr(), cap))
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record(); db.run("prm"); b.record(); torch.cuda.synchronize()
_lib.check(lib.pp_step_trace(None, 0))
print(f"prm {a.elapsed_time(b):.3f} ms")
tr = buf.view(-1, 4).cpu().numpy().astype(np.uint64)
tr = tr[tr[:, 2] != 0].astype(np.int64)
kind = (tr[:, 0] >> 56) & 0xff; j = (tr[:, 0] >> 40) & 0xffff
t0 = tr[:, 1]; t1 = tr[:, 2]; tw = tr[:, 3]; base = t0.min()
s, e = (t0 - base) / 1e3, (t1 - base) / 1e3
w = np.where(tw > 0, (tw - base) / 1e3, s)   # end of the PDL wait
print(f"{len(tr)} CTAs, span {e.max():.1f} us")
for k, nm in ((1, "expand"), (2, "combine")):
    m = kind == k
    d = e[m] - s[m]
    print(f"{nm}: {m.sum()} CTAs, CTA time mean {d.mean():.2f} us p50 {np.median(d):.2f} p90 {np.percentile(d, 90):.2f} max {d.max():.1f}; total CTA-us {d.sum() / 1e3:.1f} ms")
    dw = w[m] - s[m]
    print(f"    of which PDL wait mean {dw.mean():.2f} us (total {dw.sum() / 1e3:.1f} ms), after wait mean {(e[m] - w[m]).mean():.2f} us")
for jj in (1, 8, 16, 32, 48, 62):
    for k, nm in ((1, "E"), (2, "C")):
        m = (kind == k) & (j == jj)
        if m.any():
            print(f"  j={jj:2d} {nm}: CTAs {m.sum():5d}  window [{s[m].min():8.1f}, {e[m].max():8.1f}] = {e[m].max() - s[m].min():6.1f} us  CTA mean {np.mean(e[m] - s[m]):5.2f} max {np.max(e[m] - s[m]):5.2f} post-wait {np.mean(e[m] - w[m]):5.2f}")
# per-step window: first CTA start of E(j) to last end of C(j), and gaps
ws = []
for jj in range(1, int(j.max()) + 1):
    me, mc = (kind == 1) & (j == jj), (kind == 2) & (j == jj)
    if me.any() and mc.any():
        ws.append((jj, s[me].min(), e[me].max(), s[mc].min(), e[mc].max()))
ws = np.array(ws)
print("mean expand window %.1f us, combine window %.1f us, E->C gap %.1f us, C->E(next) gap %.1f us" % (
    np.mean(ws[:, 2] - ws[:, 1]), np.mean(ws[:, 4] - ws[:, 3]), np.mean(ws[:, 3] - ws[:, 2]),
    np.mean(ws[1:, 1] - ws[:-1, 4])))
