"""Per-step (j) average launch durations of the per-step DP kernels from an ncu launch csv."""
import csv, sys
import numpy as np
rows = list(csv.reader(open(sys.argv[1])))
groups = int(sys.argv[2]) if len(sys.argv) > 2 else 4
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; data = rows[hi + 1:]
ki = h.index('Kernel Name'); vi = h.index('Metric Value')
seq = [(r[ki].split('(')[0].replace('void ', '').replace('pp::', ''), float(r[vi].replace(',', '')) / 1e3) for r in data]
for name in ("k_combine_s", "k_expand_s", "k_combine_s_p", "k_expand_s_p"):
    v = np.array([x for n, x in seq if n == name])
    if v.size % groups:
        continue
    g = v.reshape(groups, -1)
    print(name, "total per group", np.round(g.sum(1), 1))
    print("  by j:", " ".join(f"{j + 1}:{g[:, j].mean():.1f}" for j in range(0, g.shape[1], 4)))
