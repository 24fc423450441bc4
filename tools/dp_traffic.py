"""ncu CSV (dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum over one
bench step) -> profiles/ncu_dp_traffic.json: python tools/dp_traffic.py in.csv out.json [steps]."""
import csv, json, re, sys
from collections import defaultdict

src, dst = sys.argv[1], sys.argv[2]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
warm = len(sys.argv) > 4 and sys.argv[4] == "warm"   # captured with --cache-control none
rows = [r for r in csv.reader(open(src)) if r and not r[0].startswith("==")]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
per = defaultdict(lambda: {"read": 0.0, "write": 0.0, "time_ns": 0.0, "launches": 0})
for r in rows[1:]:
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("pp::", "").strip()
    v = float(r[vi].replace(",", ""))
    m = r[mi]
    if m == "dram__bytes_read.sum":
        per[name]["read"] += v
        per[name]["launches"] += 1
    elif m == "dram__bytes_write.sum":
        per[name]["write"] += v
    elif m == "gpu__time_duration.sum":
        per[name]["time_ns"] += v
dp = re.compile(r"k_(prep|base|sdedup|stab|expand|combine|backtrack)")
rd = sum(p["read"] for k, p in per.items() if dp.match(k)) / steps
wr = sum(p["write"] for k, p in per.items() if dp.match(k)) / steps
out = {"what": "DRAM bytes (read+write) of the DP phase (pp_prm graph: prep, base, sdedup, stab, expand, combine, "
               "backtrack kernels) per C3 12-instance step; ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
               + ("--cache-control none (caches NOT flushed between kernels: the warm traffic of a steady-state step, "
                  "kernels serialised)" if warm else "(ncu flushes caches per kernel: cold-cache upper bound)"),
       "dram_bytes_per_step": rd + wr, "read": rd, "write": wr,
       "per_kernel": {k: {kk: (vv / steps if kk != "launches" else vv // steps) for kk, vv in p.items()}
                      for k, p in sorted(per.items(), key=lambda kv: -kv[1]["time_ns"])}}
json.dump(out, open(dst, "w"), indent=1)
print(f"DP DRAM bytes per step {rd + wr:.4g} (read {rd:.4g}, write {wr:.4g})")
