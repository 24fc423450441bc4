"""Print the hottest SASS instructions (stall samples) of an ncu report: python tools/ncu_hot_sass.py rep [N]."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
r = list(csv.reader(out))
h = r[1]
rows = r[2:]
si, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(float(x[si]) for x in rows if x[si])
texec = sum(float(x[ei]) for x in rows if x[ei])
print(f"samples {tot:.0f}  warp-instructions executed {texec:.0f}")
for k, x in enumerate(rows):
    x.append(k)
for x in sorted(rows, key=lambda x: -float(x[si] or 0))[:n]:
    print(f"{100 * float(x[si]) / tot:5.1f}%  #{x[-1]:5d} exec {x[ei]:>8s}  {x[1].strip()[:90]}")
