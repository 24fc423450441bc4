"""Instructions / stall samples per CUDA source line of an ncu report:
python tools/ncu_lines.py rep [N] [stall]   (stall: order by stall samples)."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
res, f, hdr = [], None, None
for r in csv.reader(out):
    if r and r[0] == 'File Path':
        f = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No':
        hdr = r; continue
    if r and r[0] and r[0].isdigit() and hdr:
        d = dict(zip(hdr[4:], r[4:]))
        try:
            ex = float(d.get('Instructions Executed', '0') or 0); st = float(d.get('Warp Stall Sampling (All Samples)', '0') or 0)
        except ValueError:
            continue
        res.append((ex, st, f, r[0], r[1].strip()[:90]))
tot = sum(x[0] for x in res) or 1; tst = sum(x[1] for x in res) or 1
print(f"total warp-inst {tot:.3e}  stall samples {tst:.0f}")
key = (lambda x: (x[1], x[0])) if "stall" in sys.argv[3:] else (lambda x: x)
for x in sorted(res, key=key, reverse=True)[:n]:
    print(f"{100*x[0]/tot:5.1f}% inst {100*x[1]/tst:5.1f}% stall  {x[2]}:{x[3]}  {x[4]}")
