import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; data = rows[hi+1:]
ki = h.index('Kernel Name'); vi = h.index('Metric Value')
tot = collections.defaultdict(float); cnt = collections.Counter(); per = collections.defaultdict(list)
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for r in data:
    name = r[ki].split('(')[0]
    v = float(r[vi].replace(',',''))
    tot[name] += v; cnt[name] += 1; per[name].append(v)
T = sum(tot.values())
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:20s} {cnt[k]:5d} {tot[k]/steps/1e3:10.1f} us/step {100*tot[k]/T:5.1f}%")
for nm in ('k_combine', 'k_expand'):
    if nm in per:
        c = per[nm][:len(per[nm])//steps]
        print(nm, "per launch (us):", [round(x/1e3,1) for x in c[::4]])
