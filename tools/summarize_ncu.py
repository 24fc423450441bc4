import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
keep = ('Duration','Elapsed Cycles','Compute (SM) Throughput','Memory Throughput','DRAM Throughput','L2 Cache Throughput','Executed Ipc Active','Issue Slots Busy','Grid Size','Block Size','Registers Per Thread','Achieved Occupancy','Theoretical Occupancy','Waves Per SM','Warp Cycles Per Issued Instruction','Eligible Warps Per Scheduler','No Eligible','Dynamic Shared Memory Per Block','Static Shared Memory Per Block')
for row in r[1:]:
    name = row[h.index('Metric Name')]
    if name in keep:
        print(f"{name[:40]:40s} {row[h.index('Metric Value')]:>14s} {row[h.index('Metric Unit')]}")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, v = r[0], r[2]
st = []
for k, name in enumerate(h):
    if name.startswith('smsp__average_warps_issue_stalled_') and name.endswith('_per_issue_active.ratio'):
        try: st.append((float(v[k]), name[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]))
        except ValueError: pass
    if 'inst_executed_pipe_' in name and name.endswith('avg.pct_of_peak_sustained_active'):
        try:
            if float(v[k]) > 2: print("pipe", name.split('inst_executed_pipe_')[1].split('.')[0], v[k])
        except ValueError: pass
    if name in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg'):
        print(name, v[k], r[1][k])
print("stalls:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:7]))
