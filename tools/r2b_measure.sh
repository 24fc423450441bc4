#!/bin/bash
# Round-2 measurement set (GPU box, repo root; outputs in gpurun_out/r2b_*)
set -x
python bench.py --steps 200 --warmup 5 > gpurun_out/r2b_c3.json 2> gpurun_out/r2b_c3.err


python bench.py --workload c4 --steps 10 --warmup 3 > gpurun_out/r2b_c4.json 2> gpurun_out/r2b_c4.err
python bench.py --workload c5 --steps 20 --warmup 3 > gpurun_out/r2b_c5.json 2> gpurun_out/r2b_c5.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches_c3.csv python bench.py --profile-steps 1 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r2b_traffic_warm.csv python bench.py --profile-steps 1 > /dev/null 2>&1
python tools/dp_traffic.py gpurun_out/r2b_traffic_warm.csv gpurun_out/r02b_dp_traffic_warm.json 1 warm
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_traffic_cold.csv python bench.py --profile-steps 1 > /dev/null 2>&1
python tools/dp_traffic.py gpurun_out/r2b_traffic_cold.csv gpurun_out/r02b_dp_traffic_cold.json 1
for k in k_combine_s_p:120 k_expand_m_p:60 k_rdo_cut:0 "k_rdo<":0 k_pe_sweep_w:0 k_event_merge:0 k_select:0 k_backtrack_p:0 k_stab_big_p:0; do
  name=${k%%:*}; skip=${k##*:}
  ncu --set full --import-source on --clock-control none -k regex:"${name}" -s $skip -c 1 -o /tmp/r2b_ncu_${name//</_} python bench.py --profile-steps 1 > /dev/null 2>&1
  (python tools/summarize_ncu.py /tmp/r2b_ncu_${name//</_}.ncu-rep; python tools/ncu_lines.py /tmp/r2b_ncu_${name//</_}.ncu-rep 25) > gpurun_out/r2b_ncu_${name//</_}.txt 2>&1
done
bash tools/prof_c4.sh > /dev/null 2>&1
(python tools/summarize_ncu.py gpurun_out/dpinst_c4.ncu-rep; python tools/ncu_lines.py gpurun_out/dpinst_c4.ncu-rep 25) > gpurun_out/r2b_ncu_dp_inst_c4.txt 2>&1
rm -f gpurun_out/*.ncu-rep
python tools/step_trace.py 12 > gpurun_out/r2b_trace12.txt 2>&1
python tools/step_trace.py 1 > gpurun_out/r2b_trace1.txt 2>&1
(python tools/phases.py c3 1; python tools/phases.py c3 12; python tools/phases.py c4) > gpurun_out/r2b_phases.txt 2>&1
python tools/e2e_breakdown.py > gpurun_out/r2b_e2e.txt 2>&1
tail -c 600 gpurun_out/r2b_c3.json
