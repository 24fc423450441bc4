#!/bin/bash
# Round-end measurement set (run on the GPU box from the repo root; outputs in gpurun_out/).
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/fin_c3.json 2> gpurun_out/fin_c3.err
python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/fin_c4.json 2>&1
python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/fin_c5.json 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin_ref.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches.csv python bench.py --profile-steps 1 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_traffic.csv python bench.py --profile-steps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_combine_s_p -s 120 -c 1 -o gpurun_out/fin_comb python bench.py --profile-steps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_expand -s 120 -c 1 -o gpurun_out/fin_exp python bench.py --profile-steps 1 > /dev/null 2>&1
python tools/step_trace.py 12 > gpurun_out/fin_trace12.txt 2>&1
python tools/step_trace.py 1 > gpurun_out/fin_trace1.txt 2>&1
(python tools/phases.py c3 1; python tools/phases.py c3 12; python tools/phases.py c4) > gpurun_out/fin_phases.txt 2>&1
python tools/e2e_breakdown.py > gpurun_out/fin_e2e.txt 2>&1
tail -c 400 gpurun_out/fin_c3.json
