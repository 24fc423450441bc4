python bench.py --steps 200 --warmup 5 > gpurun_out/r18_c3.json 2> gpurun_out/r18_c3.err
python bench.py --workload c4 --steps 10 --warmup 3 > gpurun_out/r18_c4.json 2> gpurun_out/r18_c4.err
(python tools/phases.py c3 1; python tools/phases.py c3 12; python tools/phases.py c4) > gpurun_out/r18_phases.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r18_launches_c3.csv python bench.py --profile-steps 1 > /dev/null 2>&1
python tools/e2e_breakdown.py > gpurun_out/r18_e2e.txt 2>&1
