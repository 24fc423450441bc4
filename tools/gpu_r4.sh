timeout 900 python -m pytest tests/test_gpu_dp_modes.py tests/test_gpu_scale.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
bash tools/ab_c4.sh build/v2.so 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4_launch_c3n1.csv python tools/phases.py c3 1 > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/r4_launch_c3n1.csv 4 > gpurun_out/r4_launch_c3n1.txt 2>&1
bash tools/prof_c4.sh
(python tools/summarize_ncu.py gpurun_out/dpinst_c4.ncu-rep; python tools/ncu_lines.py gpurun_out/dpinst_c4.ncu-rep 40) > gpurun_out/r4_ncu_dp_inst_c4.txt 2>&1
rm -f gpurun_out/dpinst_c4.ncu-rep
