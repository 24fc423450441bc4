bash tools/prof_c4.sh
(python tools/summarize_ncu.py gpurun_out/dpinst_c4.ncu-rep; python tools/ncu_lines.py gpurun_out/dpinst_c4.ncu-rep 50) > gpurun_out/r7_ncu_dp_inst_c4.txt 2>&1
ls -la gpurun_out/dpinst_c4.ncu-rep
python tools/summarize_launches.py gpurun_out/c4_launches.csv 1 > gpurun_out/r7_c4_launches.txt 2>&1
