timeout 900 python -m pytest tests/test_gpu_dp_modes.py tests/test_gpu_scale.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
bash tools/ab_c4.sh build/v1.so 2>&1
bash tools/prof_c4.sh
(python tools/summarize_ncu.py gpurun_out/dpinst_c4.ncu-rep; python tools/ncu_lines.py gpurun_out/dpinst_c4.ncu-rep 40) > gpurun_out/r3_ncu_dp_inst_c4.txt 2>&1
rm -f gpurun_out/dpinst_c4.ncu-rep
