timeout 1200 python -m pytest tests/test_gpu_dp_modes.py tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x > gpurun_out/r14_pytest.txt 2>&1; tail -3 gpurun_out/r14_pytest.txt
bash tools/ab_c4.sh build/v10b.so build/v11b.so 2>&1
