timeout 1200 python -m pytest tests/test_gpu_dp_modes.py tests/test_gpu_parity.py tests/test_gpu_baselines.py tests/test_gpu_c3_headline.py -q -x > gpurun_out/r11_pytest.txt 2>&1; tail -3 gpurun_out/r11_pytest.txt
bash tools/ab_c4.sh build/v7b.so build/v8.so 2>&1
