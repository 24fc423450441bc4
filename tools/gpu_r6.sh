timeout 1200 python -m pytest tests/test_gpu_dp_modes.py tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_gpu_baselines.py tests/test_gpu_c3_headline.py -v -x > gpurun_out/r6_pytest.txt 2>&1
tail -80 gpurun_out/r6_pytest.txt
