timeout 1200 python -m pytest tests/test_gpu_dp_modes.py tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_gpu_baselines.py tests/test_gpu_c3_headline.py -q -x 2>&1 | tail -3
bash tools/ab_c4.sh build/v2.so build/v5.so 2>&1
