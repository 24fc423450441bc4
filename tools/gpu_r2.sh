timeout 600 python -m pytest tests/test_gpu_divfixed.py tests/test_gpu_dp_modes.py tests/test_gpu_scale.py -q -x 2>&1 | tail -4
bash tools/ab_c4.sh build/base.so 2>&1
