timeout 1200 python -m pytest tests/test_gpu_dp_modes.py tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_gpu_baselines.py -q -x > gpurun_out/r9_pytest.txt 2>&1; tail -3 gpurun_out/r9_pytest.txt
bash tools/ab_c4.sh build/v6.so 2>&1
for w in 1 1.25 1.5 2; do echo "== n=1 PP_BIS_WAVES=$w"; PP_BIS_WAVES=$w python tools/phases.py c3 1 2>&1 | tail -2; done
