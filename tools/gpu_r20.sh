timeout 900 python -m pytest tests/test_gpu_dp_modes.py tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x > gpurun_out/r20_pytest.txt 2>&1; tail -3 gpurun_out/r20_pytest.txt
for lib in main build/head2.so main build/head2.so; do
  if [ "$lib" = main ]; then unset PP_LIB_OVERRIDE; else export PP_LIB_OVERRIDE=$PWD/$lib; fi
  echo "== $lib"; timeout 180 python tools/phases.py c4 2>&1 | tail -2
done
