timeout 900 python -m pytest tests/test_gpu_rdo.py tests/test_gpu_parity.py tests/test_gpu_c3_headline.py -q -x > gpurun_out/r16_pytest.txt 2>&1; tail -3 gpurun_out/r16_pytest.txt
for lib in main build/head.so main build/head.so; do
  if [ "$lib" = main ]; then unset PP_LIB_OVERRIDE; else export PP_LIB_OVERRIDE=$PWD/$lib; fi
  echo "== $lib"
  timeout 180 python tools/phases.py c3 1 2>&1 | tail -2
  timeout 180 python tools/phases.py c4 2>&1 | tail -1
done
