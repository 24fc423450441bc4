for lib in main build/v12.so build/prerdo.so main; do
  if [ "$lib" = main ]; then unset PP_LIB_OVERRIDE; else export PP_LIB_OVERRIDE=$PWD/$lib; fi
  echo "== $lib"
  timeout 300 python tools/c5_rdo.py 2>&1 | tail -1
  timeout 180 python tools/phases.py c3 1 2>&1 | tail -1
  timeout 180 python tools/phases.py c4 2>&1 | tail -1
done
timeout 900 python -m pytest tests/test_gpu_rdo.py -q -x 2>&1 | tail -2
