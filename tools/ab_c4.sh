#!/bin/bash
# C4 DP A/B on one box: tools/ab_c4.sh lib1.so lib2.so ... (in-tree library = main)
for lib in main "$@"; do
  if [ "$lib" = main ]; then unset PP_LIB_OVERRIDE; else export PP_LIB_OVERRIDE=$PWD/$lib; fi
  echo "== $lib"
  timeout 180 python tools/phases.py c4 2>&1 | tail -2
  timeout 180 python tools/phases.py c3 12 2>&1 | tail -1
  timeout 180 python tools/phases.py c3 1 2>&1 | tail -1
done
