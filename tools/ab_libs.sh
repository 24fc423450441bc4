#!/bin/bash
# Same-box A/B of library builds: tools/ab_libs.sh "<dp_ab args>" lib1.so lib2.so ...
# (the in-tree library is "main"); prints dp_ab lines and bench value per build.
args=$1; shift
for lib in main "$@"; do
  if [ "$lib" = main ]; then unset PP_LIB_OVERRIDE; else export PP_LIB_OVERRIDE=$PWD/$lib; fi
  echo "== $lib"
  MODES=${MODES:-0} python tools/dp_ab.py $args 2>&1 | grep early_exit=True
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench value', round(d['value']), 'p50', round(d['p50_latency_ms'],3), 'e2e', round(d['e2e']['value']), 'phases', {k: round(v,3) for k,v in d['roofline']['phase_ms'].items()})"
done
