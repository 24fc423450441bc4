#!/bin/bash
# Same-box A/B of the in-tree library against variant builds: tools/ab_quick.sh "<dp_ab args>" build/a.so ...
args=$1; shift
for lib in main "$@"; do
  if [ "$lib" = main ]; then unset PP_LIB_OVERRIDE; else export PP_LIB_OVERRIDE=$PWD/$lib; fi
  echo "== $lib"; MODES=${MODES:-0} python tools/dp_ab.py $args 2>&1 | grep early_exit=True
done
