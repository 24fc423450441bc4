# Same-box A/B of variant library builds on the per-step DP: tools/ab_libs2.sh "<n ...>" build/a.so ...
ns=$1; shift
for lib in main "$@"; do
  if [ "$lib" = main ]; then unset PP_LIB_OVERRIDE; else export PP_LIB_OVERRIDE=$PWD/$lib; fi
  echo "== $lib $EXTRA"; env $EXTRA python tools/dp_combine_ab.py $ns | grep tiles | awk 'NR%2==1'
done
