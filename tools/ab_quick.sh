for lib in main build/ab_tl4.so build/ab_trw4.so; do
  if [ "$lib" = main ]; then unset PP_LIB_OVERRIDE; else export PP_LIB_OVERRIDE=$PWD/$lib; fi
  echo "== $lib"; MODES=0 python tools/dp_ab.py 1 12 24 2>&1 | grep early_exit=True
done
