for cfg in "X=0" "PP_EXPAND_WIDE=1" "PP_EXPAND_WIDE=4" "PP_EXPAND_RB_MIN=2" "PP_EXPAND_RB_MIN=8" "PP_COMBINE_SPLIT=4" "PP_BULK=0" "PP_DP_GROUPS=5" "PP_DP_GROUPS=8" "PP_EXPAND_RB=3" "X=0"; do
  echo "== $cfg"; env $cfg timeout 120 python tools/phases.py c3 12 2>&1 | tail -2
done
