for cfg in "X=0" "PP_DP_GROUPS=1" "PP_DP_GROUPS=2" "PP_DP_GROUPS=3" "PP_DP_GROUPS=1 PP_COMBINE_WAVES=4" "PP_DP_GROUPS=2 PP_COMBINE_WAVES=3"; do
  echo "== $cfg"; env $cfg python tools/phases.py c3 12 2>&1 | tail -2
done
