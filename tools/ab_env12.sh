for cfg in "PP_PDL=1" "PP_PDL=0" "PP_DP_GROUPS=1" "PP_DP_GROUPS=2" "PP_DP_GROUPS=3" "PP_DP_GROUPS=4" "PP_DP_GROUPS=12" "PP_DP_GROUPS=2 PP_PDL=0" "PP_DP_GROUPS=3 PP_PDL=0"; do
  echo "== $cfg"; env $cfg python tools/dp_combine_ab.py 12 24 | grep tiles | head -2
done
