for cfg in "PP_CRIT_FUSED=0" "PP_CRIT_FUSED=1 PP_CRIT_CLUSTER=4" "PP_CRIT_FUSED=1 PP_CRIT_CLUSTER=8" "PP_CRIT_FUSED=1 PP_CRIT_CLUSTER=16"; do
  echo "== $cfg"; env $cfg python tools/dp_combine_ab.py 1 2 | grep bis | awk 'NR%2==1'
done
