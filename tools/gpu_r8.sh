# C3 n = 12 env-knob sweep on one box (phases.py: device ms per spp phase)
for cfg in "X=0" "PP_PDL=0" "PP_DP_GROUPS=4" "PP_DP_GROUPS=12" "PP_DP_GROUPS=12 PP_PDL=0" "PP_COMBINE_WAVES=1" "PP_COMBINE_WAVES=4" "PP_EXPAND_RB=1" "PP_BIS_MAX_INST=2" "PP_DP_SPLIT=12"; do
  echo "== $cfg"; env $cfg python tools/phases.py c3 12 2>&1 | tail -2
done
for cfg in "X=0" "PP_C1_PARTS=16" "PP_C1_PARTS=48" "PP_BIS_WAVES=1" "PP_BIS_WAVES=4" "PP_PDL=0"; do
  echo "== n=1 $cfg"; env $cfg python tools/phases.py c3 1 2>&1 | tail -2
done
