for cfg in "1 1" "1 2" "1 4" "0.5 1"; do set -- $cfg; echo "WAVES=$1 RB=$2"; PP_BIS_WAVES=$1 PP_BIS_RB=$2 python tools/dp_combine_ab.py 12 24 | grep bis; done
PP_BIS_WAVES=1 PP_BIS_RB=1 python tools/step_trace.py 12 > gpurun_out/r2_tr12_bis.txt 2>&1
PP_COMBINE_BIS=0 python tools/step_trace.py 12 > gpurun_out/r2_tr12_tiles.txt 2>&1
