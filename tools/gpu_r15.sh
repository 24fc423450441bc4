PP_DP_GROUPS=1 python tools/step_trace.py 12 > gpurun_out/r15_trace_g1.txt 2>&1
PP_DP_GROUPS=1 PP_PDL=0 python tools/step_trace.py 12 > gpurun_out/r15_trace_g1_nopdl.txt 2>&1
