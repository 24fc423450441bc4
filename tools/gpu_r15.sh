PP_DP_GROUPS=1 python tools/step_trace.py 12 > gpurun_out/r15_trace_g1.txt 2>&1
PP_DP_GROUPS=1 PP_PDL=0 python tools/step_trace.py 12 > gpurun_out/r15_trace_g1_nopdl.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/r15_smoke.txt 2>&1
