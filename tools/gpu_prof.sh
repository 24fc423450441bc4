# usage: bash tools/gpu_prof.sh <kernel-regex> <skip> <out-name>
ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/$3 python bench.py --profile-steps 1 > /dev/null 2>&1
