for tool in memcheck racecheck synccheck; do
  echo "== $tool"; timeout 900 compute-sanitizer --tool $tool python tools/small_modes.py 2>&1 | tail -3
done
timeout 900 python tools/c5_full_dp.py > gpurun_out/r21_c5_full_dp.txt 2>&1; tail -5 gpurun_out/r21_c5_full_dp.txt
