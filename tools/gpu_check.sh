timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/chk_pytest.txt 2>&1; tail -3 gpurun_out/chk_pytest.txt
timeout 400 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/chk_c3.json 2> gpurun_out/chk_c3.err
timeout 400 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/chk_c4.json 2> gpurun_out/chk_c4.err
python tools/phases.py c3 12 > gpurun_out/chk_phases.txt 2>&1; python tools/phases.py c4 >> gpurun_out/chk_phases.txt 2>&1
tail -c 400 gpurun_out/chk_c3.json
