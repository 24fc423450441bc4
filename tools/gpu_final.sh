timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/final_pytest.txt
tail -3 gpurun_out/final_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1; tail -1 gpurun_out/final_smoke.txt
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -c 300 gpurun_out/final_bench.json
timeout 600 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; tail -c 200 gpurun_out/final_ref.json
