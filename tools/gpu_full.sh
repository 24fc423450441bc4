timeout 1500 python -m pytest tests -m gpu -v > gpurun_out/full_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/full_pytest.txt
tail -5 gpurun_out/full_pytest.txt
