timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'p50', d['p50_latency_ms'], d['roofline']['phase_ms'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'])"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv python bench.py --profile-steps 2 > /dev/null 2>&1
