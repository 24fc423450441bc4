for s in 1 2 4; do
  PP_COMBINE_SPLIT=$s timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split', $s, 'value', round(d['value']), d['roofline']['phase_ms'])"
done
