timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in C5; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]);print('$c',d['value'],d['roofline']['phase_ms_per_step'])"; done
