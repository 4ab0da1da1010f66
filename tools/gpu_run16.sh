timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt16.log 2>&1; tail -2 gpurun_out/pt16.log
for c in C4 C2; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; python -c "
import json
for l in open('gpurun_out/bench_$c.json'):
    if l.startswith('{'):
        d=json.loads(l); print('$c',d['value'],d['roofline']['frac'],d['roofline']['phase_ms_per_step'])
"; done
