timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt14.log 2>&1; tail -2 gpurun_out/pt14.log
for c in C1 C4 C5; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; python -c "
import json
for l in open('gpurun_out/bench_$c.json'):
    if l.startswith('{'):
        d=json.loads(l); print('$c',d['value'],d['roofline']['frac'],d['roofline']['phase_ms_per_step'])
"; tail -1 gpurun_out/bench_$c.err; done
