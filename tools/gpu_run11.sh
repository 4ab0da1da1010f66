mkdir -p gpurun_out/s12
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s12/pytest.log 2>&1; tail -2 gpurun_out/s12/pytest.log
OB_HOST_TIMING=1 timeout 120 python tools/host_overhead.py 2>&1 | grep -v "^ " | sed -n 8,12p
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/s12/bench_C2.json 2> gpurun_out/s12/bench_C2.err; python -c "import json;d=json.loads(open('gpurun_out/s12/bench_C2.json').read().strip().splitlines()[-1]);print(d['value'],d['e2e']['value'],d['roofline']['frac'])"
