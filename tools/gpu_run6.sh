mkdir -p gpurun_out/s7
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s7/pytest.log 2>&1; tail -3 gpurun_out/s7/pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/s7/bench_C2.json 2> gpurun_out/s7/bench_C2.err; head -c 400 gpurun_out/s7/bench_C2.json; echo
timeout 120 python tools/profile_step.py --config C2 --policy revolve:8 --phases > gpurun_out/s7/phases_tc.txt 2>&1; cat gpurun_out/s7/phases_tc.txt
for c in C1 C3 C4 C5; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/s7/bench_$c.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/s7/bench_$c.json').read().strip().splitlines()[-1]);print('$c',d['value'],d['roofline']['phase_ms_per_step'])"; done
