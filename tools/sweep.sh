set -x
mkdir -p gpurun_out/sweep
python -m pytest tests -m gpu -x -q > gpurun_out/sweep/pytest_gpu.log 2>&1; tail -3 gpurun_out/sweep/pytest_gpu.log
for c in C2 C1 C3 C4 C5; do
  timeout 600 python bench.py --config $c > gpurun_out/sweep/bench_$c.json 2> gpurun_out/sweep/bench_$c.err; tail -c 600 gpurun_out/sweep/bench_$c.json
done
timeout 600 python bench.py --impl reference > gpurun_out/sweep/bench_ref_C2.json 2> gpurun_out/sweep/bench_ref.err; tail -c 400 gpurun_out/sweep/bench_ref_C2.json
