mkdir -p gpurun_out/s3
timeout 600 python -m pytest tests/test_gpu_tensor_cores.py -x -q > gpurun_out/s3/pytest_tc.log 2>&1; tail -30 gpurun_out/s3/pytest_tc.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/s3/bench_C2.json 2> gpurun_out/s3/bench_C2.err; tail -c 1500 gpurun_out/s3/bench_C2.json; tail -5 gpurun_out/s3/bench_C2.err
