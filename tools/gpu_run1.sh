set -x
mkdir -p gpurun_out/s2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2/pytest_gpu.log 2>&1; tail -3 gpurun_out/s2/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/s2/smoke.log 2>&1; tail -3 gpurun_out/s2/smoke.log
timeout 600 python bench.py > gpurun_out/s2/bench_C2.json 2> gpurun_out/s2/bench_C2.err; tail -c 300 gpurun_out/s2/bench_C2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s2/launches_C2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/s2/ncu_launch.log 2>&1
timeout 900 bash tools/ncu_capture.sh rk_reverse_c2 rk_reverse_kernel -- python bench.py --steps 1 --warmup 0 --no-cpu-baseline
mv gpurun_out/rk_reverse_c2_* gpurun_out/s2/ 2>/dev/null
ls gpurun_out/s2
