# final r01 sweep: all five configs with CPU baselines, reference arm, launch list, ncu of the C2 kernels
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final/pytest_gpu.log 2>&1; tail -2 gpurun_out/final/pytest_gpu.log
for c in C2 C1 C3 C4 C5; do timeout 600 python bench.py --config $c > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err; done
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_ref_C2.json 2> gpurun_out/final/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_C2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/final/ncu_launch.log 2>&1
timeout 600 bash tools/ncu_capture.sh rk_reverse_tc rk_reverse_kernel -- python tools/profile_step.py --config C2 --policy revolve:8 --iters 2
timeout 600 bash tools/ncu_capture.sh rk_forward_tc rk_forward_kernel -- python tools/profile_step.py --config C2 --policy revolve:8 --iters 2
mv gpurun_out/rk_*_tc_* gpurun_out/final/ 2>/dev/null
timeout 120 python tools/profile_step.py --config C2 --policy revolve:8 --phases > gpurun_out/final/phases_C2.txt 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/final/smoke.log 2>&1; tail -2 gpurun_out/final/smoke.log
ls gpurun_out/final
