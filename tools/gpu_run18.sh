mkdir -p gpurun_out/final2
for c in C2 C4; do timeout 600 python bench.py --config $c > gpurun_out/final2/bench_$c.json 2> gpurun_out/final2/bench_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final2/launches_C2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/final2/ncu_launch.log 2>&1
timeout 600 bash tools/ncu_capture.sh rk_forward_tc rk_forward_kernel -- python tools/profile_step.py --config C2 --policy revolve:8 --iters 2
mv gpurun_out/rk_forward_tc_* gpurun_out/final2/
