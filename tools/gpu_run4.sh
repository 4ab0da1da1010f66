mkdir -p gpurun_out/s5
timeout 600 bash tools/ncu_capture.sh rk_reverse_tc rk_reverse_kernel -- python tools/profile_step.py --config C2 --policy revolve:8 --iters 2
timeout 600 bash tools/ncu_capture.sh rk_forward_tc rk_forward_kernel -- python tools/profile_step.py --config C2 --policy revolve:8 --iters 2
mv gpurun_out/rk_*_tc_* gpurun_out/s5/ 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s5/launches_C2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/s5/ncu_launch.log 2>&1
ls -la gpurun_out/s5
