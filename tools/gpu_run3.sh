mkdir -p gpurun_out/s4
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4/pytest_gpu.log 2>&1; tail -5 gpurun_out/s4/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/s4/bench_C2.json 2> gpurun_out/s4/bench_C2.err; tail -c 1200 gpurun_out/s4/bench_C2.json
timeout 120 python tools/profile_step.py --config C2 --policy revolve:8 --phases > gpurun_out/s4/phases_tc.txt 2>&1; cat gpurun_out/s4/phases_tc.txt
OB_NO_TC=1 timeout 120 python tools/profile_step.py --config C2 --policy revolve:8 --phases > gpurun_out/s4/phases_simt.txt 2>&1; cat gpurun_out/s4/phases_simt.txt
timeout 600 bash tools/ncu_capture.sh rk_reverse_tc rk_reverse_kernel -- python tools/profile_step.py --config C2 --policy revolve:8 --iters 1
mv gpurun_out/rk_reverse_tc_* gpurun_out/s4/ 2>/dev/null
