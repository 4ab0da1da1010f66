mkdir -p gpurun_out/s6
timeout 600 python -m pytest tests/test_gpu_tensor_cores.py tests/test_gpu_parity.py -x -q > gpurun_out/s6/pytest.log 2>&1; tail -3 gpurun_out/s6/pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/s6/bench_C2.json 2> gpurun_out/s6/bench_C2.err; tail -c 900 gpurun_out/s6/bench_C2.json
timeout 120 python tools/profile_step.py --config C2 --policy revolve:8 --phases > gpurun_out/s6/phases_tc.txt 2>&1; cat gpurun_out/s6/phases_tc.txt
timeout 600 bash tools/ncu_capture.sh rk_reverse_tc rk_reverse_kernel -- python tools/profile_step.py --config C2 --policy revolve:8 --iters 2
mv gpurun_out/rk_*_tc_* gpurun_out/s6/ 2>/dev/null
