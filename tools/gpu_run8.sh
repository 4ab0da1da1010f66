mkdir -p gpurun_out/s9
timeout 900 bash tools/ncu_capture.sh rk_reverse_c4 rk_reverse_kernel -- python tools/profile_step.py --config C4 --iters 2
timeout 900 bash tools/ncu_capture.sh rk_reverse_c3 rk_reverse_kernel -- python tools/profile_step.py --config C3 --iters 2
mv gpurun_out/rk_reverse_c4_* gpurun_out/rk_reverse_c3_* gpurun_out/s9/ 2>/dev/null
timeout 300 python tools/profile_step.py --config C4 --phases > gpurun_out/s9/phases_c4.txt 2>&1; cat gpurun_out/s9/phases_c4.txt
