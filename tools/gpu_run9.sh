mkdir -p gpurun_out/s10
timeout 300 python tools/profile_step.py --config C5 --iters 1 --phases > gpurun_out/s10/phases_c5.txt 2>&1; cat gpurun_out/s10/phases_c5.txt
timeout 900 bash tools/ncu_capture.sh theta_fwd_c5 theta_forward_kernel -- python tools/profile_step.py --config C5 --iters 2
mv gpurun_out/theta_fwd_c5_* gpurun_out/s10/ 2>/dev/null
