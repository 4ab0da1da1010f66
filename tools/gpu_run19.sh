mkdir -p gpurun_out/final3
timeout 900 bash tools/ncu_capture.sh rk_reverse_c4 rk_reverse_kernel -- python tools/profile_step.py --config C4 --iters 2
timeout 900 bash tools/ncu_capture.sh rk_reverse_c3 rk_reverse_kernel -- python tools/profile_step.py --config C3 --iters 2
timeout 900 bash tools/ncu_capture.sh theta_fwd_c5 theta_forward_kernel -- python tools/profile_step.py --config C5 --iters 2
timeout 900 bash tools/ncu_capture.sh rk_reverse_c1 rk_reverse_kernel -- python tools/profile_step.py --config C1 --iters 2
mv gpurun_out/rk_reverse_c4_* gpurun_out/rk_reverse_c3_* gpurun_out/theta_fwd_c5_* gpurun_out/rk_reverse_c1_* gpurun_out/final3/ 2>/dev/null
ls gpurun_out/final3 | wc -l
