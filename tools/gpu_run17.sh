timeout 600 bash tools/ncu_capture.sh rk_reverse_tc rk_reverse_kernel -- python tools/profile_step.py --config C2 --policy revolve:8 --iters 2
mkdir -p gpurun_out/s17; mv gpurun_out/rk_reverse_tc_* gpurun_out/s17/
timeout 120 python tools/profile_step.py --config C2 --policy revolve:8 --phases > gpurun_out/s17/phases.txt 2>&1
