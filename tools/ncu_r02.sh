#!/bin/bash
# ncu_r02.sh -- round-2 profile set (GPU box): launch list of the default bench command,
# full-section captures of the C2 reverse kernel (headline) and the C4 tcgen05 kernels.
mkdir -p gpurun_out/ncu_r02
#ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
#  --log-file python bench.py --per-config "" --steps 2 --warmup 1 --no-cpu-baseline \
#  >
bash tools/ncu_capture.sh ncu_r02/c2_reverse "rk_reverse_kernel" -- python tools/profile_step.py --config C2 --policy revolve:8 --iters 3
bash tools/ncu_capture.sh ncu_r02/c4_reverse "rk_reverse_kernel" -- python tools/profile_step.py --config C4 --iters 3
bash tools/ncu_capture.sh ncu_r02/c4_forward "rk_forward_kernel" -- python tools/profile_step.py --config C4 --iters 3
ls -la gpurun_out/ncu_r02
