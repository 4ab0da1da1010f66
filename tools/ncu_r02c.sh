#!/bin/bash
# ncu_r02c.sh -- profile refresh after the clusters-of-two change (GPU box): launch list of the
# default bench command and a full-section capture of the C1 reverse kernel.
mkdir -p gpurun_out/ncu_r02
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/ncu_r02/launches_default_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/ncu_r02/launches_default_bench.log 2>&1
bash tools/ncu_capture.sh ncu_r02/c1_reverse "rk_reverse_kernel" -- python tools/profile_step.py --config C1 --iters 3
bash tools/ncu_capture.sh ncu_r02/c1_forward "rk_forward_kernel" -- python tools/profile_step.py --config C1 --iters 3
ls -la gpurun_out/ncu_r02
