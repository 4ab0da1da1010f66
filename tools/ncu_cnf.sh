#!/bin/bash
mkdir -p gpurun_out/ncu_cnf
ncu --metrics gpu__time_duration.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,lts__t_bytes.sum.per_second,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__m_xbar2l1tex_read_bytes.sum.per_second,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --kernel-name-base demangled -k regex:TcCnf -c 2 --csv python tools/profile_step.py --config C4 --iters 1 > gpurun_out/ncu_cnf/metrics.csv 2> gpurun_out/ncu_cnf/err.txt
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/ncu_cnf/metrics.csv").read().splitlines()[2:] if False else open("gpurun_out/ncu_cnf/metrics.csv")))
for r in rows:
    if len(r) > 14 and r[0] not in ("ID",):
        print(r[4][:40], r[12], r[13], r[14])
PY
