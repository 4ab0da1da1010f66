#!/bin/bash
# ncu_capture.sh NAME KERNEL_REGEX -- CMD...   (run on the GPU box)
# Full-section capture of one launch of the kernel, exported to small CSVs in
# gpurun_out/ (the .ncu-rep itself embeds the whole cubin and is too large to
# bring back).
name=$1; shift; regex=$1; shift; [ "$1" = "--" ] && shift
rep=/tmp/${name}.ncu-rep
mkdir -p $(dirname $rep) $(dirname gpurun_out/${name})
ncu $(cat tools/ncu_sections.txt) --clock-control none --import-source on -k regex:${regex} -s 1 -c 1 -f -o ${rep%.ncu-rep} "$@" > gpurun_out/${name}_ncu.log 2>&1
ncu -i $rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
ncu -i $rep --page details --csv > gpurun_out/${name}_details.csv 2>/dev/null
ncu -i $rep --page source --csv --print-source cuda,sass > gpurun_out/${name}_source.csv 2>/dev/null
gzip -f gpurun_out/${name}_source.csv
ls -la gpurun_out/${name}_*
