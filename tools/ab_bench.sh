#!/bin/bash
# ab_bench.sh V1 V2 ... -- C2 bench lines for library variants (base = the in-tree build)
mkdir -p gpurun_out/ab
for i in 1 2; do
for v in "$@"; do
  if [ $v = base ]; then unset OB_LIB_VARIANT; else export OB_LIB_VARIANT=tools/libodeblock_$v.so; fi
  timeout 300 python bench.py --per-config "" --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab/$v$i.json 2>gpurun_out/ab/$v$i.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab/$v$i.json').read().splitlines()[-1]);p=d['roofline']['phase_ms_per_step'];print('%-8s %.4g samples/s  fwd %.3f ms  rev %.3f ms' % ('$v', d['value'], p['ms_forward'], p['ms_reverse']))"
done; done
