mkdir -p gpurun_out/ab
for i in 1 2; do
for v in old new; do
  if [ $v = old ]; then export OB_LIB_VARIANT=tools/libodeblock_old.so; else unset OB_LIB_VARIANT; fi
  timeout 300 python bench.py --per-config "" --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab/$v$i.json 2>gpurun_out/ab/$v$i.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab/$v$i.json').read().splitlines()[-1]);print('$v', d['value'],d['ms_per_step'],d['roofline']['phase_ms_per_step'])"
done; done
