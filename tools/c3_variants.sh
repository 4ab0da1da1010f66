#!/bin/bash
# c3_variants.sh V1 V2 ... -- C3 phase profile (cycles per CTA) for library variants (base = in-tree)
for v in "$@"; do
  if [ $v = base ]; then unset OB_LIB_VARIANT; else export OB_LIB_VARIANT=tools/libodeblock_$v.so; fi
  echo "== $v"; timeout 200 python tools/profile_step.py --config C3 --iters 2 --phases 2>&1 | tail -9
done
