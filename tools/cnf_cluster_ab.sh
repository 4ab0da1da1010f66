#!/bin/bash
# C4 tcgen05 tile: parity + timing for weight-stream cluster sizes 1 / 2 / 4
for cl in ${CLS:-1 2 4}; do
  echo "== OB_CNF_CLUSTER=$cl"
  OB_CNF_CLUSTER=$cl timeout 300 python tools/cnf_tc_check.py 2>&1 | grep -v simt | grep -v "^frame" | head -12
done
