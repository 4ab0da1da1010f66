#!/bin/bash
# sanitize.sh OUT -- compute-sanitizer memcheck / racecheck / synccheck / initcheck over
# tools/sanitize_cases.py (toy sizes, every kernel family).  Run on the GPU box.
out=gpurun_out/${1:-sanitize}
mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool --target-processes all --print-limit 20 python tools/sanitize_cases.py all \
    > $out/$tool.log 2>&1
  echo "$tool rc=$?  $(grep -E 'ERROR SUMMARY' $out/$tool.log | tail -1)"
done
# racecheck (shared-memory hazards) is the slowest tool: one kernel family per process
for c in tc simt cnf conv theta adaptive; do
  timeout 1200 $CS --tool racecheck --racecheck-report all --target-processes all --print-limit 20 \
    python tools/sanitize_cases.py $c > $out/racecheck_$c.log 2>&1
  echo "racecheck $c rc=$?  $(grep -E 'RACECHECK SUMMARY|ERROR SUMMARY' $out/racecheck_$c.log | tail -1)"
done
