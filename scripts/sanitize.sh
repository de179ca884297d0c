#!/bin/bash
# compute-sanitizer over scripts/sanitize_driver.py (on a B200 box):
#   bash scripts/sanitize.sh OUTDIR
# one log per tool; the summary lines are copied into profiles/ by hand.
out=${1:-gpurun_out}
mkdir -p $out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python scripts/sanitize_driver.py > $out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|FAILS' $out/sanitize_$tool.log | tr '\n' ' ')"
done
