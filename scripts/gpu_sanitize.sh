#!/bin/bash
# compute-sanitizer over scripts/sanitize.py (eager + graph map-update steps, inference, checkpoint)
mkdir -p gpurun_out
OUT=gpurun_out/sanitizer.txt; : > $OUT
for t in memcheck racecheck synccheck initcheck; do
  echo "=== sanitizer_$t (compute-sanitizer --tool $t python scripts/sanitize.py)" >> $OUT
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize.py >> $OUT 2>&1
  echo "rc=$?" >> $OUT
done
grep -E "===|SUMMARY|ok|rc=" $OUT
