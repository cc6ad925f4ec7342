#!/bin/bash
# compute-sanitizer over one small launch of every kernel family (run under gpurun)
OUT=${1:-gpurun_out}
mkdir -p $OUT
python scripts/sanitize_driver.py > $OUT/sanitize_plain.log 2>&1; echo "plain rc=$?"; tail -1 $OUT/sanitize_plain.log
for tool in memcheck racecheck synccheck initcheck; do
  # --num-cuda-barriers: the NW kernel's per-slot mbarriers over 148 CTAs overflow the default tracking
  timeout 1200 compute-sanitizer --tool $tool --num-cuda-barriers 65536 --print-limit 20 --error-exitcode 7 \
      python scripts/sanitize_driver.py > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/sanitize_$tool.log | tail -1)"
done
