#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py; summaries to $1 (default gpurun_out)
out=${1:-gpurun_out}
for tool in memcheck racecheck synccheck initcheck; do
  for c in factors fwht pair ff16k fused-ffma2 fused-tcgen05 head; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 python tools/sanitize_cases.py $c \
      > $out/san_${tool}_$c.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $out/san_${tool}_$c.log | tail -1)"
  done
done
