#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the hot path
# (tools/sanitize_run.py); logs to gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  [ "$tool" = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra \
      --print-limit 5000 python tools/sanitize_run.py > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}.log | tail -1)"
  # distinct hazard sites
  grep -oE "(Write|Read) Thread \([0-9]+,0,0\) at [^ ]+ in [a-z_.]+:[0-9]+" gpurun_out/sanitize_${tool}.log \
      | sed -E 's/Thread \([0-9]+,0,0\) at ([a-zA-Z_:<>]+)[^ ]* in/\1 in/' | sort | uniq -c | head -20
done
