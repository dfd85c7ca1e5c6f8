#!/bin/bash
# compute-sanitizer over one small invocation of every libmm kernel path (tools/sanitize_paths.py):
# memcheck, racecheck (shared-memory hazards), synccheck (barrier misuse), initcheck.
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for cfg in c1 small; do
    timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_paths.py $cfg > gpurun_out/san_${tool}_${cfg}.log 2>&1
    echo "$tool $cfg rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san_${tool}_${cfg}.log | tail -2 | tr '\n' ' ')"
  done
done
