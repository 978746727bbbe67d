#!/bin/bash
# compute-sanitizer over every libharag kernel (tests/sanitize_driver.py, tiny shapes, outputs checked
# against the oracle): memcheck, racecheck (shared-memory hazards), synccheck (barrier misuse),
# initcheck (reads of uninitialised device memory).  Logs in gpurun_out/sanitize/.
mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 99 \
    python tests/sanitize_driver.py > gpurun_out/sanitize/$tool.txt 2>&1
  echo "$tool rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY\|LEAK SUMMARY' gpurun_out/sanitize/$tool.txt | tr '\n' ' ')"
done
