#!/bin/bash
# compute-sanitizer over every libharag kernel (tests/sanitize_driver.py, tiny shapes, outputs checked
# against the oracle): memcheck (+ leak check), racecheck (shared-memory hazards), synccheck (barrier
# misuse), initcheck (reads of uninitialised device memory).  Raw logs and a classified summary
# (tools/sanitize_summary.py) in gpurun_out/sanitize/.
mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck initcheck initcheck_nopass16; do
  if [ "$tool" = initcheck_nopass16 ]; then export HARAG_SAN_NO_PASS16=1; t=initcheck; else t=$tool; fi
  extra="--print-limit 200"
  [ "$t" = memcheck ] && extra="$extra --leak-check full"
  [ "$t" = initcheck ] && extra="--print-limit 100000"
  timeout 1500 compute-sanitizer --tool $t $extra --error-exitcode 99 \
    python tests/sanitize_driver.py > gpurun_out/sanitize/$tool.txt 2>&1
  echo "== $tool rc=$?" | tee gpurun_out/sanitize/$tool.summary.txt
  python tools/sanitize_summary.py gpurun_out/sanitize/$tool.txt | tee -a gpurun_out/sanitize/$tool.summary.txt
  grep -h "sanitize_driver ok" gpurun_out/sanitize/$tool.txt | tee -a gpurun_out/sanitize/$tool.summary.txt
  # keep the raw log small (gpurun brings back <= 64 MiB): its head and the summary lines
  { head -n 300 gpurun_out/sanitize/$tool.txt; echo "[... truncated ...]"; grep "SUMMARY" gpurun_out/sanitize/$tool.txt; } \
    > gpurun_out/sanitize/$tool.head.txt
  rm -f gpurun_out/sanitize/$tool.txt
done
