#!/bin/bash
# compute-sanitizer over the tiny config (tools/sanitize_tiny.py); summaries to gpurun_out/sanitize/
mkdir -p gpurun_out/sanitize
python tools/sanitize_tiny.py > gpurun_out/sanitize/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
for T in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $T --print-limit 20 --error-exitcode 9 \
      python tools/sanitize_tiny.py > gpurun_out/sanitize/$T.log 2>&1
  echo "$T rc=$?" >> gpurun_out/sanitize/summary.txt
  tail -3 gpurun_out/sanitize/$T.log >> gpurun_out/sanitize/summary.txt
done
