#!/bin/bash
# compute-sanitizer over profiles/sanitize_run.py (every algorithm of the C ABI on a
# small R-MAT graph, checked against the oracle): memcheck, racecheck (shared memory),
# synccheck.  Summaries -> gpurun_out/sanitize_<tool>.txt
cd "$(dirname "$0")/.."
for tool in memcheck racecheck synccheck; do
  timeout 400 compute-sanitizer --tool $tool --print-limit 20 python profiles/sanitize_run.py \
    > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.txt >> gpurun_out/sanitize_summary.txt
done
