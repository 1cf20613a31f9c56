#!/bin/bash
# compute-sanitizer over scripts/sanitize_case.py (small configs of every kernel family), one tool at a
# time; summaries into gpurun_out/sanitizer_<tool>.txt (run on the GPU box: gpurun -- bash scripts/sanitize.sh)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --target-processes all \
      python scripts/sanitize_case.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "== $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Hazard|error' gpurun_out/sanitizer_$tool.txt | tail -3 | tr '\n' ' ')"
done
