#!/bin/bash
# compute-sanitizer over scripts/sanitize_case.py (small configs of every kernel family), one tool at a
# time; full logs into gpurun_out/sanitizer_<tool>.txt plus a per-kernel / per-source-line digest
# (run on the GPU box: gpurun -- bash scripts/sanitize.sh [tools...])
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tools="${*:-memcheck racecheck synccheck initcheck}"
for tool in $tools; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 100000 --target-processes all \
      python scripts/sanitize_case.py > gpurun_out/sanitizer_$tool.txt 2>&1
  rc=$?
  echo "== $tool rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitizer_$tool.txt | tail -1)"
  # digest: which kernel / source line each reported access comes from
  grep -oE '(Write|Read|by) [Tt]hread \([0-9,]+\) (in block \([0-9,]+\) )?at [^+]+\+0x[0-9a-f]+ in [a-z_0-9.]+:[0-9]+|at [a-zA-Z_:0-9]+\(.*\)\+0x[0-9a-f]+ in [a-z_0-9.]+:[0-9]+' \
      gpurun_out/sanitizer_$tool.txt | sed -E 's/\([0-9,]+\)//g; s/\+0x[0-9a-f]+//' | sort | uniq -c | sort -rn | head -20
  grep -E '^[A-Za-z]*Error|RuntimeError|sanitize case done' gpurun_out/sanitizer_$tool.txt | tail -2
done
