#!/bin/bash
# Round evidence on one B200 (gpurun -- bash scripts/gpu_evidence.sh): smoke, full bench line,
# ncu launch list of a short bench, ncu --set full of the top kernels (one launch each).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log > gpurun_out/bench_line.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-dense --e2e-steps 1 > gpurun_out/b_ncu.log 2>&1; echo "ncu launches rc=$?"
python scripts/ncu_sum.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'tc_diag|tc_pass|kv_cand' -c 3 \
    -o gpurun_out/full_r02 python scripts/run_once.py 131072 > gpurun_out/full.log 2>&1; echo "ncu full rc=$?"
