#!/bin/bash
# Round evidence on one B200 (gpurun -- bash scripts/gpu_evidence.sh): smoke, full bench line,
# ncu launch list of a short bench, ncu --set full of the pass kernels and of kv_cand, tau sweep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log > gpurun_out/bench_line.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-dense --e2e-steps 1 > gpurun_out/b_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'tc_diag|tc_pass' -c 2 \
    -o gpurun_out/full_r02 python scripts/run_once.py 131072 > gpurun_out/full.log 2>&1; echo "ncu full rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'kv_cand|q_rank|sel_sort' -c 3 \
    -o gpurun_out/plan_r02 python scripts/plan_c3_once.py > gpurun_out/planfull.log 2>&1; echo "ncu plan rc=$?"
[ "$1" = "sweep" ] && { timeout 1800 python scripts/tau_sweep.py --out gpurun_out/tau_sweep_r02.json > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"; }
true
