set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo gputest rc=$?; tail -3 gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -c 3000 gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/b_ncu.log 2>&1; echo ncu rc=$?
bash scripts/sanitize.sh
