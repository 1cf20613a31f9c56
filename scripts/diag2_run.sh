#!/bin/bash
# A/B of the two-tile diagonal kernel (S2O_DIAG2=1) against tc_diag_kernel: parity, then time
# (args: abv/<variant> builds to time as well).
cd "$(dirname "$0")/.."
{
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k "variant" 2>&1 | tail -5
S2O_DIAG2=1 timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -x -q 2>&1 | tail -5
python scripts/p1_time.py
S2O_DIAG2=1 python scripts/p1_time.py
for v in "$@"; do S2O_DIAG2=1 S2O_LIB_PATH=abv/$v/lib/libs2o_cuda.so timeout 120 python scripts/p1_time.py; done
} > gpurun_out/d2.txt 2>&1
