#!/bin/bash
# timing aids / A/B builds of the two-tile diagonal kernel (abv/<variant> builds, args = names)
cd "$(dirname "$0")/.."
{
S2O_DIAG2=1 python scripts/p1_time.py
S2O_POISON_CHECK=0 S2O_DIAG2=1 python scripts/p1_time.py
for v in "$@"; do S2O_DIAG2=1 S2O_LIB_PATH=abv/$v/lib/libs2o_cuda.so timeout 120 python scripts/p1_time.py; S2O_POISON_CHECK=0 S2O_DIAG2=1 S2O_LIB_PATH=abv/$v/lib/libs2o_cuda.so timeout 120 python scripts/p1_time.py; done
} > gpurun_out/d2v.txt 2>&1
