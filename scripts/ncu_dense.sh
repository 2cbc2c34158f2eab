#!/bin/bash
# ncu --set full of the digit-row tensor-core kernel on one Dense(1024 -> 1024)
# k = 8 garbler pass over 4096 inferences (BASELINE configs[4] linear sweep)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_linear -s 1 -c 1 \
  -o gpurun_out/tc_dense4096_r02 python scripts/time_linear.py 4096 > gpurun_out/ncu_dense.log 2>&1
tail -2 gpurun_out/ncu_dense.log
