#!/bin/bash
# ncu --set full of the evaluation launch of LeNet-5's first ReLU layer
# (act_kernel<0>, the second act_kernel launch of a pass) and of the first
# act_out_kernel (garbler output labels), LeNet-5 b64.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:act_kernel -s 1 -c 1 \
  -o gpurun_out/act_eval_b64 python scripts/ncu_target.py 64 > gpurun_out/ncu_eval.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:act_out_kernel -s 0 -c 1 \
  -o gpurun_out/act_out_b64 python scripts/ncu_target.py 64 > gpurun_out/ncu_out.log 2>&1
tail -n 2 gpurun_out/ncu_eval.log gpurun_out/ncu_out.log
