#!/bin/bash
# ncu --set full of the garbling launch (act_kernel<garble>, LeNet-5 b64) and
# of the first evaluation launch (act_kernel<eval>)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-r02}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:act_kernel -s 0 -c 2 \
  -o gpurun_out/act_b64_$tag python scripts/ncu_target.py 64 > gpurun_out/ncu_act_$tag.log 2>&1
tail -2 gpurun_out/ncu_act_$tag.log
