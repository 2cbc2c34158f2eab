#!/bin/bash
# Evidence for profiles/: launch list of the bench command (cold-cache,
# serialised: compare shares), ncu --set full of the dominant kernel
# (act_kernel<garble>, LeNet-5 b64) and of the tensor-core linear kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/bench_launches.csv python bench.py --no-cpu --steps 2 --warmup 1 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/bench_launches.csv > gpurun_out/bench_launch_list.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:act_kernel -s 0 -c 1 \
  -o gpurun_out/act_garble_b64 python scripts/ncu_target.py 64 > gpurun_out/ncu_act.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_linear -s 0 -c 8 \
  -o gpurun_out/tc_linear_b64 python scripts/ncu_target.py 64 > gpurun_out/ncu_tc.log 2>&1
tail -n 2 gpurun_out/ncu_act.log gpurun_out/ncu_tc.log
cat gpurun_out/bench_launch_list.txt
