#!/bin/bash
# launch list of Model A batch 1 (BASELINE configs[0]) and ncu of its garbling launch
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/model_a_b1_launches.csv python bench.py --model model_a --batch 1 --no-cpu --steps 2 --warmup 1 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/model_a_b1_launches.csv > gpurun_out/model_a_b1_launch_list.txt
cat gpurun_out/model_a_b1_launch_list.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:act_lv_garble -s 0 -c 1 \
  -o gpurun_out/model_a_b1_lv python scripts/ncu_target.py 1 model_a > /dev/null 2>&1
echo done
