#!/bin/bash
# All BASELINE configs on one B200 -> gpurun_out/measure/*.json (copied to profiles/ by hand)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/measure
timeout 600 python bench.py > gpurun_out/measure/headline.json 2> gpurun_out/measure/headline.err
timeout 600 python bench.py --impl reference > gpurun_out/measure/reference.json 2> gpurun_out/measure/reference.err
for cfg in "model_a 8 1" "model_a 8 64" "lenet5 8 64 --private" "minionn 9 256" "resnet20 8 512"; do
  set -- $cfg
  tag="$1_b$3${4:+_private}"
  timeout 1200 python bench.py --model $1 --k $2 --batch $3 $4 --steps 3 --warmup 3 --no-cpu \
    > gpurun_out/measure/$tag.json 2> gpurun_out/measure/$tag.err
done
# BASELINE configs[4]: the whole grid, k = 2..8 x N = 2^16..2^26 (even powers)
G="--sweep-log2 16,18,20,22,24,26 --sweep-k 2,3,4,5,6,7,8"
timeout 1500 python bench.py --sweep proj $G > gpurun_out/measure/sweep_proj.jsonl 2> gpurun_out/measure/sweep_proj.err
timeout 900 python bench.py --sweep tproj $G > gpurun_out/measure/sweep_tproj.jsonl 2> gpurun_out/measure/sweep_tproj.err
timeout 900 python bench.py --sweep linear $G > gpurun_out/measure/sweep_linear.jsonl 2> gpurun_out/measure/sweep_linear.err
tail -n 3 gpurun_out/measure/sweep_*.err
for f in gpurun_out/measure/*.json; do echo "$f: $(python -c "import json,sys;d=json.load(open('$f'));print(round(d.get('value',0),2), d.get('unit'))" 2>&1 | tail -1)"; done
