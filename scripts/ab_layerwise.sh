#!/bin/bash
# A/B of dashgpu_infer's whole-GC vs layer-windowed sub-batches on the
# configs whose GCs exceed HBM (MiniONN b256, ResNet-20 b512), plus the
# streamed-garbling parity tests.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_streamed.py -m gpu -x -q 2>&1 | tail -3
for cfg in "minionn 9 256" "resnet20 8 512"; do
  set -- $cfg
  for lw in 0 auto; do
    if [ $lw = auto ]; then unset DASHGPU_LAYERWISE; else export DASHGPU_LAYERWISE=$lw; fi
    timeout 900 python bench.py --model $1 --k $2 --batch $3 --steps 2 --warmup 3 --no-cpu \
      > gpurun_out/lw_$1_$lw.json 2> gpurun_out/lw_$1_$lw.err
    python - "$1" "$lw" <<'PY'
import json, sys
l = json.loads(open(f"gpurun_out/lw_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
c = l["config"]; print(sys.argv[1], sys.argv[2], l["value"], l["e2e"]["value"], c.get("sub_batches_per_step"), c.get("schedule"), l["ms_per_step"])
PY
  done
done
