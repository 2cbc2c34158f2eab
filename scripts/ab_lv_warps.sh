#!/bin/bash
# A/B of the level-parallel garbling shape for batch-1 launches (Model A b1):
# DASH_LV_WARPS = warps per element cap, DASH_LV_CTAS = 16-warp CTAs per SM assumed resident
cd "$(dirname "$0")/.."
for cfg in "8 1" "16 2" "16 3" "16 4"; do
  set -- $cfg
  export DASH_LV_WARPS=$1 DASH_LV_CTAS=$2
  r=$(timeout 300 python -m pytest tests/test_engine.py tests/test_batch_parity.py -m gpu -x -q -k "model_a or level or lane_group" 2>&1 | tail -1)
  v=$(timeout 300 python bench.py --model model_a --k 8 --batch 1 --steps 200 --warmup 20 --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(d['value'],1),round(d['e2e']['value'],1),{k:round(v,3) for k,v in d['kernels_ms_per_step'].items()})")
  echo "W=$1 ctas=$2 | $r | $v"
done
