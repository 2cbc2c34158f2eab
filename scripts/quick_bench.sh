#!/bin/bash
# quick A/B timing on the GPU box: parity subset + the headline bench line
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests -m gpu -x -q -k "golden or lenet or tensor_core or streamed or extension" 2>&1 | tail -1
timeout 200 python bench.py --no-cpu --steps 5 --warmup 3 > gpurun_out/qb.json 2>gpurun_out/qb.err || tail -3 gpurun_out/qb.err
python -c "import json;d=json.load(open('gpurun_out/qb.json'));print('inf/s %.1f'%d['value'],{k:round(v,2) for k,v in d['kernels_ms_per_step'].items()})"
