#!/bin/bash
# tensor-core linear knobs (env) on the Dense(1024 -> 1024) k = 8 sweep point
cd "$(dirname "$0")/.."
for env in "" "DASH_TC_RS=2" "DASH_TC_BNMAX=128" "DASH_TC_BNMAX=128 DASH_TC_RS=2"; do
  env $env python bench.py --sweep linear --sweep-log2 24 --sweep-k 8 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('[$env]', d['labels'], 'lin ms %.2f'%d['linear_kernel_ms'], 'int8 %.3g'%d['int8_ops_per_s_kernel'])"
done
