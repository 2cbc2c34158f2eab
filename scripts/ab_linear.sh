#!/bin/bash
# A/B of tensor-core linear builds on the Dense(1024 -> 1024) sweep point
# (k = 8, B = 4096 and 16384): in-tree library vs variants/*.so given as args,
# then the tensor-core parity tests on the in-tree library
cd "$(dirname "$0")/.."
for lib in "" "$@"; do
  for j in 22 24; do
    DASHGPU_LIB=$lib python bench.py --sweep linear --sweep-log2 $j --sweep-k 8 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('[${lib:-in-tree}]', d['labels'], 'lin ms %.2f'%d['linear_kernel_ms'], 'int8 %.3g'%d['int8_ops_per_s_kernel'])"
  done
done
timeout 600 python -m pytest tests -m gpu -x -q -k "tensor_core or linear or lenet_batch or golden" 2>&1 | tail -2
