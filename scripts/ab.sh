#!/bin/bash
# A/B of library builds on the GPU box: LeNet-5 b64 step timing per variant
# (scripts/exp_time.py), then the parity subset on the in-tree library.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/exp_time.py "$@" 2>&1 | tee gpurun_out/ab.txt
timeout 600 python -m pytest tests -m gpu -x -q -k "golden or lenet or batch_parity" 2>&1 | tail -2 | tee -a gpurun_out/ab.txt
