#!/bin/bash
# Round-end refresh without the ncu captures (kernels unchanged since the last profile_round): -m gpu suite, smoke, every config and the configs[4] grid
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/gpu_tests.txt 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.txt
tail -3 gpurun_out/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
bash scripts/measure_all.sh
