#!/bin/bash
# compute-sanitizer over this round's kernels: the digit-row tensor-core
# kernel on the window-TMA path (dense1024, batch 8, single CTAs and CTA
# pairs), the expanded-digit kernel and chunked garbling (LeNet-5 batch 2)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py dense1024:8 \
    > gpurun_out/sanitizer/${tool}_dense1024.txt 2>&1
  echo "$tool dense1024: $(tail -1 gpurun_out/sanitizer/${tool}_dense1024.txt)"
done
DASH_TC_CG=2 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py dense1024:8 \
  > gpurun_out/sanitizer/memcheck_dense1024_pairs.txt 2>&1
echo "memcheck dense1024 pairs: $(tail -1 gpurun_out/sanitizer/memcheck_dense1024_pairs.txt)"
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py lenet5:2 \
  > gpurun_out/sanitizer/memcheck_lenet5.txt 2>&1
echo "memcheck lenet5: $(tail -1 gpurun_out/sanitizer/memcheck_lenet5.txt)"
for tool in memcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_stream.py \
    > gpurun_out/sanitizer/${tool}_stream.txt 2>&1
  echo "$tool stream: $(tail -1 gpurun_out/sanitizer/${tool}_stream.txt)"
done
