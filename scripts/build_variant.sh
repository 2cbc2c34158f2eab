#!/bin/bash
# Build a tuning variant of libdashgpu.so into variants/<name>.so with extra
# nvcc flags (e.g. -DDASH_GARBLE_WARPS=24); variants/ is git-ignored but
# travels to the GPU box for scripts/exp_time.py A/B runs.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p variants
make -s -C paper_2302_06361_b200/csrc OUT=$PWD/variants/$name.so BUILD=$PWD/variants/build_$name NVCC="nvcc $*" > /dev/null
echo "variants/$name.so"
