#!/bin/bash
# usage: tools/gpu_ncu.sh <tag> <views> [kernel-regex] [count]
# one ncu --set full capture of the hot kernels of a bench step (single GPU)
mkdir -p gpurun_out
TAG=${1:-x}; V=${2:-100}; K=${3:-"compress_tc|fa_tc|select_tc|pool_kernel"}; C=${4:-4}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -c $C -o gpurun_out/prof_$TAG \
  python bench.py --views $V --steps 1 --warmup 0 --no-dense --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_$TAG.log
tail -5 gpurun_out/ncu_$TAG.log
