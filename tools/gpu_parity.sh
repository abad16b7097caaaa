#!/bin/bash
# usage: tools/gpu_parity.sh <tag> — full GPU suite (incl. scale parity) + default bench line with its parity field
mkdir -p gpurun_out
TAG=${1:-x}
export GSA_PARITY_LOG=gpurun_out/scale_parity_$TAG.jsonl
rm -f $GSA_PARITY_LOG
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu_$TAG.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_v1000_$TAG.txt 2>&1
tail -25 gpurun_out/pytest_gpu_$TAG.txt; cat $GSA_PARITY_LOG; tail -c 1500 gpurun_out/bench_v1000_$TAG.txt
