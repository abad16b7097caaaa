#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --views 100 --steps 3 --warmup 2 --no-cpu-baseline --no-dense > gpurun_out/bench_v100.txt 2>&1
tail -25 gpurun_out/pytest_gpu.txt; tail -c 2500 gpurun_out/bench_v100.txt
