#!/bin/bash
# usage: tools/gpu_round.sh <tag>  — gpu tests, V=100 and V=1000 bench lines, V=1000 launch list
mkdir -p gpurun_out
TAG=${1:-x}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu_$TAG.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_$TAG.txt 2>&1
timeout 400 python bench.py --views 100 --steps 5 --warmup 3 > gpurun_out/bench_v100_$TAG.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_v1000_$TAG.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v1000_$TAG.csv python bench.py --steps 2 --warmup 1 --no-dense --no-cpu-baseline --no-e2e > /dev/null 2>&1
tail -3 gpurun_out/pytest_gpu_$TAG.txt; tail -2 gpurun_out/smoke_$TAG.txt; tail -c 1500 gpurun_out/bench_v100_$TAG.txt; tail -c 2500 gpurun_out/bench_v1000_$TAG.txt
