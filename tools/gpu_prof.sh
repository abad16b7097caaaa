#!/bin/bash
# usage: tools/gpu_prof.sh <kernel-regex> <tag> [views]
# tests (gpu), a bench line, the launch list and one ncu --set full capture of <kernel-regex>
mkdir -p gpurun_out
K=${1:-select_tc}; TAG=${2:-x}; V=${3:-100}
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu_$TAG.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.txt
timeout 400 python bench.py --views $V --steps 3 --warmup 2 --no-cpu-baseline --no-dense > gpurun_out/bench_$TAG.txt 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --views $V --steps 2 --warmup 1 --no-dense --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_$TAG python bench.py --views $V --steps 1 --warmup 1 --no-dense --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/pytest_gpu_$TAG.txt; tail -c 1500 gpurun_out/bench_$TAG.txt; tail -3 gpurun_out/ncu_$TAG.log
