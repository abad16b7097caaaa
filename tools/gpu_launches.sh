#!/bin/bash
# usage: tools/gpu_launches.sh <tag> [views]  — ncu launch list (per-kernel device time) of one bench step
mkdir -p gpurun_out
TAG=${1:-x}; V=${2:-1000}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --views $V --steps 1 --warmup 1 --no-dense --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/launches_$TAG.csv
