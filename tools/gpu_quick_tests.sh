#!/bin/bash
# usage: tools/gpu_quick_tests.sh <tag> <pytest args...>
mkdir -p gpurun_out
TAG=$1; shift
timeout 1500 python -m pytest -q -p no:cacheprovider --durations=10 "$@" > gpurun_out/pytest_$TAG.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.txt
tail -30 gpurun_out/pytest_$TAG.txt
