#!/bin/bash
# first GPU validation: environment, gpu tests, smoke, short bench, launch list
mkdir -p gpurun_out
{ nvidia-smi; free -g; nproc; lscpu | grep -E "Model name|Socket|Thread|Core"; } > gpurun_out/env.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --views 100 --steps 3 --warmup 2 > gpurun_out/bench_v100.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v100.csv python bench.py --views 100 --steps 2 --warmup 1 --no-dense --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/smoke.txt | tail -3; tail -c 3000 gpurun_out/bench_v100.txt
