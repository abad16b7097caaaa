#!/bin/bash
# round-2 pass: the whole GPU suite (no -x) + one ncu --set full capture of the V=1000 step's hot kernels
mkdir -p gpurun_out
T=${1:-r02k}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu_$T.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$T.txt
tail -3 gpurun_out/pytest_gpu_$T.txt; grep -E "^FAILED" gpurun_out/pytest_gpu_$T.txt | head
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"compress_tc|fa_tc|rescore|pool_kernel" -c 5 -o gpurun_out/prof_$T \
  python bench.py --views 1000 --steps 1 --warmup 0 --no-dense --no-cpu-baseline --no-e2e --no-parity > gpurun_out/ncu_$T.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/ncu_$T.log
