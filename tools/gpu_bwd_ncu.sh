#!/bin/bash
# ncu --set full of the backward's tensor-core kernels at 100 views (dense passes, selection passes, projection)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"bwd_tc_kernel|sel_bwd_tc_kernel" -c 6 -o gpurun_out/bwd_v100 -f \
  python tools/bwd_timing.py --views 100 --ncu > gpurun_out/bwd_ncu.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/bwd_ncu.log
bash tools/gpu_bwd_launches.sh 1000
bash tools/gpu_bwd_launches.sh 100
