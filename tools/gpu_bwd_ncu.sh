#!/bin/bash
# ncu --set full of the backward's dense and selection kernels at 100 views
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"dense_bwd_dkdv|dense_bwd_dq|sel16_bwd" -c 4 -o gpurun_out/bwd_v100 -f \
  python tools/bwd_timing.py --views 100 --ncu > gpurun_out/bwd_ncu.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/bwd_ncu.log
