#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_bwd_launches.sh 1000
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"sel_bwd_tc" -c 2 -o gpurun_out/selbwd_v100 -f python tools/bwd_timing.py --views 100 --ncu > gpurun_out/selbwd_ncu.log 2>&1
echo "ncu exit $?"
