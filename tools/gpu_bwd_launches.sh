#!/bin/bash
# launch list of one backward (attention part) at the given views
mkdir -p gpurun_out
V=${1:-1000}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/bwd_launches_v$V.csv python tools/bwd_timing.py --views $V --ncu > /dev/null 2>&1
echo "ncu exit $?"
