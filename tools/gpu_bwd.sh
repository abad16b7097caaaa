#!/bin/bash
# backward: GPU tests (backward + C++ drop-in), timing at 100/300/1000 views, ncu launch list at 100 views
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_backward.py tests/test_cpp_api.py -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_bwd.txt
tail -5 gpurun_out/pytest_bwd.txt
timeout 900 python tools/bwd_timing.py --views ${VIEWS:-100,300,1000} 2>&1 | tee gpurun_out/bwd_timing.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/bwd_launches_v100.csv python tools/bwd_timing.py --views 100 --ncu > /dev/null 2>&1
echo "ncu exit $?"
