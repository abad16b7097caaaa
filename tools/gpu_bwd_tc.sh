#!/bin/bash
# tensor-core backward bring-up: backward tests first (bounded), then timing
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_backward.py -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_bwd_tc.txt
echo "pytest exit ${PIPESTATUS[0]}"; tail -25 gpurun_out/pytest_bwd_tc.txt
if grep -q "passed" gpurun_out/pytest_bwd_tc.txt && ! grep -q "failed" gpurun_out/pytest_bwd_tc.txt; then
  timeout 600 python tools/bwd_timing.py --views 100,1000 2>&1 | tee gpurun_out/bwd_timing_tc.jsonl
fi
