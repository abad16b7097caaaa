#!/bin/bash
# compute-sanitizer memcheck + racecheck over the backward tests (every backward kernel at small sizes)
mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_backward.py -m gpu -q -p no:cacheprovider -x \
  -k "reference_context or bf16 or pool_and_upsample or rejects or project" > gpurun_out/sanitize_bwd.txt 2>&1
echo "memcheck exit $?"; grep -E "ERROR SUMMARY|passed|failed|Invalid|out of bounds" gpurun_out/sanitize_bwd.txt | head -10
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_backward.py -m gpu -q -p no:cacheprovider -x \
  -k "reference_context" > gpurun_out/racecheck_bwd.txt 2>&1
echo "racecheck exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|hazard" gpurun_out/racecheck_bwd.txt | head -10
