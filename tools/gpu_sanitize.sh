#!/bin/bash
# compute-sanitizer memcheck over small GPU cases of every kernel path (tensor-core selection
# in bf16 / f32 / packed-stride modes, CSR plans, the layer incl. hybrid, tiled attention)
mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x \
  -k "block_sparse or plan_and_block or forward_with_plan or golden or hybrid_fast or tiled_attention_tc or small_k or compress or pool or gate" > gpurun_out/sanitize.txt 2>&1
echo "exit $?"; grep -E "ERROR SUMMARY|passed|failed|Invalid|out of bounds" gpurun_out/sanitize.txt | head -20
