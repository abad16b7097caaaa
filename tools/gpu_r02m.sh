#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -k "select or sparse or forward or hybrid or spec or scale or cpp or dist or stack" > gpurun_out/pytest_r02m.txt 2>&1
tail -2 gpurun_out/pytest_r02m.txt; grep -E "^FAILED" gpurun_out/pytest_r02m.txt | head
bash tools/gpu_variants2.sh 2 -- main libgsa_head.so
