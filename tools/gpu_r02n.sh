#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_r02n.txt 2>&1
tail -2 gpurun_out/pytest_r02n.txt; grep -E "^FAILED|^E  .*assert" gpurun_out/pytest_r02n.txt | head -20
bash tools/gpu_variants2.sh 2 -- main libgsa_head.so
