#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -k "sparse or select or forward or hybrid or dist" > gpurun_out/pytest_r02w.txt 2>&1
tail -2 gpurun_out/pytest_r02w.txt; grep -E "^FAILED" gpurun_out/pytest_r02w.txt | head
bash tools/gpu_variants2.sh 3 -- main libgsa_nohint.so
