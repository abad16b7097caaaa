#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x -k "compress or topk or clustered or oversmoothed or ties or scale_parity" > gpurun_out/pytest_pf.txt 2>&1
tail -2 gpurun_out/pytest_pf.txt; grep -E "^FAILED|^E  " gpurun_out/pytest_pf.txt | head -5
bash tools/gpu_variants2.sh 2 -- main libgsa_nopf.so
