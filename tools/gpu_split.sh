#!/bin/bash
# K2 split-row variant: correctness (compress / scale / layer tests with it as the library) and A/B timing
mkdir -p gpurun_out
cp paper_2603_08055_b200/libgsa_sm100.so /tmp/libgsa_main.so
cp paper_2603_08055_b200/libgsa_split.so paper_2603_08055_b200/libgsa_sm100.so
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 120 -x -k "compress or topk or scale or forward or clustered or oversmoothed or ties or spec or hybrid" > gpurun_out/pytest_split.txt 2>&1
tail -2 gpurun_out/pytest_split.txt; grep -E "^FAILED|^E  " gpurun_out/pytest_split.txt | head -10
cp /tmp/libgsa_main.so paper_2603_08055_b200/libgsa_sm100.so
bash tools/gpu_variants2.sh 2 -- main libgsa_split.so
bash tools/gpu_variants2.sh 1 --data clustered -- main libgsa_split.so; bash tools/gpu_variants2.sh 1 --topk 64 --views 500 -- main libgsa_split.so
