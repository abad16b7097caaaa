#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -k "compress or topk or scale or spec or forward or clustered or oversmoothed or ties" > gpurun_out/pytest_r02r.txt 2>&1
tail -2 gpurun_out/pytest_r02r.txt; grep -E "^FAILED|^E  .*assert" gpurun_out/pytest_r02r.txt | head -10
cp paper_2603_08055_b200/libgsa_sm100.so /tmp/libgsa_main.so
cp paper_2603_08055_b200/libgsa_sm100_prof.so paper_2603_08055_b200/libgsa_sm100.so
timeout 300 python bench.py --views 1000 --steps 1 --warmup 1 --no-cpu-baseline --no-dense --no-e2e --no-parity 2>&1 | grep "compress prof" | sort -u
cp /tmp/libgsa_main.so paper_2603_08055_b200/libgsa_sm100.so
bash tools/gpu_variants2.sh 2 -- main libgsa_head.so
bash tools/gpu_variants2.sh 1 --data clustered -- main
