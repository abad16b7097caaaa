#!/bin/bash
mkdir -p gpurun_out
cp paper_2603_08055_b200/libgsa_sm100.so /tmp/libgsa_main.so
cp paper_2603_08055_b200/libgsa_splitwd.so paper_2603_08055_b200/libgsa_sm100.so
timeout 240 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "test_compress_topk_exact" > gpurun_out/pytest_split2.txt 2>&1
echo "exit $?"; tail -5 gpurun_out/pytest_split2.txt; grep -E "watchdog|^E  " gpurun_out/pytest_split2.txt | head -10
cp /tmp/libgsa_main.so paper_2603_08055_b200/libgsa_sm100.so
