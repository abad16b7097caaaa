#!/bin/bash
mkdir -p gpurun_out
cp paper_2603_08055_b200/libgsa_sm100.so /tmp/libgsa_main.so
cp paper_2603_08055_b200/libgsa_fastream2.so paper_2603_08055_b200/libgsa_sm100.so
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "tiled or special or forward or golden or hybrid or cpp or dense or v100 or spec" > gpurun_out/pytest_fastream.txt 2>&1
tail -2 gpurun_out/pytest_fastream.txt; grep -E "^FAILED|^E  .*assert" gpurun_out/pytest_fastream.txt | head -6
cp /tmp/libgsa_main.so paper_2603_08055_b200/libgsa_sm100.so
bash tools/gpu_variants2.sh 2 -- main libgsa_fastream1.so libgsa_fastream2.so libgsa_fastream4.so
