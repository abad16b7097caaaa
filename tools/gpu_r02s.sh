#!/bin/bash
mkdir -p gpurun_out
cp paper_2603_08055_b200/libgsa_sm100.so /tmp/libgsa_main.so
cp paper_2603_08055_b200/libgsa_sm100_prof.so paper_2603_08055_b200/libgsa_sm100.so
timeout 300 python bench.py --views 1000 --steps 1 --warmup 1 --no-cpu-baseline --no-dense --no-e2e --no-parity 2>&1 | grep "compress prof" | sort -u
cp /tmp/libgsa_main.so paper_2603_08055_b200/libgsa_sm100.so
bash tools/gpu_variants2.sh 2 -- main ${1:-libgsa_head2.so}
