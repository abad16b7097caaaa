#!/bin/bash
# COMPRESS_PROF build: per-phase cycle counters of K2 (softmax warp 0 and the MMA warp of CTA 0)
# usage: tools/gpu_cprof.sh [debug values...]
cp paper_2603_08055_b200/libgsa_sm100.so /tmp/libgsa_sm100_main.so
cp paper_2603_08055_b200/libgsa_sm100_prof.so paper_2603_08055_b200/libgsa_sm100.so
for d in ${@:-0}; do echo "debug=$d"; GSA_DEBUG_COMPRESS=$d timeout 300 python bench.py --views 1000 --steps 1 --warmup 1 --no-cpu-baseline --no-dense --no-e2e 2>&1 | grep "prof\|stats" | grep -v metric | sort | uniq -c | sort -rn | head -6; done
cp /tmp/libgsa_sm100_main.so paper_2603_08055_b200/libgsa_sm100.so
