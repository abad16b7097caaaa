#!/bin/bash
# K2 anatomy: cycle counters (COMPRESS_PROF) with and without the streaming top-k, and timing without it
mkdir -p gpurun_out
cp paper_2603_08055_b200/libgsa_sm100.so /tmp/libgsa_main.so
for v in libgsa_sm100_prof.so libgsa_prof_notopk.so; do
  cp paper_2603_08055_b200/$v paper_2603_08055_b200/libgsa_sm100.so
  echo "== $v"; timeout 300 python bench.py --views 1000 --steps 1 --warmup 1 --no-cpu-baseline --no-dense --no-e2e --no-parity 2>&1 | grep "prof" | sort | uniq -c | sort -rn | head -8
done
cp /tmp/libgsa_main.so paper_2603_08055_b200/libgsa_sm100.so
bash tools/gpu_variants2.sh 2 -- main libgsa_notopk.so
