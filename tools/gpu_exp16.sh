#!/bin/bash
# K5 exp2 in f16x2: tiled-attention parity with each variant as the library, then A/B timing
mkdir -p gpurun_out
cp paper_2603_08055_b200/libgsa_sm100.so /tmp/libgsa_main.so
for v in libgsa_exp16_1.so libgsa_exp16_2.so; do
  cp paper_2603_08055_b200/$v paper_2603_08055_b200/libgsa_sm100.so
  timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "tiled or special or forward_matches or golden or hybrid or cpp or scale_parity" > gpurun_out/pytest_$v.txt 2>&1
  echo "$v: $(tail -1 gpurun_out/pytest_$v.txt)"; grep -E "^E  .*assert" gpurun_out/pytest_$v.txt | head -4
done
cp /tmp/libgsa_main.so paper_2603_08055_b200/libgsa_sm100.so
bash tools/gpu_variants2.sh 2 -- main libgsa_exp16_1.so libgsa_exp16_2.so
