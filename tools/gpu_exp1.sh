#!/bin/bash
mkdir -p gpurun_out
cp paper_2603_08055_b200/libgsa_sm100.so /tmp/main.so
cp paper_2603_08055_b200/libgsa_v_fa16mix.so paper_2603_08055_b200/libgsa_sm100.so
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "tiled_attention or golden or hybrid or dense_degeneration" > gpurun_out/pytest_fa16mix.txt 2>&1
tail -3 gpurun_out/pytest_fa16mix.txt; grep -E "^E " gpurun_out/pytest_fa16mix.txt | head -10
cp /tmp/main.so paper_2603_08055_b200/libgsa_sm100.so
bash tools/gpu_variants2.sh 2 -- libgsa_sm100.so libgsa_v_fa16mix.so
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"select_tc" -c 1 -o gpurun_out/prof_sel300 \
  python bench.py --views 300 --steps 1 --warmup 0 --no-dense --no-cpu-baseline --no-e2e --no-parity > gpurun_out/ncu_sel300.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/ncu_sel300.log
