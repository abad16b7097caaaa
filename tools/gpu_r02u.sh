#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02u}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"select_tc" -c 1 -o gpurun_out/prof_sel_$T \
  python bench.py --views 1000 --steps 1 --warmup 0 --no-dense --no-cpu-baseline --no-e2e --no-parity > gpurun_out/ncu_sel_$T.log 2>&1
echo "ncu exit $?"; grep -E "==PROF==|==ERROR==" gpurun_out/ncu_sel_$T.log | tail -3
bash tools/gpu_variants2.sh 2 -- main libgsa_g32ns3.so libgsa_selns3.so libgsa_fapoly2.so
