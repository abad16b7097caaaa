#!/bin/bash
# round-2 evidence pass A: launch list + ncu --set full of every hot kernel at V=1000 (one GPU)
mkdir -p gpurun_out
T=${1:-r02t}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v1000_$T.csv \
  python bench.py --steps 2 --warmup 1 --no-dense --no-cpu-baseline --no-e2e --no-parity > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/launches_v1000_$T.csv | head -24
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"compress_tc|fa_tc|rescore|pool_kernel|select_tc|v16_kernel|vmax_kernel" -c 8 -o gpurun_out/prof_$T \
  python bench.py --views 1000 --steps 1 --warmup 0 --no-dense --no-cpu-baseline --no-e2e --no-parity > gpurun_out/ncu_$T.log 2>&1
echo "ncu exit $?"; grep -E "==PROF==|==ERROR==|==WARNING==" gpurun_out/ncu_$T.log | tail -5
