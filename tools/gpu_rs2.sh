#!/bin/bash
cp paper_2603_08055_b200/libgsa_sm100.so /tmp/libgsa_main.so
for v in main libgsa_head3.so main libgsa_head3.so; do
  if [ "$v" = "main" ]; then cp /tmp/libgsa_main.so paper_2603_08055_b200/libgsa_sm100.so; else cp paper_2603_08055_b200/$v paper_2603_08055_b200/libgsa_sm100.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control base -k regex:rescore --csv --log-file gpurun_out/launches_rs_$v.csv python bench.py --steps 1 --warmup 1 --no-dense --no-cpu-baseline --no-e2e --no-parity > /dev/null 2>&1
  echo "$v"; python tools/summarize_launches.py gpurun_out/launches_rs_$v.csv | grep -i "rescore"
done
cp /tmp/libgsa_main.so paper_2603_08055_b200/libgsa_sm100.so
