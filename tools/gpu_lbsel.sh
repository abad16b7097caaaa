#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x -k "compress or topk or clustered or oversmoothed or ties or scale_parity or spec or forward" > gpurun_out/pytest_lbsel.txt 2>&1
tail -2 gpurun_out/pytest_lbsel.txt; grep -E "^FAILED|^E  " gpurun_out/pytest_lbsel.txt | head -5
cp paper_2603_08055_b200/libgsa_sm100.so /tmp/libgsa_main.so
for v in main libgsa_nolb.so; do
  if [ "$v" = "main" ]; then cp /tmp/libgsa_main.so paper_2603_08055_b200/libgsa_sm100.so; else cp paper_2603_08055_b200/$v paper_2603_08055_b200/libgsa_sm100.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control base -k regex:"rescore|largek" --csv --log-file gpurun_out/launches_lb_$v.csv python bench.py --steps 1 --warmup 1 --no-dense --no-cpu-baseline --no-e2e --no-parity > /dev/null 2>&1
  echo "$v"; grep -o '_kernel<[0-9a-z, ]*>.*"ns","[0-9]*"' gpurun_out/launches_lb_$v.csv | sed 's/(const.*"ns",/ /'
done
cp /tmp/libgsa_main.so paper_2603_08055_b200/libgsa_sm100.so
bash tools/gpu_variants2.sh 2 -- main libgsa_nolb.so
bash tools/gpu_variants2.sh 1 --data clustered -- main libgsa_nolb.so
