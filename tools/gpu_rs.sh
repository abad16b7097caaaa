#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x -k "compress or topk or clustered or oversmoothed or ties or scale_parity or spec" > gpurun_out/pytest_rs.txt 2>&1
tail -2 gpurun_out/pytest_rs.txt; grep -E "^FAILED|^E  " gpurun_out/pytest_rs.txt | head -5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rs.csv python bench.py --steps 1 --warmup 1 --no-dense --no-cpu-baseline --no-e2e --no-parity > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/launches_rs.csv | grep -i "rescore\|largek\|compress_tc"
bash tools/gpu_variants2.sh 2 -- main libgsa_head3.so
