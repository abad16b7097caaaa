#!/bin/bash
mkdir -p gpurun_out
T=r02h
make -s -j8 -C paper_2603_08055_b200/csrc EXTRA="-DGSA_WATCHDOG" BUILD=/tmp/bw > /dev/null 2>&1
export GSA_PARITY_LOG=gpurun_out/scale_parity_$T.jsonl
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "huge or beyond" -m gpu > gpurun_out/pytest_$T.txt 2>&1
tail -4 gpurun_out/pytest_$T.txt
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_scale_parity.py -k "k4050 or k10125 or k2025" -m gpu --durations=5 >> gpurun_out/pytest_$T.txt 2>&1
tail -12 gpurun_out/pytest_$T.txt
cat $GSA_PARITY_LOG
for k in 810 2025 4050 10125; do
timeout 600 python bench.py --views 500 --topk $k --steps 2 --warmup 1 --no-dense --no-cpu-baseline --no-e2e --no-parity 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('k=$k', round(l['ms_per_step'],2), l['stage_ms'])"
done
