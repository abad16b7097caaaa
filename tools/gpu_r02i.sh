#!/bin/bash
mkdir -p gpurun_out
T=r02i
make -s -j8 -C paper_2603_08055_b200/csrc EXTRA="-DGSA_WATCHDOG" BUILD=/tmp/bw > /dev/null 2>&1
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_stack.py -m gpu -x > gpurun_out/pytest_$T.txt 2>&1
tail -15 gpurun_out/pytest_$T.txt
make -s -j8 -C paper_2603_08055_b200/csrc > /dev/null 2>&1
timeout 900 python bench.py --layers 24 --steps 1 --warmup 1 > gpurun_out/stack24_$T.json 2>&1
tail -1 gpurun_out/stack24_$T.json | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('stack', round(l['ms_per_step'],1), round(l['ms_per_layer'],2), l['stage_ms_layer0'], l['projection_and_concat_ms_per_layer'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_stack_$T.csv python bench.py --layers 2 --steps 1 --warmup 0 > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/launches_stack_$T.csv | head -20
