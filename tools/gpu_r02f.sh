#!/bin/bash
mkdir -p gpurun_out
T=r02f
make -s -j8 -C paper_2603_08055_b200/csrc EXTRA="-DGSA_WATCHDOG" BUILD=/tmp/bw > /dev/null 2>&1
timeout 900 python -m pytest -q -p no:cacheprovider tests -m gpu --timeout 300 -k "not test_sampled_rows_at_scale" > gpurun_out/pytest_$T.txt 2>&1
grep -E "^FAILED|passed|failed" gpurun_out/pytest_$T.txt | head -40
grep -E "^E  .*assert|^E +where|^E +AssertionError" gpurun_out/pytest_$T.txt | head -40
timeout 300 python bench.py --steps 3 --warmup 2 --no-dense --no-cpu-baseline --no-e2e > gpurun_out/bench_$T.txt 2>&1
tail -1 gpurun_out/bench_$T.txt | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('iid', round(l['ms_per_step'],2), l['stage_ms'], l['parity'])"
