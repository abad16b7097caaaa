#!/bin/bash
mkdir -p gpurun_out
T=r02e
timeout 300 python tools/diag_cfg.py 2 > gpurun_out/diag_cfg_$T.txt 2>&1; tail -2 gpurun_out/diag_cfg_$T.txt
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_dist.py tests/test_spec_properties.py tests/test_gpu_parity.py -m gpu > gpurun_out/pytest_$T.txt 2>&1
tail -6 gpurun_out/pytest_$T.txt
timeout 300 python bench.py --steps 3 --warmup 2 --shard --no-dense --no-cpu-baseline --no-e2e --no-parity > gpurun_out/bench_shard_$T.txt 2> gpurun_out/bench_shard_$T.err
tail -1 gpurun_out/bench_shard_$T.txt | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('shard1', round(l['ms_per_step'],2), l['stage_ms'])"
grep -m3 "NCCL INFO" gpurun_out/bench_shard_$T.err
