#!/bin/bash
mkdir -p gpurun_out
T=r02d
timeout 300 python tools/diag_cfg.py 2 > gpurun_out/diag_cfg_$T.txt 2>&1
tail -3 gpurun_out/diag_cfg_$T.txt
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_spec_properties.py tests/test_cpp_api.py -m gpu > gpurun_out/pytest_$T.txt 2>&1
tail -8 gpurun_out/pytest_$T.txt
for d in normal clustered; do
  timeout 300 python bench.py --steps 3 --warmup 2 --data $d --no-dense --no-cpu-baseline --no-e2e --no-parity 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$d', round(l['ms_per_step'],2), l['stage_ms'])"
done
timeout 300 python bench.py --steps 3 --warmup 2 --hybrid 100 --no-dense --no-cpu-baseline --no-e2e --no-parity 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('hybrid', round(l['ms_per_step'],2), l['stage_ms'])"
bash tools/gpu_diag_clustered.sh
