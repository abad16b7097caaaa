#!/bin/bash
# usage: tools/gpu_quick.sh <tag> [pytest -k expr] — gpu tests + quick V=100 / V=1000 bench lines (no baselines)
mkdir -p gpurun_out
TAG=${1:-x}; KX=${2:-""}
if [ -n "$KX" ]; then timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "$KX" > gpurun_out/pytest_gpu_$TAG.txt 2>&1
else timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu_$TAG.txt 2>&1; fi
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python bench.py --views 100 --steps 5 --warmup 3 --no-cpu-baseline --no-dense --no-e2e > gpurun_out/bench_v100_$TAG.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-dense --no-e2e > gpurun_out/bench_v1000_$TAG.txt 2>&1
tail -15 gpurun_out/pytest_gpu_$TAG.txt
python - <<PY
import json
for v in ("v100", "v1000"):
    try:
        d = json.loads(open("gpurun_out/bench_%s_$TAG.txt" % v).read().strip().splitlines()[-1])
        print(v, "ms", round(d["ms_per_step"], 2), "stages", d["stage_ms"], "launches", d["gpu_launches"])
    except Exception as e:
        print(v, "failed", e); print(open("gpurun_out/bench_%s_$TAG.txt" % v).read()[-2000:])
PY
