#!/bin/bash
# round-end regression: GPU tests, smoke, forward bench lines, backward bench line
mkdir -p gpurun_out
TAG=${1:-x}
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu_$TAG.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_$TAG.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_v1000_$TAG.txt 2>&1
timeout 600 python bench.py --backward --steps 3 --warmup 1 > gpurun_out/bench_bwd_v1000_$TAG.txt 2>/dev/null
tail -3 gpurun_out/pytest_gpu_$TAG.txt; tail -1 gpurun_out/smoke_$TAG.txt
python - <<PY
import json
for f in ("gpurun_out/bench_v1000_$TAG.txt", "gpurun_out/bench_bwd_v1000_$TAG.txt"):
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
        print(f, d["value"], d["ms_per_step"], d.get("stage_ms"), d["clocks"]["reasons"])
    except Exception as e:
        print(f, "ERR", e)
PY
