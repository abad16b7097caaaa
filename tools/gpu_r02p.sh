#!/bin/bash
# full GPU suite + the headline bench line (V=1000, all legs) + V=100
mkdir -p gpurun_out
T=${1:-r02p}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu_$T.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$T.txt
tail -3 gpurun_out/pytest_gpu_$T.txt; grep -E "^FAILED|^E  .*assert" gpurun_out/pytest_gpu_$T.txt | head -20
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_$T.txt 2>&1; tail -1 gpurun_out/smoke_$T.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_v1000_$T.json 2> gpurun_out/bench_v1000_$T.err
timeout 600 python bench.py --views 100 --steps 5 --warmup 3 > gpurun_out/bench_v100_$T.json 2> gpurun_out/bench_v100_$T.err
python - <<PY
import json
for v in ("v1000", "v100"):
    try:
        d = json.loads(open("gpurun_out/bench_%s_$T.json" % v).read().strip().splitlines()[-1])
        print(v, round(d["ms_per_step"], 2), d["stage_ms"], "e2e", d.get("e2e", {}).get("ms_per_step"), "parity", d.get("parity", {}).get("topk_mismatches"), d.get("parity", {}).get("rel_l2"), "dense x", d.get("dense", {}).get("speedup_sparse_vs_dense"), d["roofline"]["frac"], d["clocks"])
    except Exception as e:
        print(v, "failed", e)
PY
