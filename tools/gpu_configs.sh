#!/bin/bash
# BASELINE.json configs beyond the headline: pi3 geometry (configs[3]) and the
# top-k budget sweep at 500 views (configs[4]); one bench line each
mkdir -p gpurun_out
TAG=${1:-x}
OUT=gpurun_out/configs_$TAG.jsonl; : > $OUT
timeout 300 python bench.py --views 200 --grid 36x76 --specials-per-view 0 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> $OUT
for K in 8 16 32 64 128 810 2025; do
  timeout 600 python bench.py --views 500 --topk $K --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-dense 2>/dev/null | tail -1 >> $OUT
done
python - <<PY
import json
for l in open("$OUT"):
    try:
        d = json.loads(l)
        print(d["config"]["workload"][:90], "| ms", round(d["ms_per_step"], 2), "| stages", d["stage_ms"], "| dense x", round(d.get("dense", {}).get("speedup_sparse_vs_dense") or 0, 1))
    except Exception as e:
        print("bad line", l[:200])
PY
# clustered activations (the reference's kClustered recipe) at 1000 views
timeout 600 python bench.py --views 1000 --data clustered --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-dense 2>/dev/null | tail -1 >> $OUT
# hybrid (VGGT reference frames every 100 views) at 1000 views
timeout 600 python bench.py --views 1000 --hybrid 100 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-dense 2>/dev/null | tail -1 >> $OUT
tail -1 $OUT | cut -c1-600
