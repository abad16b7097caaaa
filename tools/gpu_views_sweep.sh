#!/bin/bash
# layer time and sparse-vs-dense speedup as the sequence grows (the paper's scaling claim)
mkdir -p gpurun_out
OUT=gpurun_out/views_sweep.jsonl; : > $OUT
for V in 50 100 200 400 600 800 1000; do
  timeout 600 python bench.py --views $V --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-parity 2>/dev/null | tail -1 >> $OUT
done
python - <<PY
import json
for l in open("$OUT"):
    d = json.loads(l)
    print(d["config"]["views"], d["config"]["tokens"], round(d["ms_per_step"], 2), "dense", round(d["dense"]["ms"], 1), "x", round(d["dense"]["speedup_sparse_vs_dense"], 1))
PY
