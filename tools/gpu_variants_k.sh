#!/bin/bash
# A/B of alternative builds at V=500 and top-k K (default 128): tools/gpu_variants_k.sh K a.so b.so ...
K=$1; shift
cp paper_2603_08055_b200/libgsa_sm100.so /tmp/m.so
for v in "$@"; do cp paper_2603_08055_b200/$v paper_2603_08055_b200/libgsa_sm100.so; echo "== $v"; GSA_DEBUG_STATS=1 timeout 300 python bench.py --views 500 --topk $K --steps 2 --warmup 1 --no-cpu-baseline --no-dense --no-e2e 2>&1 | grep "compress stats" | tail -1; timeout 300 python bench.py --views 500 --topk $K --steps 2 --warmup 1 --no-cpu-baseline --no-dense --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stage_ms'])"; done
cp /tmp/m.so paper_2603_08055_b200/libgsa_sm100.so
