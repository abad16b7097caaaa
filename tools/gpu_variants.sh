#!/bin/bash
# time alternative builds of the library: tools/gpu_variants.sh libA.so libB.so ...  (V=1000 stage times)
cp paper_2603_08055_b200/libgsa_sm100.so /tmp/libgsa_sm100_main.so
for v in "$@"; do
  cp paper_2603_08055_b200/$v paper_2603_08055_b200/libgsa_sm100.so
  echo "== $v"; timeout 300 python bench.py --views 1000 --steps 2 --warmup 1 --no-cpu-baseline --no-dense --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stage_ms'])"
done
cp /tmp/libgsa_sm100_main.so paper_2603_08055_b200/libgsa_sm100.so
