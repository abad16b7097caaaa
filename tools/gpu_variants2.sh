#!/bin/bash
# A/B of alternative library builds, interleaved over repeats (box-to-box and run-to-run clock
# noise hits every variant alike): tools/gpu_variants2.sh <reps> <bench args> -- main libA.so libB.so ... (main = the tree's libgsa_sm100.so)
REPS=$1; shift; ARGS=""
while [ "$1" != "--" ]; do ARGS="$ARGS $1"; shift; done; shift
cp paper_2603_08055_b200/libgsa_sm100.so /tmp/libgsa_main.so
for r in $(seq $REPS); do for v in "$@"; do
  if [ "$v" = "main" ]; then cp /tmp/libgsa_main.so paper_2603_08055_b200/libgsa_sm100.so
  else cp paper_2603_08055_b200/$v paper_2603_08055_b200/libgsa_sm100.so; fi
  timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-dense --no-e2e --no-parity $ARGS 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],2), d['stage_ms'], d['clocks']['sm_mhz'])" || echo "$v failed"
done; done
cp /tmp/libgsa_main.so paper_2603_08055_b200/libgsa_sm100.so
