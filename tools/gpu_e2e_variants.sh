#!/bin/bash
# e2e host pipeline granularity: heads per group x device slot sets (V=1000)
for cfg in "2 2" "2 3" "3 3" "4 3" "4 2"; do
  set -- $cfg
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-dense --no-parity --e2e-heads-per-group $1 --e2e-slots $2 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('g=$1 slots=$2 layer', round(d['ms_per_step'],1), 'e2e', round(d['e2e']['ms_per_step'],1))" || echo "g=$1 slots=$2 failed"
done
