#!/bin/bash
# round-2 evidence pass B: BASELINE configs sweep, 24-layer stack, C++ drop-in host->host
mkdir -p gpurun_out
T=${1:-r02v}
bash tools/gpu_configs.sh $T
timeout 1200 python bench.py --layers 24 --steps 1 --warmup 1 --no-cpu-baseline --no-dense --no-e2e --no-parity > gpurun_out/stack24_$T.json 2> gpurun_out/stack24_$T.err
tail -1 gpurun_out/stack24_$T.json | cut -c1-900
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_stack_$T.csv python bench.py --layers 2 --steps 1 --warmup 0 --no-cpu-baseline --no-dense --no-e2e --no-parity > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/launches_stack_$T.csv | head -16
for P in bf16 f32; do
  timeout 1500 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-dense --no-e2e --no-parity --e2e-cpp $P > gpurun_out/e2ecpp_${P}_$T.json 2> gpurun_out/e2ecpp_${P}_$T.err
  tail -1 gpurun_out/e2ecpp_${P}_$T.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('e2e_cpp $P', d.get('e2e_cpp'))"
done
