#!/bin/bash
# usage: tools/gpu_ab.sh <tag> [pytest -k expr]: the GPU suite (or a subset, no -x), V=1000 iid + clustered
# stage times (3 steps), and the r02 baseline build's V=1000 stage times when /tmp/prev.so is shipped as
# paper_2603_08055_b200/libgsa_prev.so
mkdir -p gpurun_out
T=${1:-x}; KX=${2:-""}
if [ -n "$KX" ]; then timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "$KX" > gpurun_out/pytest_gpu_$T.txt 2>&1
else timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_$T.txt 2>&1; fi
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$T.txt
tail -2 gpurun_out/pytest_gpu_$T.txt; grep -E "^FAILED" gpurun_out/pytest_gpu_$T.txt | head
run() { timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-dense --no-e2e $2 > gpurun_out/bench_$1_$T.txt 2>&1;
  tail -1 gpurun_out/bench_$1_$T.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2), d['stage_ms'], d.get('parity',{}).get('topk_mismatches'), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/bench_$1_$T.txt; }
run iid ""
run clu "--data clustered"
if [ -f paper_2603_08055_b200/libgsa_prev.so ]; then
  cp paper_2603_08055_b200/libgsa_sm100.so /tmp/cur.so; cp paper_2603_08055_b200/libgsa_prev.so paper_2603_08055_b200/libgsa_sm100.so
  run prev_iid ""
  cp /tmp/cur.so paper_2603_08055_b200/libgsa_sm100.so
fi
