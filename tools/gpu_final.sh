#!/bin/bash
# final pass: regression (tests, smoke, forward + backward bench), backward CLI rows + gradient suite, sanitizers
bash tools/gpu_round2.sh r02z2
timeout 600 python -m paper_2603_08055_b200.cli --mode gsa --backward --frames 8,16,32,64,128 --repeats 3 \
  --specials-per-frame 5 --csv gpurun_out/bwd_cli.csv 2> gpurun_out/bwd_cli.err; cat gpurun_out/bwd_cli.csv; tail -1 gpurun_out/bwd_cli.err
timeout 600 python -m paper_2603_08055_b200.cli --verify gradient 2>&1 | tee gpurun_out/bwd_verify.txt
timeout 900 python bench.py --backward --hybrid 100 --steps 2 --warmup 1 2>/dev/null > gpurun_out/bench_bwd_hybrid_v1000.json
bash tools/gpu_sanitize_bwd.sh
