#!/bin/bash
# backward bench line (1000 views), CLI --backward rows and the gradient verification suite
mkdir -p gpurun_out
timeout 900 python bench.py --backward --steps 3 --warmup 1 2> gpurun_out/bwd_bench.err | tee gpurun_out/bwd_bench.json
timeout 600 python -m paper_2603_08055_b200.cli --mode gsa --backward --frames 8,16,32,64,128 --repeats 3 \
  --specials-per-frame 5 --csv gpurun_out/bwd_cli.csv 2> gpurun_out/bwd_cli.err; cat gpurun_out/bwd_cli.csv gpurun_out/bwd_cli.err
timeout 600 python -m paper_2603_08055_b200.cli --verify gradient 2>&1 | tee gpurun_out/bwd_verify.txt
