#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-x}
timeout 600 python -m pytest tests/test_dist.py tests/test_gpu_parity.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu_$TAG.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.txt
timeout 600 python bench.py --shard --steps 3 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/bench_shard_$TAG.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-dense --views 100 > gpurun_out/bench_torchrun_$TAG.txt 2>&1
tail -5 gpurun_out/pytest_gpu_$TAG.txt; tail -c 1500 gpurun_out/bench_shard_$TAG.txt; tail -c 600 gpurun_out/bench_torchrun_$TAG.txt
