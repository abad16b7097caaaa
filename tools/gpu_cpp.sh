#!/bin/bash
# C++ drop-in host->host at V=1000 (f32 / bf16) with its time breakdown, + the C++ API tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cpp_api.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_cpp.txt 2>&1; tail -2 gpurun_out/pytest_cpp.txt
make -s -C tests/cpp
for P in f32 bf16; do timeout 900 tests/cpp/gsa_cpp_driver --time 1000 2 $P; done
