#!/bin/bash
# backward bring-up: the backward tests on the B200 (bounded)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_backward.py -x -q -m gpu 2>&1 | tail -40 > gpurun_out/pytest_bwd.txt
cat gpurun_out/pytest_bwd.txt | tail -40
