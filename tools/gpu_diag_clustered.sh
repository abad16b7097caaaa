#!/bin/bash
# candidate statistics of K2 on iid / clustered / hybrid V=1000 (stats build, synchronises; timing meaningless)
mkdir -p gpurun_out
make -s -j8 -C paper_2603_08055_b200/csrc EXTRA="-DGSA_DEBUG_STATS" BUILD=/tmp/bstats > /dev/null
for d in normal clustered; do
  echo "== $d" ; timeout 300 python bench.py --steps 1 --warmup 0 --data $d --no-dense --no-cpu-baseline --no-e2e --no-parity 2>&1 | grep -E "compress stats|flagged row" | head -6
done
echo "== hybrid"; timeout 300 python bench.py --steps 1 --warmup 0 --hybrid 100 --no-dense --no-cpu-baseline --no-e2e --no-parity 2>&1 | grep -E "compress stats" | head -3
