#!/bin/bash
# degree-9 generator kernel variants: f2 d=8 (64 subdomains, 19 iterations) and d=5 throughput per library in $LIBS
mkdir -p gpurun_out
for L in $LIBS; do
  echo "== $L"
  HCUB_B200_LIB=$(realpath $L) timeout 600 python tools/bench_gm9.py 8 19 64 2>&1 | tail -1
  HCUB_B200_LIB=$(realpath $L) timeout 600 python tools/bench_gm9.py 5 24 0 2>&1 | tail -1
done
