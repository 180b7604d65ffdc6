#!/bin/bash
# One gpurun pass: GPU parity tests, a short bench, the K1 ncu capture.
#   gpurun -- bash tools/gpu_check.sh [tag]
tag=${1:-run}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/${tag}_tests.log
tail -3 gpurun_out/${tag}_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench_rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_gm_eval -s 21 -c 1 \
  -o gpurun_out/${tag}_k1 -f python tools/profile_k1.py 22 > gpurun_out/${tag}_ncu.log 2>&1; echo "ncu_rc=$?"
