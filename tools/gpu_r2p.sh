#!/bin/bash
# degree-9 generator kernel: parity (tables, traces, region sets) + throughput
mkdir -p gpurun_out
T=${TAG:-r2p}
timeout 900 python -m pytest tests/test_gpu_tables.py tests/test_gpu_integrate.py tests/test_gpu_region_sets.py -k "gm9 or table" -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo tests_rc=$?; tail -20 gpurun_out/${T}_tests.log
timeout 600 python tools/bench_gm9.py 8 16 64 > gpurun_out/${T}_gm9_d8.json 2>&1; tail -c 800 gpurun_out/${T}_gm9_d8.json
timeout 600 python tools/bench_gm9.py 8 19 64 > gpurun_out/${T}_gm9_d8_19.json 2>&1; tail -c 800 gpurun_out/${T}_gm9_d8_19.json
timeout 600 python tools/bench_gm9.py 5 22 0 > gpurun_out/${T}_gm9_d5.json 2>&1; tail -c 800 gpurun_out/${T}_gm9_d5.json
