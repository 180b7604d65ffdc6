#!/bin/bash
# degree-9 table parity + throughput, distributed protocol cost probe
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tables.py tests/test_gpu_integrate.py -k "gm9 or table" -q -p no:cacheprovider > gpurun_out/r2b_tests.log 2>&1; echo tests_rc=$?; tail -15 gpurun_out/r2b_tests.log
timeout 600 python tools/bench_gm9.py 8 16 64 > gpurun_out/r2b_gm9_d8.json 2>&1; echo gm9_rc=$?; cat gpurun_out/r2b_gm9_d8.json | tail -c 900
timeout 600 python tools/bench_gm9.py 5 22 0 > gpurun_out/r2b_gm9_d5.json 2>&1; tail -c 900 gpurun_out/r2b_gm9_d5.json
timeout 900 python tools/probe_protocol.py 22 > gpurun_out/r2b_protocol.jsonl 2> gpurun_out/r2b_protocol.err; echo proto_rc=$?; cat gpurun_out/r2b_protocol.jsonl; tail -5 gpurun_out/r2b_protocol.err
