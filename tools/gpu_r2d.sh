#!/bin/bash
# one-sync protocol: distributed parity on device workers, protocol probes
mkdir -p gpurun_out
T=${TAG:-r2d}
timeout 1200 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_refbridge.py -q -x -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo tests_rc=$?; tail -15 gpurun_out/${T}_tests.log
timeout 900 python tools/probe_protocol.py 22 > gpurun_out/${T}_protocol.jsonl 2> gpurun_out/${T}_protocol.err; echo proto_rc=$?; cat gpurun_out/${T}_protocol.jsonl; tail -3 gpurun_out/${T}_protocol.err
timeout 600 python tools/probe_dist_phases.py 16 > gpurun_out/${T}_phases.txt 2>&1; echo phases_rc=$?; head -40 gpurun_out/${T}_phases.txt
