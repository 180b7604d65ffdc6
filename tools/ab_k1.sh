#!/bin/bash
# K1 A/B on the GPU box: parity subset on the default library, then
# tools/k1_variants.py over $LIBS on configs[1] (f2 d=5 to tolerance) and the north-star prefix (f2 d=8 init 64).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_k1.py tests/test_gpu_integrate.py tests/test_gpu_region_sets.py tests/test_gpu_distributed.py -q -x -p no:cacheprovider > gpurun_out/ab1_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/ab1_tests.log
L="${LIBS:-paper_2511_01573_b200/libhcub_nopipe.so paper_2511_01573_b200/libhcub_b200.so}"
D=5 INIT=0 ITS=40 timeout 600 python tools/k1_variants.py $L 2>&1 | tee gpurun_out/ab1_d5.txt
D=8 INIT=64 ITS=24 timeout 600 python tools/k1_variants.py $L 2>&1 | tee gpurun_out/ab1_d8.txt
