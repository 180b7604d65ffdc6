#!/bin/bash
# K3 classify A/B: parity subset on the default library, K3 time over $LIBS on
# configs[1] (f2 d=5 to tolerance), one ncu capture of the default K3.
mkdir -p gpurun_out
T=${TAG:-k3}
timeout 900 python -m pytest tests/test_gpu_integrate.py tests/test_gpu_region_sets.py tests/test_gpu_distributed.py tests/test_gpu_edges.py -q -x -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/${T}_tests.log
D=5 INIT=0 ITS=40 timeout 900 python tools/k1_variants.py $LIBS 2>&1 | tee gpurun_out/${T}_d5.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k3_classify -s 31 -c 1 \
  -o gpurun_out/${T}_k3d5 -f python tools/profile_ttt.py f2 5 1e-6 > gpurun_out/${T}_ncu.log 2>&1; echo ncu_rc=$?
