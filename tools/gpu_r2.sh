#!/bin/bash
# Round-2 GPU pass: parity tests, then ncu captures of K1 and K3 classify on
# BASELINE configs[1] (f2 d=5 time-to-tolerance, last iteration = largest launch).
#   gpurun -- bash tools/gpu_r2.sh <tag> [tests|ncu5|all]
tag=${1:-r2}
what=${2:-all}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
if [[ $what == tests || $what == all ]]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests_rc=$?" | tee -a gpurun_out/${tag}_tests.log
  tail -5 gpurun_out/${tag}_tests.log
fi
if [[ $what == ncu5 || $what == all ]]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_gm_eval -s 32 -c 1 \
    -o gpurun_out/${tag}_k1d5 -f python tools/profile_ttt.py f2 5 1e-6 > gpurun_out/${tag}_ncu_k1d5.log 2>&1; echo "ncu_k1d5_rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_classify -s 31 -c 1 \
    -o gpurun_out/${tag}_k3d5 -f python tools/profile_ttt.py f2 5 1e-6 > gpurun_out/${tag}_ncu_k3d5.log 2>&1; echo "ncu_k3d5_rc=$?"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_f2d5_ttt.csv \
    python tools/profile_ttt.py f2 5 1e-6 > /dev/null 2>&1; echo "launches_rc=$?"
fi
