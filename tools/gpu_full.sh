#!/bin/bash
# Round-end style pass: GPU tests, default bench (with CPU baseline), reference
# arm, torchrun N=2 smoke on one GPU (gloo fallback), launch list, K1 ncu.
#   gpurun -- bash tools/gpu_full.sh <tag>
tag=${1:-full}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests_rc=$?" | tee -a gpurun_out/${tag}_tests.log
tail -2 gpurun_out/${tag}_tests.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench_rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err; echo "ref_rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 2 --warmup 1 --iterations 18 > gpurun_out/${tag}_tr2.json 2> gpurun_out/${tag}_tr2.err; echo "tr2_rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_f2d8_26its.csv \
  python tools/profile_k1.py 26 > /dev/null 2>&1; echo "launches_rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_gm_eval -s 21 -c 1 \
  -o gpurun_out/${tag}_k1 -f python tools/profile_k1.py 22 > gpurun_out/${tag}_ncu.log 2>&1; echo "ncu_rc=$?"
