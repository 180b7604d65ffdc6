#!/bin/bash
# One GPU pass: parity tests, bench (N=1) + reference arm, launch list and
# ncu captures of K1 / K3 classify on BASELINE configs[1] (f2 d=5 to tolerance).
#   gpurun -- bash tools/gpu_pass.sh <tag> [tests] [bench] [ref] [ncu5] [launch8]
tag=${1:-r2}; shift
what=" $* "
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
if [[ $what == *" tests "* ]]; then
  timeout 1500 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1
  echo "tests_rc=$?" | tee -a gpurun_out/${tag}_tests.log; tail -3 gpurun_out/${tag}_tests.log
fi
if [[ $what == *" smoke "* ]]; then
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke_rc=$?"
fi
if [[ $what == *" bench "* ]]; then
  timeout 1200 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench_rc=$?"
  tail -c 600 gpurun_out/${tag}_bench.json
fi
if [[ $what == *" ref "* ]]; then
  timeout 900 python bench.py --impl reference > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err; echo "ref_rc=$?"
fi
if [[ $what == *" ncu5 "* ]]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_gm_eval -s 32 -c 1 \
    -o gpurun_out/${tag}_k1d5 -f python tools/profile_ttt.py f2 5 1e-6 > gpurun_out/${tag}_ncu_k1d5.log 2>&1; echo "ncu_k1d5_rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_classify -s 31 -c 1 \
    -o gpurun_out/${tag}_k3d5 -f python tools/profile_ttt.py f2 5 1e-6 > gpurun_out/${tag}_ncu_k3d5.log 2>&1; echo "ncu_k3d5_rc=$?"
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches_f2d5_ttt.csv python tools/profile_ttt.py f2 5 1e-6 > /dev/null 2>&1; echo "launches5_rc=$?"
fi
if [[ $what == *" launch8 "* ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_f2d8.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${tag}_bench_under_ncu.log 2>&1; echo "launch8_rc=$?"
fi
