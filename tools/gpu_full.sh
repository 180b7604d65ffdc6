#!/bin/bash
# Round-end style pass: GPU tests, default bench (with CPU baseline), reference
# arm, torchrun N=2 smoke on one GPU (gloo fallback), launch list, K1 ncu.
#   gpurun -- bash tools/gpu_full.sh <tag>
tag=${1:-full}
mkdir -p gpurun_out
timeout 900 python -X faulthandler -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo "tests_rc=$?" | tee -a gpurun_out/${tag}_tests.log
tail -2 gpurun_out/${tag}_tests.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench_rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err; echo "ref_rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 2 --warmup 1 --iterations 18 > gpurun_out/${tag}_tr2.json 2> gpurun_out/${tag}_tr2.err; echo "tr2_rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_f2d8_26its.csv \
  python tools/profile_k1.py 26 > /dev/null 2>&1; echo "launches_rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_gm_eval -s 21 -c 1 \
  -o gpurun_out/${tag}_k1 -f python tools/profile_k1.py 22 > gpurun_out/${tag}_ncu.log 2>&1; echo "ncu_rc=$?"
# reports are summarised on the box (gpurun brings back <= 64 MiB)
python tools/ncu_summary.py gpurun_out/${tag}_k1.ncu-rep 27942912 401 gpurun_out/${tag}_k1_ncu_summary.json "f2 d=8 north-star workload, 22nd K1 launch (27.9 M regions)" > /dev/null 2>&1
python tools/ncu_sass_stalls.py gpurun_out/${tag}_k1.ncu-rep > gpurun_out/${tag}_k1_stalls.txt 2>&1
rm -f gpurun_out/${tag}_k1.ncu-rep
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke_rc=$?"
# K1 at d=5 (configs[1] to tolerance): one full capture of the 33rd launch
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_gm_eval -s 32 -c 1 \
  -o gpurun_out/${tag}_k1d5 -f python tools/profile_ttt.py f2 5 1e-6 > gpurun_out/${tag}_ncu5.log 2>&1; echo "ncu5_rc=$?"
python tools/ncu_summary.py gpurun_out/${tag}_k1d5.ncu-rep 62690816 93 gpurun_out/${tag}_k1d5_ncu_summary.json "configs[1] f2 d=5 to tolerance, 33rd K1 launch (62.7M regions; grid x block upper bound)" > /dev/null 2>&1
rm -f gpurun_out/${tag}_k1d5.ncu-rep
# degree-9 generator kernel: one full capture of a late launch (f2 d=8, 19 iterations, 64 subdomains)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_gm9_eval -s 9 -c 1 \
  -o gpurun_out/${tag}_k9 -f python -c "
import sys; sys.path.insert(0, '.')
import paper_2511_01573_b200 as hb
hb.integrate(hb.make_integrand('f2', 8), hb.HyperRect.unit_cube(8), hb.DriverConfig(1e-6, max_iterations=19, max_regions=1 << 40, rule='gm9'), initial_regions=64)
" > gpurun_out/${tag}_ncu9.log 2>&1; echo "ncu9_rc=$?"
python tools/ncu_sass_stalls.py gpurun_out/${tag}_k9.ncu-rep > gpurun_out/${tag}_k9_stalls.txt 2>&1
ncu -i gpurun_out/${tag}_k9.ncu-rep --page raw --csv > gpurun_out/${tag}_k9_raw.csv 2>/dev/null
rm -f gpurun_out/${tag}_k9.ncu-rep
