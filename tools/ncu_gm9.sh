#!/bin/bash
# one full ncu capture of the degree-9 generator kernel (last of 10 launches of a 19-iteration f2 d=8 run), summarised on the box
tag=${1:-gm9}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_gm9_eval -s 9 -c 1 \
  -o gpurun_out/${tag}_k9 -f python -c "
import sys; sys.path.insert(0, '.')
import paper_2511_01573_b200 as hb
hb.integrate(hb.make_integrand('f2', 8), hb.HyperRect.unit_cube(8), hb.DriverConfig(1e-6, max_iterations=19, max_regions=1 << 40, rule='gm9'), initial_regions=64)
" > gpurun_out/${tag}_ncu9.log 2>&1; echo "ncu9_rc=$?"
python tools/ncu_sass_stalls.py gpurun_out/${tag}_k9.ncu-rep > gpurun_out/${tag}_k9_stalls.txt 2>&1
ncu -i gpurun_out/${tag}_k9.ncu-rep --page raw --csv > gpurun_out/${tag}_k9_raw.csv 2>/dev/null
rm -f gpurun_out/${tag}_k9.ncu-rep
