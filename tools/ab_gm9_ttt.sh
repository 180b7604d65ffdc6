#!/bin/bash
# degree-9 time to tolerance (configs[1], configs[3]) and fixed-work d=8 per library in $LIBS
for L in $LIBS; do
  echo "== $L"
  for c in "5 1e-6 0 f2" "10 1e-5 80 f3"; do
    HCUB_B200_LIB=$(realpath $L) timeout 300 python -c "
import sys, json, statistics; sys.path.insert(0, '.')
import paper_2511_01573_b200 as hb
d, tau, init, fid = '$c'.split(); d = int(d); tau = float(tau); init = int(init) or None
f = hb.make_integrand(fid, d); cfg = hb.DriverConfig(tau, max_regions=1 << 40, rule='gm9')
ts = []
for i in range(4):
    st = {}; r = hb.integrate(f, hb.HyperRect.unit_cube(d), cfg, initial_regions=init, stats=st)
    if i: ts.append(st['device_ms'])
print(json.dumps({'cfg': '$c', 'median_device_ms': statistics.median(ts), 'its': r.iterations, 'reason': r.termination_reason.value, 'evals': r.total_f_evals}))
"
  done
  HCUB_B200_LIB=$(realpath $L) timeout 600 python tools/bench_gm9.py 8 19 64 2>&1 | tail -1
done
