"""Does the degree-9 rule reach the north-star tolerance (f2 d=8 rtol 1e-6)
where the degree-7 rule cannot?  Runs integrate() to its own
termination with max_regions sized to HBM and prints the per-iteration trace
plus the result (true error from the closed form).
  python tools/probe_gm9_ttt.py [rule] [d] [tau] [init] [integrand]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01573_b200 as hb

rule = sys.argv[1] if len(sys.argv) > 1 else "gm9"
d = int(sys.argv[2]) if len(sys.argv) > 2 else 8
tau = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-6
init = int(sys.argv[4]) if len(sys.argv) > 4 else 0
fid = sys.argv[5] if len(sys.argv) > 5 else "f2"
f = hb.make_integrand(fid, d)
exact = hb.reference_integral(fid, d)[0]
tr = []
st = {}
t0 = time.perf_counter()
r = hb.integrate(f, hb.HyperRect.unit_cube(d), hb.DriverConfig(tau, max_regions=1 << 40, rule=rule), trace=tr.append,
                 initial_regions=init or None, stats=st)
wall = time.perf_counter() - t0
for t in tr:
    print(json.dumps({"it": t.iteration, "n": t.active_regions, "I": t.integral, "eps_over_I": t.error / abs(t.integral),
                      "true_rel": abs(t.integral - exact) / exact}))
print(json.dumps({"rule": rule, "integrand": fid, "d": d, "tau": tau, "init": init, "reason": r.termination_reason.value,
                  "iterations": r.iterations, "integral": r.integral, "error": r.error, "exact": exact,
                  "true_rel_error": abs(r.integral - exact) / exact, "evals": r.total_f_evals,
                  "peak_regions": r.peak_regions, "wall_s": wall, "device_ms": st.get("device_ms"),
                  "capacity_limited": st.get("capacity_limited")}))
