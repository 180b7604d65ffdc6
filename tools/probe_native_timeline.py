"""Per-iteration wall time of the native integrate loop (trace callback
timestamps) for one config, warm run: where small-store iterations spend
their time (launch chain + status sync) vs the device work.
  python tools/probe_native_timeline.py [rule] [integrand] [d] [tau] [init]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01573_b200 as hb

rule = sys.argv[1] if len(sys.argv) > 1 else "gm9"
fid = sys.argv[2] if len(sys.argv) > 2 else "f2"
d = int(sys.argv[3]) if len(sys.argv) > 3 else 5
tau = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-6
init = int(sys.argv[5]) if len(sys.argv) > 5 else 0
f = hb.make_integrand(fid, d)
cfg = hb.DriverConfig(tau, max_regions=1 << 40, rule=rule)
for _ in range(2):
    hb.integrate(f, hb.HyperRect.unit_cube(d), cfg, initial_regions=init or None)
stamps = []
st = {}
t0 = time.perf_counter()
r = hb.integrate(f, hb.HyperRect.unit_cube(d), cfg, initial_regions=init or None,
                 trace=lambda t: stamps.append((time.perf_counter(), t.active_regions)), stats=st)
prev = t0
rows = []
for t, n in stamps:
    rows.append({"n": n, "us": round(1e6 * (t - prev))})
    prev = t
print(json.dumps({"rule": rule, "f": fid, "d": d, "iterations": r.iterations, "device_ms": st["device_ms"],
                  "k1_ms": st["k1_ms"], "k2_ms": st["k2_ms"], "k3_ms": st["k3_ms"], "launches": st["launches"],
                  "wall_ms": 1e3 * (stamps[-1][0] - t0), "per_iteration": rows}))
