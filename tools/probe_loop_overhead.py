"""Where the time-to-tolerance goes outside the kernels: integrate() on the
BASELINE configs (best of 5 after a warm run), device time vs the summed
K1 / K2 / K3 kernel times; the rest is the per-iteration host round trip
(status read, decision, next launches).
  python tools/probe_loop_overhead.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01573_b200 as hb

CASES = [("configs[0]", "f4", 3, 1e-6, 0, "gm"), ("configs[1]", "f2", 5, 1e-6, 0, "gm"),
         ("configs[1]", "f2", 5, 1e-6, 0, "gm9"), ("configs[3]", "f3", 10, 1e-5, 80, "gm9")]
for name, fid, d, tau, init, rule in CASES:
    f = hb.make_integrand(fid, d)
    cfg = hb.DriverConfig(tau, max_regions=1 << 40, rule=rule)
    best = None
    for rep in range(6):
        st = {}
        r = hb.integrate(f, hb.HyperRect.unit_cube(d), cfg, initial_regions=init or None, stats=st)
        if rep and (best is None or st["device_ms"] < best[0]["device_ms"]):
            best = (st, r)
    st, r = best
    kern = st["k1_ms"] + st.get("k2_ms", 0.0) + st["k3_ms"]
    print(json.dumps({"config": name, "rule": rule, "iterations": r.iterations, "device_ms": st["device_ms"],
                      "k1_ms": st["k1_ms"], "k2_ms": st.get("k2_ms"), "k3_ms": st["k3_ms"],
                      "outside_kernels_ms": st["device_ms"] - kern,
                      "outside_per_iteration_us": (st["device_ms"] - kern) / r.iterations * 1e3}), flush=True)
