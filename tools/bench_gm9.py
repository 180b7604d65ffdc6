"""Throughput of the explicit-table K1 (k1_table_eval) on the degree-9 table
(rule9.py) vs the generator K1 on the degree-7 GM rule, same integrand and
loop: python tools/bench_gm9.py [d] [iterations] [init]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01573_b200 as hb

d = int(sys.argv[1]) if len(sys.argv) > 1 else 8
its = int(sys.argv[2]) if len(sys.argv) > 2 else 16
init = int(sys.argv[3]) if len(sys.argv) > 3 else 64
f = hb.make_integrand("f2", d)
out = {}
for rule in ("gm", "gm9"):
    cfg = hb.DriverConfig(1e-6, max_iterations=its, max_regions=1 << 40, rule=rule)
    best = None
    for rep in range(3):
        st = {}
        r = hb.integrate(f, hb.HyperRect.unit_cube(d), cfg, initial_regions=init or None, stats=st)
        if rep and (best is None or st["k1_ms"] < best[0]["k1_ms"]):
            best = (st, r)
    st, r = best
    out[rule] = {"nodes": hb.get_rule(rule, d).node_count, "iterations": r.iterations, "evals": r.total_f_evals,
                 "k1_ms": st["k1_ms"], "k1_evals_per_s": r.total_f_evals / st["k1_ms"] * 1e3,
                 "fp64_tflops_alg": r.total_f_evals / st["k1_ms"] * 1e3 * (6 * d + 5) / 1e12,
                 "integral": r.integral, "error": r.error}
print(json.dumps({"d": d, "integrand": "f2", "init": init, **out}))
