"""K1 lane shapes on configs[1] (f2 d=5 to tolerance): forced lanes per region (-1 = automatic)."""
import json, sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01573_b200 as hb
f = hb.make_integrand("f2", 5)
cfg = hb.DriverConfig(1e-6, max_regions=1 << 40)
for lg in (-1, 0, 1, 2):
    hb.set_k1_lanes(lg)
    best = None
    for rep in range(4):
        st = {}
        r = hb.integrate(f, hb.HyperRect.unit_cube(5), cfg, stats=st)
        if rep and (best is None or st["k1_ms"] < best["k1_ms"]): best = st
    print(json.dumps({"log2_lanes": lg, "k1_ms": best["k1_ms"], "device_ms": best["device_ms"], "I": r.integral}), flush=True)
