"""Compare K1 build variants on the fixed-work f2 d=8 workload:
  python tools/k1_variants.py lib1.so lib2.so ...   (one subprocess per library)"""
import json
import os
import subprocess
import sys

CHILD = r'''
import json, sys
sys.path.insert(0, "%s")
import paper_2511_01573_b200 as hb
its = int(sys.argv[1]); fid = sys.argv[2]; d = int(sys.argv[3]); init = int(sys.argv[4]) or None
f = hb.make_integrand(fid, d)
cfg = hb.DriverConfig(float(sys.argv[6]), max_iterations=its, max_regions=1 << 40, rule=sys.argv[5])
best = None
for rep in range(3):
    st = {}
    r = hb.integrate(f, hb.HyperRect.unit_cube(d), cfg, initial_regions=init, stats=st)
    if rep and (best is None or st["k1_ms"] < best[0]["k1_ms"]):
        best = (st, r)
st, r = best
print(json.dumps({"k1_ms": st["k1_ms"], "k3_ms": st["k3_ms"], "device_ms": st["device_ms"], "evals": r.total_f_evals,
                  "k1_evals_per_s": r.total_f_evals / st["k1_ms"] * 1e3, "integral": r.integral, "error": r.error}))
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

its = os.environ.get("ITS", "24")
fid = os.environ.get("FN", "f2")
d = os.environ.get("D", "8")
init = os.environ.get("INIT", "64")
rule = os.environ.get("RULE", "gm")
tau = os.environ.get("TAU", "1e-6")
for lib in sys.argv[1:]:
    env = dict(os.environ, HCUB_B200_LIB=os.path.abspath(lib))
    p = subprocess.run([sys.executable, "-c", CHILD, its, fid, d, init, rule, tau], env=env, capture_output=True,
                       text=True)
    line = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else p.stderr[-500:]
    print(os.path.basename(lib), line, flush=True)
