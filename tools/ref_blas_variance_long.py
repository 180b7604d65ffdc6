"""tools/ref_blas_variance.py for the long reference traces (tens of minutes
of CPU each): the reference's per-iteration (n, I, eps) under another
OpenBLAS kernel vs its own long golden.  Build container only.
  python tools/ref_blas_variance_long.py <trace name> [coretype] [out.json]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, sys
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(%(root)r, "tests", "golden"))
import hcub
from make_golden import make_f, domain
g = json.load(open(os.path.join(%(root)r, "tests", "golden", "trace_%(name)s.json")))
spec = g["spec"]
cfg = hcub.DriverConfig(spec["tau"], max_iterations=spec["max_iterations"], max_regions=spec["max_regions"])
tr = []
hcub.integrate(make_f(spec), domain(spec), cfg, trace=tr.append, initial_regions=spec.get("init"))
k = min(len(tr), len(g["trace"]))
print(json.dumps({"counts_equal": [t.active_regions for t in tr] == [t[1] for t in g["trace"]],
    "max_rel_I": max(abs(tr[i].integral - g["trace"][i][2]) / abs(g["trace"][i][2]) for i in range(k)),
    "max_rel_eps": max(abs(tr[i].error - g["trace"][i][3]) / abs(g["trace"][i][3]) for i in range(k)),
    "rel_eps_per_iteration": [abs(tr[i].error - g["trace"][i][3]) / abs(g["trace"][i][3]) for i in range(k)]}))
'''
name = sys.argv[1]
core = sys.argv[2] if len(sys.argv) > 2 else "Sandybridge"
env = dict(os.environ, OPENBLAS_CORETYPE=core, OPENBLAS_NUM_THREADS="1", PYTHONDONTWRITEBYTECODE="1")
p = subprocess.run([sys.executable, "-c", CHILD % {"root": ROOT, "name": name}], env=env, capture_output=True, text=True)
if p.returncode:
    sys.exit(p.stderr[-3000:])
doc = {"trace": name, "coretype": core, **json.loads(p.stdout)}
if len(sys.argv) > 3:
    with open(sys.argv[3], "w") as fh:
        json.dump(doc, fh, indent=1)
print(json.dumps({k: v for k, v in doc.items() if k != "rel_eps_per_iteration"}))
