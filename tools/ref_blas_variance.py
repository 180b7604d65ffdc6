"""How far the REFERENCE moves from its own goldens when numpy's OpenBLAS
picks another CPU kernel (DYNAMIC_ARCH: OPENBLAS_CORETYPE), on the same
inputs.  The goldens were made with the Haswell kernel (tests/golden/meta.json);
the GPU box's host may select another one.  This self-variance is the floor
of any meaningful parity tolerance on BLAS-summed quantities (the rule sums
vals @ w, and the error cascade |main - emb| that amplifies their rounding,
ref rules.py:515-516, 443-451).  Build container only (imports the reference).

  python tools/ref_blas_variance.py [coretype] [out.json]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(%(root)r, "tests"))
sys.path.insert(0, os.path.join(%(root)r, "tests", "golden"))
import hcub
from conftest import golden_names, load_json, load_k1
from make_golden import make_f, domain
out = {"k1": {}, "trace": {}}
for name in golden_names("k1"):
    z = load_k1(name)
    spec = z["spec"]
    I, E, S, ev = hcub.apply_rule_batch(hcub.get_rule("gm", spec["d"]), z["lo"], z["hi"], make_f(spec))
    gi, ge = z["integral"], z["error"]
    big = ge > 1e-9 * ge.max()
    out["k1"][name] = {
        "integral_max_rel": float(np.max(np.abs(I - gi) / np.maximum(np.abs(gi), 1e-300))),
        "error_max_rel_big": float(np.max(np.abs(E - ge)[big] / ge[big])),
        "error_max_abs_over_integral": float(np.max(np.abs(E - ge) / np.maximum(np.abs(gi), 1e-300))),
        "axis_agree": float(np.mean(np.argmax(S, 1) == z["axis"])), "scores_equal": bool(np.array_equal(S, z["scores"]))}
for name in golden_names("trace"):
    g = load_json("trace", name)
    spec = g["spec"]
    if name.startswith(("gk", "long")) or spec.get("rule", "gm") != "gm":
        continue
    cfg = hcub.DriverConfig(spec["tau"], max_iterations=spec["max_iterations"], max_regions=spec.get("max_regions", 1 << 24))
    tr = []
    r = hcub.integrate(make_f(spec), domain(spec), cfg, trace=tr.append, initial_regions=spec.get("init"))
    k = min(len(tr), len(g["trace"]))
    out["trace"][name] = {
        "counts_equal": [t.active_regions for t in tr] == [t[1] for t in g["trace"]],
        "max_rel_I": max(abs(tr[i].integral - g["trace"][i][2]) / abs(g["trace"][i][2]) for i in range(k)),
        "max_rel_eps": max(abs(tr[i].error - g["trace"][i][3]) / abs(g["trace"][i][3]) for i in range(k))}
print(json.dumps(out))
''' % {"root": ROOT}

core = sys.argv[1] if len(sys.argv) > 1 else "Sandybridge"
env = dict(os.environ, OPENBLAS_CORETYPE=core, OPENBLAS_NUM_THREADS="1", PYTHONDONTWRITEBYTECODE="1")
p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
if p.returncode:
    sys.exit(p.stderr[-3000:])
doc = {"note": f"reference (hcub, unmodified) re-run with OPENBLAS_CORETYPE={core} vs its own goldens "
               f"(Haswell kernel); tools/ref_blas_variance.py", "coretype": core, **json.loads(p.stdout)}
if len(sys.argv) > 2:
    with open(sys.argv[2], "w") as fh:
        json.dump(doc, fh, indent=1)
for sec in ("k1", "trace"):
    for k, v in doc[sec].items():
        print(sec, k, v)
