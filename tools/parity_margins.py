"""Measured parity margins of the device path against the reference goldens
(sets the tolerances written in tests/): per-region K1 integral / error
relative deviations, per-iteration I / eps relative deviations of integrate.
  python tools/parity_margins.py [out.json]"""
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2511_01573_b200 as hb  # noqa: E402
from conftest import golden_names, load_json, load_k1  # noqa: E402


def fn_of(spec):
    if spec["f"] == "pp":
        return hb.make_product_peak(spec["d"], spec.get("center", 0.5), spec.get("sharpness", 50.0))[0]
    return hb.make_integrand(spec["f"], spec["d"])


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    den = np.maximum(np.abs(b), 1e-300)
    return float(np.max(np.abs(a - b) / den)) if a.size else 0.0


out = {"k1": {}, "trace": {}}
for name in golden_names("k1"):
    z = load_k1(name)
    spec = z["spec"]
    d = spec["d"]
    row = {}
    for lanes in (-1, 0):
        hb.set_k1_lanes(lanes)
        try:
            I, E, S, _ = hb.apply_rule_batch(hb.build_gm_rule(d), z["lo"], z["hi"], fn_of(spec))
        finally:
            hb.set_k1_lanes(-1)
        big = z["error"] > 1e-9 * np.max(z["error"])
        row[f"lanes{lanes}"] = dict(integral=rel(I, z["integral"]), error=rel(E, z["error"]),
                                    error_big=rel(E[big], z["error"][big]),
                                    error_abs_over_integral=float(np.max(np.abs(E - z["error"]) /
                                                                         np.maximum(np.abs(z["integral"]), 1e-300))),
                                    axis_agree=float(np.mean(np.argmax(S, 1) == z["axis"])),
                                    scores_equal=bool(np.array_equal(S, z["scores"])))
    out["k1"][name] = row
    print(name, row, flush=True)
for name in golden_names("trace"):
    g = load_json("trace", name)
    spec = g["spec"]
    if spec.get("rule", "gm") != "gm" or name.startswith("gk"):
        continue
    dom = hb.HyperRect(spec["lo"], spec["hi"]) if "lo" in spec else hb.HyperRect.unit_cube(spec["d"])
    cfg = hb.DriverConfig(spec["tau"], max_iterations=spec["max_iterations"],
                          max_regions=spec.get("max_regions", 1 << 24))
    tr = []
    r = hb.integrate(fn_of(spec), dom, cfg, trace=tr.append, initial_regions=spec.get("init"))
    same = [t.active_regions for t in tr] == [t[1] for t in g["trace"]]
    k = min(len(tr), len(g["trace"]))
    dI = max((abs(tr[i].integral - g["trace"][i][2]) / abs(g["trace"][i][2]) for i in range(k)), default=0)
    dE = max((abs(tr[i].error - g["trace"][i][3]) / abs(g["trace"][i][3]) for i in range(k)), default=0)
    out["trace"][name] = dict(counts_equal=same, iterations=len(tr), ref_iterations=len(g["trace"]),
                              max_rel_I=dI, max_rel_eps=dE, reason=r.termination_reason.value,
                              ref_reason=g["result"]["termination_reason"])
    print(name, out["trace"][name], flush=True)
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as fh:
        json.dump(out, fh, indent=1)
