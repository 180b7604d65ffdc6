"""First-GPU-call diagnostics: deviations of K1 vs golden, integrate traces."""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2511_01573_b200 as hb
from paper_2511_01573_b200.rules import apply_rule_batch_axes
from conftest import golden_names, load_k1, load_json
for name in golden_names("k1"):
    g = load_k1(name); spec = g["spec"]
    f = hb.make_product_peak(spec["d"], spec.get("center", .5), spec.get("sharpness", 50.))[0] if spec["f"] == "pp" else hb.make_integrand(spec["f"], spec["d"])
    t = time.time()
    I, E, S, ax, ev = apply_rule_batch_axes(hb.build_gm_rule(spec["d"]), g["lo"], g["hi"], f)
    rI = np.abs(I - g["integral"]) / np.maximum(np.abs(g["integral"]), 1e-300)
    rE = np.abs(E - g["error"]) / np.maximum(np.abs(g["error"]), 1e-300)
    print(json.dumps(dict(k1=name, n=len(I), maxrelI=float(rI.max()), p99I=float(np.quantile(rI, .99)), maxrelE=float(rE.max()),
        medE=float(np.median(rE)), scores_exact=float(np.mean(S == g["scores"])), axis_match=float(np.mean(ax == g["axis"])), t=time.time()-t)), flush=True)
for name in ["f4_d3", "f2_d5", "f2_d8", "f2_d8_init64", "pp_d4_c01", "f2_d3_odd", "f6_d6", "f3_d10", "f1_d4", "f2_d3_maxreg", "f4_d3_init64"]:
    g = load_json("trace", name); spec = g["spec"]
    f = hb.make_product_peak(spec["d"], spec.get("center", .5), spec.get("sharpness", 50.))[0] if spec["f"] == "pp" else hb.make_integrand(spec["f"], spec["d"])
    dom = hb.HyperRect(spec["lo"], spec["hi"]) if "lo" in spec else hb.HyperRect.unit_cube(spec["d"])
    tr = []; st = {}
    t = time.time()
    r = hb.integrate(f, dom, hb.DriverConfig(spec["tau"], max_iterations=spec["max_iterations"], max_regions=spec.get("max_regions", 1 << 24)), trace=tr.append, initial_regions=spec.get("init"), stats=st)
    cm = [a.active_regions == b[1] for a, b in zip(tr, g["trace"])]
    dI = max(abs(a.integral - b[2]) / abs(b[2]) for a, b in zip(tr, g["trace"]))
    dE = max(abs(a.error - b[3]) / abs(b[3]) for a, b in zip(tr, g["trace"]))
    print(json.dumps(dict(trace=name, reason=r.termination_reason.value, ref_reason=g["result"]["termination_reason"], it=r.iterations, ref_it=g["result"]["iterations"],
        counts_match=sum(cm), n=len(cm), maxrelI=dI, maxrelE=dE, evals=r.total_f_evals, ref_evals=g["result"]["total_f_evals"], wall=time.time()-t, stats=st)), flush=True)
# throughput probe: f2 d=8, init 64
for it in (12, 16, 18):
    st = {}
    t = time.time()
    r = hb.integrate(hb.make_integrand("f2", 8), hb.HyperRect.unit_cube(8), hb.DriverConfig(1e-6, max_iterations=it, max_regions=1 << 34), initial_regions=64, stats=st)
    w = time.time() - t
    print(json.dumps(dict(probe="f2d8_init64", iters=it, peak=r.peak_regions, evals=r.total_f_evals, wall=w, evals_per_s_dev=r.total_f_evals / (st["device_ms"] * 1e-3), k1_evals_per_s=r.total_f_evals / (st["k1_ms"] * 1e-3), stats=st)), flush=True)
