"""Generate the golden fixtures under tests/golden/ by importing the REFERENCE.

Run in the build container only (needs /root/reference, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs (all small, committed):
  k1_<case>.npz     G1 - per-region rule outputs from `hcub.rules.apply_rule_batch`
                    on initial partitions, mid-run region sets and seeded
                    random dyadic boxes (fields lo, hi, integral, error,
                    scores, axis, evals)
  trace_<case>.json G2 - `hcub.driver.integrate` per-iteration traces plus an
                    order-independent sha256 of the active region set
  dist_<case>.json  G3 - `hcub.distributed.run_distributed(deterministic_sim,
                    collect_log=True)` logs, timings and results
  meta.json         numpy / BLAS provenance of the generating run

Nothing on the GPU box reads /root/reference; only these files travel.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import platform
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, OUT)

import hcub  # noqa: E402
from hcub.driver import classify_filter_split, evaluate_batch, GlobalEstimate  # noqa: E402
from hcub.regions import RegionStore, uniform_partition  # noqa: E402


def set_hash(lo, hi):
    rows = np.concatenate([lo, hi], axis=1)
    if len(rows):
        rows = rows[np.lexsort(rows.T[::-1])]
    return hashlib.sha256(np.ascontiguousarray(rows).tobytes()).hexdigest()


def make_f(spec):
    kind = spec["f"]
    d = spec["d"]
    if kind == "pp":
        f, exact = hcub.make_product_peak(d, center=spec.get("center", 0.5), sharpness=spec.get("sharpness", 50.0))
        return f
    return hcub.make_integrand(kind, d)


def domain(spec):
    d = spec["d"]
    if "lo" in spec:
        return hcub.HyperRect(np.array(spec["lo"], dtype=float), np.array(spec["hi"], dtype=float))
    return hcub.HyperRect.unit_cube(d)


def random_boxes(dom, n, seed):
    """Dyadic sub-boxes of ``dom``: per axis a level k in 0..19 and an index."""
    rng = np.random.default_rng(seed)
    d = dom.dim
    lo = np.empty((n, d))
    hi = np.empty((n, d))
    for j in range(d):
        k = rng.integers(0, 20, size=n)
        idx = np.floor(rng.random(n) * (2.0 ** k))
        ext = dom.hi[j] - dom.lo[j]
        lo[:, j] = dom.lo[j] + ext * (idx / 2.0 ** k)
        hi[:, j] = dom.lo[j] + ext * ((idx + 1) / 2.0 ** k)
    return lo, hi


def snapshots(spec, iters, cap_rows, seed):
    """Region stores as the reference loop holds them at given iterations."""
    d = spec["d"]
    f = make_f(spec)
    dom = domain(spec)
    cfg = hcub.DriverConfig(spec["tau"])
    table = hcub.get_rule("gm", d)
    store = RegionStore.from_rects(uniform_partition(dom, spec.get("init", 2 * d)))
    fin = (0.0, 0.0)
    out = []
    rng = np.random.default_rng(seed)
    for it in range(1, max(iters) + 1):
        if it in iters:
            lo, hi = store.lo, store.hi
            if len(lo) > cap_rows:
                pick = np.sort(rng.choice(len(lo), cap_rows, replace=False))
                lo, hi = lo[pick], hi[pick]
            out.append((lo.copy(), hi.copy()))
        est = evaluate_batch(store, table, f, finalized=fin)
        oc = classify_filter_split(store, est, cfg, dom)
        fin = (oc.finalized_integral, oc.finalized_error)
        store = oc.store
        if len(store) == 0:
            break
    return out


K1_CASES = {
    "f4_d3": dict(f="f4", d=3, tau=1e-6, iters=(1, 6, 12)),
    "f2_d2": dict(f="f2", d=2, tau=1e-8, iters=(1, 8)),
    "f2_d5": dict(f="f2", d=5, tau=1e-6, iters=(1, 3, 8, 12)),
    "f2_d8": dict(f="f2", d=8, tau=1e-6, iters=(1, 3, 8, 10)),
    "f2_d8_init64": dict(f="f2", d=8, tau=1e-6, init=64, iters=(1, 8)),
    "f3_d10": dict(f="f3", d=10, tau=1e-5, iters=(1, 3, 8)),
    "f6_d6": dict(f="f6", d=6, tau=1e-4, iters=(1, 3, 8, 12)),
    "f1_d4": dict(f="f1", d=4, tau=1e-8, iters=(1, 5)),
    "f5_d4": dict(f="f5", d=4, tau=1e-6, iters=(1, 5)),
    "f7_d3": dict(f="f7", d=3, tau=1e-8, iters=(1, 5)),
    "f2_d13": dict(f="f2", d=13, tau=1e-3, iters=(1,), nrand=256),
    "pp_d4_c01": dict(f="pp", d=4, center=0.1, tau=1e-6, iters=(1, 8, 16)),
    "pp_d6_s30": dict(f="pp", d=6, center=[0.2, 0.35, 0.5, 0.65, 0.8, 0.9], sharpness=30.0, tau=1e-6, iters=(1, 6)),
    "f2_d3_odd": dict(f="f2", d=3, tau=1e-8, lo=[-0.3, 0.1, 0.2], hi=[0.9, 0.7, 1.5], iters=(1, 6, 12)),
}

TRACE_CASES = {
    "f4_d3": dict(f="f4", d=3, tau=1e-6, max_iterations=1000),
    "f4_d3_init64": dict(f="f4", d=3, tau=1e-6, init=64, max_iterations=1000),
    "f2_d5": dict(f="f2", d=5, tau=1e-6, max_iterations=14),
    "f2_d8": dict(f="f2", d=8, tau=1e-6, max_iterations=11),
    "f2_d8_init64": dict(f="f2", d=8, tau=1e-6, init=64, max_iterations=10),
    "f3_d10": dict(f="f3", d=10, tau=1e-5, max_iterations=8),
    "f6_d6": dict(f="f6", d=6, tau=1e-4, max_iterations=12),
    "pp_d4_c01": dict(f="pp", d=4, center=0.1, tau=1e-6, max_iterations=1000),
    "f2_d3_odd": dict(f="f2", d=3, tau=1e-8, lo=[-0.3, 0.1, 0.2], hi=[0.9, 0.7, 1.5], max_iterations=1000),
    "f1_d4": dict(f="f1", d=4, tau=1e-8, max_iterations=1000),
    "f2_d3_maxreg": dict(f="f2", d=3, tau=1e-12, max_iterations=1000, max_regions=5000),
}

SLOW_TRACES = {  # run with `make_golden.py slow` (minutes of reference CPU time)
    "f2_d5_tau1e-3_wall": dict(f="f2", d=5, tau=1e-3, max_iterations=1000),
    # the north-star workload far enough (>= 3e5 regions) that the device takes
    # its one-region-per-lane K1 path
    "f2_d8_init64_its16": dict(f="f2", d=8, tau=1e-6, init=64, max_iterations=16),
}

# Long reference runs covering (most of) what the bench runs on the device
# (`make_golden.py long` or by name; tens of minutes to ~1 h of CPU each).
# One pass through the REAL `hcub.integrate`; the region set entering every
# evaluation is digested by wrapping `hcub.driver.evaluate_batch` (which
# `integrate` calls by module global), so the hashes and the trace come from
# the same run.  Large sets use the O(n) order-independent digest in
# setdigest.py instead of sha256 over a lexsorted copy.
LONG_TRACES = {
    # configs[1]: f2 d=5 rtol 1e-6 run to its own termination (max_regions raised)
    "long_f2_d5": dict(f="f2", d=5, tau=1e-6, max_iterations=1000, max_regions=1 << 40),
    # the north-star fixed-work workload (f2 d=8, 64-subdomain init), first 21 of 26 iterations
    "long_f2_d8_init64": dict(f="f2", d=8, tau=1e-6, init=64, max_iterations=21, max_regions=1 << 40),
    # configs[3] and configs[4] as the bench runs them (init 80 / 48)
    "long_f3_d10_init80": dict(f="f3", d=10, tau=1e-5, init=80, max_iterations=25, max_regions=1 << 40),
    "long_f6_d6_init48": dict(f="f6", d=6, tau=1e-4, init=48, max_iterations=25, max_regions=1 << 40),
    # configs[1] with the degree-9 rule, to its own termination (bench time_to_tolerance row)
    "long_gm9_f2_d5": dict(f="f2", d=5, tau=1e-6, max_iterations=1000, max_regions=1 << 40, rule="gm9"),
    # configs[3] with the degree-9 rule (d = 10 through the generator kernel), first iterations
    "long_gm9_f3_d10_init80": dict(f="f3", d=10, tau=1e-5, init=80, max_iterations=27, max_regions=1 << 40,
                                   rule="gm9"),
}

DIST_CASES = {
    "f4_d3_P2": dict(f="f4", d=3, tau=1e-6, P=2),
    "f4_d3_P4": dict(f="f4", d=3, tau=1e-6, P=4),
    "f4_d3_P8": dict(f="f4", d=3, tau=1e-6, P=8),
    "pp_d4_c01_P2": dict(f="pp", d=4, center=0.1, tau=1e-6, P=2),
    "pp_d4_c01_P3": dict(f="pp", d=4, center=0.1, tau=1e-5, P=3),
    "pp_d4_c01_P4": dict(f="pp", d=4, center=0.1, tau=1e-6, P=4),
    "pp_d4_c01_P8": dict(f="pp", d=4, center=0.1, tau=1e-6, P=8),
    "pp_d4_c01_P4_cap16": dict(f="pp", d=4, center=0.1, tau=1e-5, P=4, cap=16, per_rank=3),
    # delivery_latency > 1: batches stay in flight for several iterations, the
    # conservative in-flight bounds enter every metadata reduce (ref :475-489, :549)
    "pp_d4_c01_P4_lat2": dict(f="pp", d=4, center=0.1, tau=1e-6, P=4, latency=2),
    "pp_d4_c01_P3_lat3": dict(f="pp", d=4, center=0.1, tau=1e-5, P=3, latency=3),
    "pp_d4_c01_P8_lat2_cap16": dict(f="pp", d=4, center=0.1, tau=1e-5, P=8, cap=16, per_rank=2, latency=2),
    # the rebalancing stress shapes of BASELINE configs[3]/[4] at CPU size
    "f3_d4_P4": dict(f="f3", d=4, tau=1e-6, P=4),
    "f6_d3_P4_lat2": dict(f="f6", d=3, tau=1e-5, P=4, latency=2),
}


def gen_k1(name, spec):
    d = spec["d"]
    f = make_f(spec)
    dom = domain(spec)
    table = hcub.get_rule("gm", d)
    los, his, tags = [], [], []
    for i, (lo, hi) in enumerate(snapshots(spec, spec["iters"], 1024, seed=1)):
        los.append(lo)
        his.append(hi)
        tags += [spec["iters"][i]] * len(lo)
    lo, hi = random_boxes(dom, spec.get("nrand", 1024), seed=0)
    los.append(lo)
    his.append(hi)
    tags += [0] * len(lo)
    lo = np.concatenate(los)
    hi = np.concatenate(his)
    integral, error, scores, evals = hcub.apply_rule_batch(table, lo, hi, f)
    np.savez_compressed(
        os.path.join(OUT, f"k1_{name}.npz"),
        lo=lo, hi=hi, integral=integral, error=error, scores=scores,
        axis=np.argmax(scores, axis=1).astype(np.int64), evals=np.int64(evals),
        tag=np.array(tags, dtype=np.int64), spec=json.dumps(spec),
    )
    return len(lo)


def gen_trace(name, spec):
    d = spec["d"]
    f = make_f(spec)
    dom = domain(spec)
    cfg = hcub.DriverConfig(spec["tau"], max_iterations=spec["max_iterations"],
                            max_regions=spec.get("max_regions", 1 << 24), rule=spec.get("rule", "gm"))
    import hcub.driver as hd
    table = hd.get_rule(cfg.rule, d)
    # hashes of the active set entering each evaluation, recomputed with the
    # reference's own building blocks (same sequence integrate() runs)
    hashes = []
    store = RegionStore.from_rects(uniform_partition(dom, spec.get("init", 2 * d)))
    fin = (0.0, 0.0)
    for it in range(1, spec["max_iterations"] + 1):
        hashes.append(set_hash(store.lo, store.hi))
        est = evaluate_batch(store, table, f, finalized=fin)
        if hcub.check_convergence(est, cfg):
            break
        oc = classify_filter_split(store, est, cfg, dom)
        fin = (oc.finalized_integral, oc.finalized_error)
        store = oc.store
        if len(store) == 0 or len(store) > cfg.max_regions:
            break
    tr = []
    t0 = time.time()
    res = hcub.integrate(f, dom, cfg, trace=tr.append, initial_regions=spec.get("init"))
    wall = time.time() - t0
    doc = dict(
        spec=spec,
        trace=[[t.iteration, t.active_regions, t.integral, t.error, t.f_evals] for t in tr],
        set_hashes=hashes[: len(tr)],
        result=dict(integral=res.integral, error=res.error, converged=res.converged,
                    iterations=res.iterations, total_f_evals=res.total_f_evals,
                    peak_regions=res.peak_regions, termination_reason=res.termination_reason.value),
        wall_s=wall,
    )
    with open(os.path.join(OUT, f"trace_{name}.json"), "w") as fh:
        json.dump(doc, fh, indent=1)
    return res.iterations


def gen_long_trace(name, spec):
    from setdigest import set_digest
    import hcub.driver as drv
    d = spec["d"]
    f = make_f(spec)
    dom = domain(spec)
    cfg = hcub.DriverConfig(spec["tau"], max_iterations=spec["max_iterations"],
                            max_regions=spec.get("max_regions", 1 << 24), rule=spec.get("rule", "gm"))
    orig_get_rule = drv.get_rule
    if spec.get("rule") == "gm9":  # the reference's own parse_rule_table of the degree-9 text
        from hcub.rules import parse_rule_table
        t9 = parse_rule_table(gm9_text(d), name="gm9", degree=9, embedded_degree=7)
        drv.get_rule = lambda rule, dd: t9 if rule == "gm9" else orig_get_rule(rule, dd)
    digests, walls = [], []
    real_eval = drv.evaluate_batch
    t0 = time.time()

    def evaluate_batch(store, table, f, finalized=(0.0, 0.0)):
        digests.append(set_digest(store.lo, store.hi))
        walls.append(time.time() - t0)
        print(name, "iteration", len(digests), len(store), round(walls[-1], 1), flush=True)
        return real_eval(store, table, f, finalized=finalized)

    drv.evaluate_batch = evaluate_batch
    tr = []
    try:
        res = hcub.integrate(f, dom, cfg, trace=tr.append, initial_regions=spec.get("init"))
    finally:
        drv.evaluate_batch = real_eval
        drv.get_rule = orig_get_rule
    wall = time.time() - t0
    doc = dict(
        spec=spec,
        trace=[[t.iteration, t.active_regions, t.integral, t.error, t.f_evals] for t in tr],
        set_digests=digests,
        wall_at_iteration_s=walls,
        result=dict(integral=res.integral, error=res.error, converged=res.converged,
                    iterations=res.iterations, total_f_evals=res.total_f_evals,
                    peak_regions=res.peak_regions, termination_reason=res.termination_reason.value),
        wall_s=wall,
        host=dict(cpu=platform.processor() or platform.machine(), cores=os.cpu_count(),
                  openblas_threads=os.environ.get("OPENBLAS_NUM_THREADS")),
    )
    with open(os.path.join(OUT, f"trace_{name}.json"), "w") as fh:
        json.dump(doc, fh, indent=1)
    return res.iterations


def gen_dist(name, spec):
    d = spec["d"]
    f = make_f(spec)
    dom = domain(spec)
    cfg = hcub.DriverConfig(spec["tau"])
    rcfg = hcub.RedistributionConfig(cap=spec.get("cap", 512), initial_subdomains_per_rank=spec.get("per_rank", 8),
                                     delivery_latency=spec.get("latency", 1))
    dr = hcub.run_distributed(f, dom, cfg, rcfg, workers=spec["P"], collect_log=True)
    res = dr.result
    doc = dict(
        spec=spec,
        result=dict(integral=res.integral, error=res.error, converged=res.converged,
                    iterations=res.iterations, total_f_evals=res.total_f_evals,
                    peak_regions=res.peak_regions, termination_reason=res.termination_reason.value),
        messages_total=dr.messages_total,
        regions_transferred_total=dr.regions_transferred_total,
        final_reduce_integral=dr.final_reduce_integral,
        final_reduce_error=dr.final_reduce_error,
        timings=[dict(rank=t.rank, iterations=t.iterations, compute=t.compute_seconds, idle=t.idle_seconds,
                      messages_out=t.messages_out, regions_out=t.regions_out) for t in dr.timings],
        log=dr.iteration_log,
    )
    with open(os.path.join(OUT, f"dist_{name}.json"), "w") as fh:
        json.dump(doc, fh, indent=1)
    return res.iterations, dr.messages_total


SWEEPS = {
    "accuracy_f4_d3": ("accuracy", dict(functions=("f4",), dims=(3,), tolerances=(1e-3, 1e-4, 1e-5), workers=(1, 2))),
    "scaling_f2_d3": ("scaling", dict(functions=("f2",), dims=(3,), tolerances=(1e-4,), workers=(1, 2, 4))),
    "idle_f6_d3": ("idle", dict(functions=("f6",), dims=(3,), tolerances=(1e-3,), workers=(2, 3))),
}


def gen_sweep(name, kind_spec):
    from hcub import experiments as ex
    kind, kw = kind_spec
    spec = ex.ExperimentSpec(output_path=os.path.join(OUT, f"sweep_{name}.csv"), **kw)
    runner, cols = {"accuracy": (ex.run_accuracy_sweep, ex.ACCURACY_COLUMNS),
                    "scaling": (ex.run_scaling_sweep, ex.SCALING_COLUMNS),
                    "idle": (ex.run_idle_breakdown, ex.IDLE_COLUMNS)}[kind]
    rows = runner(spec)
    ex.write_rows(rows, cols, spec.output_path)
    return len(rows)


def gm_text(d, drop=()):
    t = hcub.build_gm_rule(d)
    return "\n".join(" ".join(map(repr, list(o.generator) + [o.weight, o.embedded_weight]))
                     for i, o in enumerate(t.orbits) if i not in drop)


def gm9_text(d):
    # the degree-9 table's text (input data; generated by the repo's rule9.py,
    # parsed and applied below by the REFERENCE's parse_rule_table / apply_rule_batch)
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from paper_2511_01573_b200.rule9 import gm9_rule_text
    return gm9_rule_text(d)


TABLE_CASES = {
    "gm_d3_text": dict(f="f2", d=3, text=gm_text(3)),
    "gm_d5_text_f4": dict(f="f4", d=5, text=gm_text(5)),
    "gm_d3_no_lam3": dict(f="f2", d=3, text=gm_text(3, drop=(2,))),
    "d1_five_point": dict(f="f2", d=1, text="0 1.1 0.9\n0.5 0.3 0.4\n0.9 0.15 0.15"),
    "pp_d4_gm_text": dict(f="pp", d=4, center=0.1, text=gm_text(4)),
    # degree-9 fully symmetric rule (3-nonzero orbit, O(d^3) nodes), SURVEY.md 8f-2
    "gm9_d3_f2": dict(f="f2", d=3, text=gm9_text(3)),
    "gm9_d5_f2": dict(f="f2", d=5, text=gm9_text(5)),
    "gm9_d8_f2": dict(f="f2", d=8, text=gm9_text(8)),
    "gm9_d6_pp": dict(f="pp", d=6, center=0.3, text=gm9_text(6)),
    "gm9_d4_f4": dict(f="f4", d=4, text=gm9_text(4)),
    "gm9_d9_f2": dict(f="f2", d=9, text=gm9_text(9)),
    "gm9_d10_f3": dict(f="f3", d=10, text=gm9_text(10)),
}

# whole integrate() runs with the degree-9 table (the reference's get_rule
# resolves "gm9" to parse_rule_table(text) for these runs only)
GM9_TRACES = {
    "gm9_f4_d3": dict(f="f4", d=3, tau=1e-8, max_iterations=1000),
    "gm9_f2_d5": dict(f="f2", d=5, tau=1e-6, max_iterations=10),
    "gm9_pp_d4_c01": dict(f="pp", d=4, center=0.1, tau=1e-7, max_iterations=1000),
}


def gen_gm9_trace(name, spec):
    import hcub.driver as hd
    from hcub.rules import parse_rule_table
    orig = hd.get_rule
    table = parse_rule_table(gm9_text(spec["d"]), name="gm9", degree=9, embedded_degree=7)
    hd.get_rule = lambda rule, d: table if rule == "gm9" else orig(rule, d)
    try:
        return gen_trace(name, dict(spec, rule="gm9"))
    finally:
        hd.get_rule = orig


def gen_table(name, spec):
    from hcub.rules import parse_rule_table
    table = parse_rule_table(spec["text"])
    f = make_f(spec)
    dom = domain(spec)
    lo, hi = random_boxes(dom, 512, seed=3)
    integral, error, scores, evals = hcub.apply_rule_batch(table, lo, hi, f)
    np.savez_compressed(os.path.join(OUT, f"table_{name}.npz"), lo=lo, hi=hi, integral=integral, error=error,
                        scores=scores, axis=np.argmax(scores, axis=1).astype(np.int64), evals=np.int64(evals),
                        spec=json.dumps(spec), has_cascade=np.int64(table.axis_pairs is not None))
    return len(lo)


GK_CASES = {
    "gk_d1_f2": dict(f="f2", d=1, n=256),
    "gk_d2_f4": dict(f="f4", d=2, n=256),
    "gk_d3_pp": dict(f="pp", d=3, center=0.3, n=128),
    "gk_d4_f5": dict(f="f5", d=4, n=32),
    "gk_d6_f2": dict(f="f2", d=6, n=2),
}

GK_TRACES = {
    "gk_trace_d1_f2": dict(f="f2", d=1, tau=1e-10, rule="gm", max_iterations=1000),
    "gk_trace_d2_f4": dict(f="f4", d=2, tau=1e-8, rule="gk-tensor", max_iterations=1000),
}


def gen_gk(name, spec):
    table = hcub.build_gk_tensor_rule(spec["d"])
    f = make_f(spec)
    lo, hi = random_boxes(domain(spec), spec["n"], seed=4)
    integral, error, scores, evals = hcub.apply_rule_batch(table, lo, hi, f)
    np.savez_compressed(os.path.join(OUT, f"gk_{name}.npz"), lo=lo, hi=hi, integral=integral, error=error,
                        scores=scores, axis=np.argmax(scores, axis=1).astype(np.int64), evals=np.int64(evals),
                        spec=json.dumps(spec))
    return len(lo)


def gen_gk_trace(name, spec):
    f = make_f(spec)
    cfg = hcub.DriverConfig(spec["tau"], rule=spec["rule"], max_iterations=spec["max_iterations"])
    tr = []
    res = hcub.integrate(f, domain(spec), cfg, trace=tr.append)
    doc = dict(spec=spec, trace=[[t.iteration, t.active_regions, t.integral, t.error, t.f_evals] for t in tr],
               result=dict(integral=res.integral, error=res.error, converged=res.converged,
                           iterations=res.iterations, total_f_evals=res.total_f_evals,
                           peak_regions=res.peak_regions, termination_reason=res.termination_reason.value))
    with open(os.path.join(OUT, f"trace_{name}.json"), "w") as fh:
        json.dump(doc, fh, indent=1)
    return res.iterations


def main():
    only = set(sys.argv[1:])
    for name, spec in K1_CASES.items():
        if not only or name in only or "k1" in only:
            print("k1", name, gen_k1(name, spec), flush=True)
    for name, spec in TRACE_CASES.items():
        if not only or name in only or "trace" in only:
            print("trace", name, gen_trace(name, spec), flush=True)
    for name, spec in DIST_CASES.items():
        if not only or name in only or "dist" in only:
            print("dist", name, gen_dist(name, spec), flush=True)
    for name, spec in SLOW_TRACES.items():
        if "slow" in only or name in only:
            print("trace", name, gen_trace(name, spec), flush=True)
    for name, spec in LONG_TRACES.items():
        if "long" in only or name in only:
            print("long trace", name, gen_long_trace(name, spec), flush=True)
    for name, spec in TABLE_CASES.items():
        if not only or name in only or "table" in only:
            print("table", name, gen_table(name, spec), flush=True)
    for name, spec in GM9_TRACES.items():
        if not only or name in only or "gm9" in only:
            print("gm9 trace", name, gen_gm9_trace(name, spec), flush=True)
    for name, spec in GK_CASES.items():
        if not only or name in only or "gk" in only:
            print("gk", name, gen_gk(name, spec), flush=True)
    for name, spec in GK_TRACES.items():
        if not only or name in only or "gk" in only:
            print("gk trace", name, gen_gk_trace(name, spec), flush=True)
    for name, ks in SWEEPS.items():
        if not only or name in only or "sweep" in only:
            print("sweep", name, gen_sweep(name, ks), flush=True)
    meta = dict(numpy=np.__version__, python=platform.python_version(), machine=platform.machine(),
                blas=str(np.show_config(mode="dicts")["Build Dependencies"]["blas"].get("version")),
                generated_utc=time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
                reference=REF)
    with open(os.path.join(OUT, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
