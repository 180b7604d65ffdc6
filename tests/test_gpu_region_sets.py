"""Strongest parity check: drive the device store through the reference's
iteration (evaluate -> classify/split) and compare the sha256 of the sorted
active region set with the reference's at EVERY iteration (golden G2).

f2 / product peak: the score path is bit-exact, so every iteration must
match.  Integrands whose reference values go through libm/BLAS (exp, cos,
pow, dgemv) can flip a rounding-decided axis tie late in a run; for those the
sets must agree for at least the first MIN_SOFT iterations (and region counts
always agree - tests/test_gpu_integrate.py)."""
import hashlib
import os
import sys

import numpy as np
import pytest

from conftest import domain_of, load_json

import paper_2511_01573_b200 as hb
from paper_2511_01573_b200.regions import partition_arrays
from paper_2511_01573_b200.worker import DeviceWorker

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
from setdigest import set_digest  # noqa: E402

pytestmark = pytest.mark.gpu
MIN_SOFT = {"f1": 3}  # f1's reference dot products go through OpenBLAS dgemv (blocking-dependent)


def set_hash(lo, hi):
    rows = np.concatenate([lo, hi], axis=1)
    if len(rows):
        rows = rows[np.lexsort(rows.T[::-1])]
    return hashlib.sha256(np.ascontiguousarray(rows).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["f4_d3", "f2_d5", "f2_d8", "f2_d8_init64", "pp_d4_c01", "f2_d3_odd", "f6_d6",
                                  "f3_d10", "f1_d4",
                                  # 3.2e5..1.1e6 regions in the last iterations: the
                                  # one-region-per-lane K1 path, fused sums, device split
                                  "f2_d8_init64_its16",
                                  # 43 iterations down to an empty store (width guard)
                                  "f2_d5_tau1e-3_wall",
                                  # the degree-9 table (k1_table_eval) through the loop
                                  "gm9_f4_d3", "gm9_f2_d5", "gm9_pp_d4_c01"])
def test_region_set_hashes_every_iteration(name):
    g = load_json("trace", name)
    spec = g["spec"]
    d = spec["d"]
    if spec["f"] == "pp":
        f = hb.make_product_peak(d, spec.get("center", 0.5), spec.get("sharpness", 50.0))[0]
    else:
        f = hb.make_integrand(spec["f"], d)
    dlo, dhi = domain_of(spec)
    dom = hb.HyperRect(dlo, dhi)
    cfg = hb.DriverConfig(spec["tau"], max_iterations=spec["max_iterations"])
    w = DeviceWorker(hb.get_rule(spec.get("rule", "gm"), d), f, dom)
    lo, hi = partition_arrays(dom, spec.get("init", 2 * d))
    w.append(lo, hi)
    strict = spec["f"] in ("f2", "pp")
    for it, want in enumerate(g["set_hashes"], start=1):
        slo, shi, _, _, _ = w.read()
        if set_hash(slo, shi) != want:
            assert not strict and it > MIN_SOFT.get(spec["f"], 6), f"region set differs at iteration {it}"
            break
        I, E, _ = w.evaluate()
        if E <= max(cfg.abs_floor, abs(I) * cfg.tau_rel) or it == len(g["set_hashes"]):
            break
        oc = w.classify(I, cfg)
        if oc.split_count == 0:
            break
    w.close()


# iterations whose region sets must coincide with the reference's long runs
# (f2: every one; f3 / f6 go through libm pow / exp on the on-axis nodes)
# (measured: f3 12 of 25 - a rounding-decided axis tie flips at iteration
# 13 while the region counts stay equal to the end; f6 all 22; degree-9 f3 24 of 27)
LONG_MIN_MATCH = {"long_f2_d5": None, "long_f2_d8_init64": None, "long_f3_d10_init80": 12, "long_f6_d6_init48": None,
                  "long_gm9_f2_d5": None, "long_gm9_f3_d10_init80": 24}


@pytest.mark.parametrize("name", sorted(LONG_MIN_MATCH))
def test_long_run_region_set_digests_every_iteration(name):
    """The benchmarked workloads as far as the reference ran them on the CPU
    (tests/golden/make_golden.py long: up to 6.3e7 regions): the active
    region set entering every evaluation, digested order-independently
    (tests/golden/setdigest.py, the same numpy code on both sides), equals
    the reference's."""
    g = load_json("trace", name)
    spec = g["spec"]
    d = spec["d"]
    f = hb.make_integrand(spec["f"], d)
    dom = hb.HyperRect.unit_cube(d)
    cfg = hb.DriverConfig(spec["tau"], max_iterations=spec["max_iterations"], max_regions=spec["max_regions"])
    w = DeviceWorker(hb.get_rule(spec.get("rule", "gm"), d), f, dom)
    lo, hi = partition_arrays(dom, spec.get("init", 2 * d))
    w.append(lo, hi)
    matched = 0
    try:
        for it, want in enumerate(g["set_digests"], start=1):
            slo, shi, _, _, _ = w.read()
            got = set_digest(slo, shi)
            del slo, shi
            if got != want:
                break
            matched = it
            I, E, _ = w.evaluate()
            if E <= max(cfg.abs_floor, abs(I) * cfg.tau_rel) or it == len(g["set_digests"]):
                break
            oc = w.classify(I, cfg)
            if oc.split_count == 0:
                break
    finally:
        w.close()
    need = LONG_MIN_MATCH[name] or len(g["set_digests"])
    print(f"{name}: region sets coincide for {matched} of {len(g['set_digests'])} iterations")
    assert matched >= need, f"region set differs at iteration {matched + 1}"
