"""Pin the CPU oracle (oracle/hcub_oracle.py) against golden vectors that
tests/golden/make_golden.py produced by running the reference itself.

Quantities computed without BLAS (geometry, f2/product-peak node values,
axis scores, split axes, region-set hashes, counts) must match bit for bit;
BLAS-ordered sums (integral/error) to rounding (the GPU box's OpenBLAS may
pick another kernel than the generating host).
"""
import math

import numpy as np
import pytest

from conftest import domain_of, golden_names, load_json, load_k1, oracle_f
from oracle import hcub_oracle as orc

BITEXACT_F = {"f2", "pp"}  # no BLAS / libm on the score path


@pytest.mark.parametrize("name", golden_names("k1"))
def test_oracle_k1_matches_reference(name):
    g = load_k1(name)
    spec = g["spec"]
    tab = orc.gm_table(spec["d"])
    I, E, S, ev = orc.eval_regions(tab, g["lo"], g["hi"], oracle_f(spec))
    assert ev == int(g["evals"])
    np.testing.assert_allclose(I, g["integral"], rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(E, g["error"], rtol=1e-6, atol=1e-300)
    if spec["f"] in BITEXACT_F:
        assert np.array_equal(S, g["scores"])
        assert np.array_equal(np.argmax(S, axis=1), g["axis"])
    else:
        np.testing.assert_allclose(S, g["scores"], rtol=1e-9, atol=1e-300)
        assert np.mean(np.argmax(S, axis=1) == g["axis"]) > 0.97


@pytest.mark.parametrize("d", range(2, 14))
def test_node_count_and_degree0(d):
    tab = orc.gm_table(d)
    assert tab.K == 2 ** d + 2 * d * d + 2 * d + 1  # ref rules.py:261
    assert math.isclose(tab.w.sum(), 2.0 ** d, rel_tol=1e-13)
    assert math.isclose(tab.we.sum(), 2.0 ** d, rel_tol=1e-13)


FAST_TRACES = ["f4_d3", "f4_d3_init64", "f2_d3_odd", "f1_d4", "f2_d3_maxreg", "f6_d6", "f3_d10"]


@pytest.mark.parametrize("name", FAST_TRACES)
def test_oracle_trace_matches_reference(name):
    g = load_json("trace", name)
    spec = g["spec"]
    dlo, dhi = domain_of(spec)
    r = orc.integrate(oracle_f(spec), spec["d"], spec["tau"], dlo, dhi, init=spec.get("init"),
                      max_iterations=spec["max_iterations"], max_regions=spec.get("max_regions", 1 << 24),
                      hashes=True)
    assert r.termination_reason == g["result"]["termination_reason"]
    assert r.iterations == g["result"]["iterations"]
    assert r.total_f_evals == g["result"]["total_f_evals"]
    assert r.peak_regions == g["result"]["peak_regions"]
    assert [t[1] for t in r.trace] == [t[1] for t in g["trace"]]
    assert r.set_hashes == g["set_hashes"]
    for mine, ref in zip(r.trace, g["trace"]):
        assert math.isclose(mine[2], ref[2], rel_tol=1e-12)
        assert math.isclose(mine[3], ref[3], rel_tol=1e-9)
    assert math.isclose(r.integral, g["result"]["integral"], rel_tol=1e-12)


@pytest.mark.parametrize("name", ["f4_d3_P2", "f4_d3_P4", "f4_d3_P8", "pp_d4_c01_P3", "pp_d4_c01_P4_cap16"])
def test_oracle_distributed_matches_reference(name):
    g = load_json("dist", name)
    spec = g["spec"]
    dr = orc.run_distributed(oracle_f(spec), spec["d"], spec["tau"], spec["P"], cap=spec.get("cap", 512),
                             per_rank=spec.get("per_rank", 8))
    res = g["result"]
    assert dr.result.termination_reason == res["termination_reason"]
    assert dr.result.iterations == res["iterations"]
    assert dr.result.total_f_evals == res["total_f_evals"]
    assert dr.result.peak_regions == res["peak_regions"]
    assert dr.messages_total == g["messages_total"]
    assert dr.regions_transferred_total == g["regions_transferred_total"]
    assert len(dr.log) == len(g["log"])
    for mine, ref in zip(dr.log, g["log"]):
        for key in ("counts", "post_split_counts", "inflight_regions", "census"):
            assert mine[key] == ref[key], (key, mine["iteration"])
        assert [list(t) for t in mine["transfers"]] == [list(t) for t in ref["transfers"]]
        assert math.isclose(mine["global_integral"], ref["global_integral"], rel_tol=1e-12)
    assert [t for t in dr.compute] == [t["compute"] for t in g["timings"]]
    assert [t for t in dr.idle] == [t["idle"] for t in g["timings"]]
    assert math.isclose(dr.result.integral, res["integral"], rel_tol=1e-12)


def test_round_robin_schedule_spec_examples():
    # every unordered pair exactly once over P-1 rounds (even P) / P rounds (odd P)
    for P in range(2, 10):
        rounds = P - 1 if P % 2 == 0 else P
        seen = []
        for r in range(rounds):
            pairs = orc.rr_pairs(P, r)
            flat = [x for p in pairs for x in p]
            assert len(flat) == len(set(flat))
            seen += [tuple(sorted(p)) for p in pairs]
        assert sorted(seen) == sorted((a, b) for a in range(P) for b in range(a + 1, P))
