"""The degree-9 fully symmetric table (paper_2511_01573_b200/rule9.py, SURVEY.md
8f-2): polynomial exactness re-derived numerically from the parsed node table
(independent of the rational derivation that produced the weights), node
counts, the axis bookkeeping a loaded table gets, and identity with the
reference's own parse_rule_table on the same text (when /root/reference is
present, i.e. in the build container)."""
import math
import os
import sys

import numpy as np
import pytest

from paper_2511_01573_b200.rule9 import build_gm9_rule, gm9_lambdas, gm9_rule_text, gm9_weights
from paper_2511_01573_b200.rules import _axis_bookkeeping


def monomials(d, max_deg, rng, count):
    """Random exponent vectors of total degree <= max_deg (odd ones included:
    they must integrate to 0 by symmetry)."""
    out = [np.zeros(d, dtype=int)]
    for _ in range(count):
        deg = rng.integers(1, max_deg + 1)
        e = np.zeros(d, dtype=int)
        for _ in range(deg):
            e[rng.integers(0, d)] += 1
        out.append(e)
    return out


def cube_moment(e):
    # integral over [-1,1]^d of prod x^e, divided by 2^d
    return math.prod(0.0 if k % 2 else 1.0 / (k + 1) for k in e)


@pytest.mark.parametrize("d", [2, 3, 4, 5, 6, 8])
def test_degree9_and_embedded_degree7_exactness(d):
    t = build_gm9_rule(d)
    rng = np.random.default_rng(d)
    P, w, we = t.points, t.weights, t.embedded_weights
    scale = 2.0 ** d
    for e in monomials(d, 9, rng, 150):
        vals = np.prod(P ** e, axis=1)
        exact = cube_moment(e)
        got = vals @ w / scale
        assert abs(got - exact) <= 5e-14 * max(1.0, np.abs(w) @ np.abs(vals) / scale), (e, got, exact)
        if e.sum() <= 7:
            got7 = vals @ we / scale
            assert abs(got7 - exact) <= 5e-14 * max(1.0, np.abs(we) @ np.abs(vals) / scale), (e, got7, exact)
    # the embedded rule is genuinely lower degree: x1^8 is not integrated exactly
    e8 = np.zeros(d, dtype=int)
    e8[0] = 8
    assert abs(np.prod(P ** e8, axis=1) @ we / scale - 1.0 / 9) > 1e-6


@pytest.mark.parametrize("d", [2, 3, 5, 8, 10, 13])
def test_node_count_and_bookkeeping(d):
    t = build_gm9_rule(d)
    assert t.node_count == 1 + 8 * d + 6 * d * (d - 1) + 4 * d * (d - 1) * (d - 2) // 3 + 2 ** d
    assert t.degree == 9 and t.embedded_degree == 7
    # two smallest on-axis magnitudes: g2 (lam_in), g0 (lam_out)
    lam0, lam1, lam2, lam3 = (float(x) for x in gm9_lambdas())
    book = _axis_bookkeeping(t.points, t.orbits, d)
    assert math.isclose(book["ratio"], (math.sqrt(lam2) / math.sqrt(lam0)) ** 2, rel_tol=1e-15)
    names = [n for n, *_ in gm9_weights(d)]
    assert ("triple111" in names) == (d >= 3)
    w = {n: (a, b) for n, _, a, b in gm9_weights(d)}
    assert w["axis0"] == (0, 0)  # error-estimation nodes only (as in DCUHRE)


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree only in the build container")
@pytest.mark.parametrize("d", [3, 5, 8])
def test_reference_parses_the_same_table(d):
    sys.path.insert(0, REF)
    try:
        from hcub.rules import parse_rule_table as ref_parse
    finally:
        sys.path.remove(REF)
    mine = build_gm9_rule(d)
    ref = ref_parse(gm9_rule_text(d), name="gm9", degree=9, embedded_degree=7)
    assert ref.node_count == mine.node_count
    assert np.array_equal(ref.points, mine.points)
    assert np.array_equal(ref.weights, mine.weights)
    assert np.array_equal(ref.embedded_weights, mine.embedded_weights)
    book = _axis_bookkeeping(mine.points, mine.orbits, d)
    assert np.array_equal(ref.axis_pairs.reshape(d, 4), book["pairs"])
    assert ref.fourth_diff_ratio == book["ratio"]
    assert ref.null_axis_weight == book["null_axis"] and ref.null_center_weight == book["null_center"]
