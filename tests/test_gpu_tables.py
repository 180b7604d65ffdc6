"""Custom fully symmetric rule tables (parse_rule_table) on the device
(k1_table_eval) vs the reference's apply_rule_batch on the same tables."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2511_01573_b200 as hb
from paper_2511_01573_b200.rules import parse_rule_table

pytestmark = pytest.mark.gpu

CASES = sorted(f[6:-4] for f in os.listdir(GOLDEN) if f.startswith("table_") and f.endswith(".npz"))


def load(name):
    z = np.load(os.path.join(GOLDEN, f"table_{name}.npz"))
    g = {k: z[k] for k in z.files}
    g["spec"] = json.loads(str(g["spec"]))
    return g


@pytest.mark.parametrize("name", CASES)
def test_table_rule_matches_reference(name):
    g = load(name)
    spec = g["spec"]
    table = parse_rule_table(spec["text"])
    if spec["f"] == "pp":
        f = hb.make_product_peak(spec["d"], spec.get("center", 0.5))[0]
    else:
        f = hb.make_integrand(spec["f"], spec["d"])
    I, E, S, ev = hb.apply_rule_batch(table, g["lo"], g["hi"], f)
    assert ev == int(g["evals"])
    np.testing.assert_allclose(I, g["integral"], rtol=1e-12, atol=1e-300)
    big = g["error"] > 1e-9 * g["error"].max()
    np.testing.assert_allclose(E[big], g["error"][big], rtol=1e-6)
    if spec["f"] in ("f2", "pp"):
        assert np.array_equal(S, g["scores"])  # exact on-axis path (or extents)
        assert np.array_equal(np.argmax(S, axis=1), g["axis"])
    else:
        assert np.mean(np.argmax(S, axis=1) == g["axis"]) > 0.97


def test_integrate_with_custom_table_equals_builtin_gm():
    """DriverConfig(rule=<table>) (B200 extra): the GM table given as text
    yields the built-in rule's run (same counts, estimates to 1e-12)."""
    d = 4
    t = hb.build_gm_rule(d)
    text = "\n".join(" ".join(map(repr, list(o.generator) + [o.weight, o.embedded_weight])) for o in t.orbits)
    table = parse_rule_table(text)
    f = hb.make_integrand("f2", d)
    a, b = [], []
    ra = hb.integrate(f, hb.HyperRect.unit_cube(d), hb.DriverConfig(1e-6), trace=a.append)
    rb = hb.integrate(f, hb.HyperRect.unit_cube(d), hb.DriverConfig(1e-6, rule=table), trace=b.append)
    assert [x.active_regions for x in a] == [x.active_regions for x in b]
    assert ra.iterations == rb.iterations and ra.total_f_evals == rb.total_f_evals
    assert abs(ra.integral - rb.integral) <= 1e-12 * abs(ra.integral)


@pytest.mark.parametrize("name", [c for c in CASES if c.startswith("gm9_")])
def test_gm9_generator_kernel_matches_reference(name):
    """The degree-9 table built by rule9.build_gm9_rule is evaluated in
    generator form (csrc/k1_gm9.cuh, descriptor kind 3) - same reference
    outputs as the node-table kernel: scores bit-exact for f2 / product peak,
    integrals 1e-12, errors 1e-6 (cascade cancellation)."""
    from paper_2511_01573_b200.rule9 import build_gm9_rule
    g = load(name)
    spec = g["spec"]
    table = build_gm9_rule(spec["d"])
    assert table.descriptor().kind == 3
    if spec["f"] == "pp":
        f = hb.make_product_peak(spec["d"], spec.get("center", 0.5))[0]
    else:
        f = hb.make_integrand(spec["f"], spec["d"])
    I, E, S, ev = hb.apply_rule_batch(table, g["lo"], g["hi"], f)
    assert ev == int(g["evals"])
    np.testing.assert_allclose(I, g["integral"], rtol=1e-12, atol=1e-300)
    big = g["error"] > 1e-9 * g["error"].max()
    np.testing.assert_allclose(E[big], g["error"][big], rtol=1e-6)
    if spec["f"] in ("f2", "pp"):
        assert np.array_equal(S, g["scores"])
        assert np.array_equal(np.argmax(S, axis=1), g["axis"])
    else:
        assert np.mean(np.argmax(S, axis=1) == g["axis"]) > 0.97


def test_gm9_generator_rejects_other_tables():
    """Descriptor kind 3 is checked against the rule9 orbit layout: a table
    claiming the family without its structure raises instead of being
    mis-evaluated."""
    from paper_2511_01573_b200.rule9 import gm9_rule_text
    f = hb.make_integrand("f2", 4)
    lo = np.zeros((1, 4))
    hi = np.ones((1, 4))
    bad = parse_rule_table("\n".join(gm9_rule_text(4).splitlines()[:-1]))  # corners dropped
    bad.family = "gm9"
    with pytest.raises(ValueError):
        hb.apply_rule_batch(bad, lo, hi, f)


def test_cli_integrate_with_degree9_rule(capsys):
    """`hcub integrate --rule gm9` (B200 extra): the CLI runs the degree-9
    rule through run_distributed and reports convergence."""
    from paper_2511_01573_b200 import cli
    rc = cli.main(["integrate", "--function", "f2", "--dim", "4", "--tol", "1e-6", "--rule", "gm9"])
    out = capsys.readouterr().out
    assert rc == 0
    assert "termination" in out and "tolerance" in out
