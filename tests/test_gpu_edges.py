"""Edge cases of the drop-in surface on the B200 (the reference's own
behaviour in parentheses): empty and single-row batches, ragged/odd domains,
the largest dimension, one-iteration runs, bad configs."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_apply_rule_batch_empty_and_single_row():
    import paper_2511_01573_b200 as hb
    f = hb.make_integrand("f2", 5)
    t = hb.build_gm_rule(5)
    I, E, S, ev = hb.apply_rule_batch(t, np.zeros((0, 5)), np.zeros((0, 5)), f)  # (empty arrays, 0 evals)
    assert I.shape == (0,) and E.shape == (0,) and S.shape == (0, 5) and ev == 0
    I, E, S, ev = hb.apply_rule_batch(t, np.zeros((1, 5)), np.ones((1, 5)), f)
    assert I.shape == (1,) and ev == t.node_count


def test_max_dimension_matches_oracle():
    """d = 13, the largest Genz-Malik dimension (ref rules.py:266-269): K1 vs
    the oracle on random boxes - bit-exact scores/axes for f2."""
    import paper_2511_01573_b200 as hb
    from oracle import hcub_oracle as orc
    d = 13
    rng = np.random.default_rng(13)
    lo = rng.random((64, d)) * 0.5
    hi = lo + 0.05 + rng.random((64, d)) * 0.4
    I, E, S, ev = hb.apply_rule_batch(hb.build_gm_rule(d), lo, hi, hb.make_integrand("f2", d))
    oI, oE, oS, oev = orc.eval_regions(orc.gm_table(d), lo, hi, orc.integrand("f2", d))
    assert ev == oev
    assert np.array_equal(S, oS) and np.array_equal(np.argmax(S, axis=1), np.argmax(oS, axis=1))
    assert np.all(np.abs(I - oI) <= 1e-12 * np.abs(oI))


def test_one_iteration_and_bad_configs():
    import paper_2511_01573_b200 as hb
    f = hb.make_integrand("f4", 3)
    r = hb.integrate(f, hb.HyperRect.unit_cube(3), hb.DriverConfig(1e-6, max_iterations=1))
    assert r.iterations == 1 and r.termination_reason == hb.TerminationReason.MAX_ITERATIONS
    assert r.total_f_evals == 6 * 33 and not r.converged
    with pytest.raises(ValueError):
        hb.DriverConfig(-1.0)
    with pytest.raises(TypeError):  # no CPU fallback for arbitrary callables
        hb.integrate(lambda x: x[:, 0], hb.HyperRect.unit_cube(3), hb.DriverConfig(1e-6))


def test_ragged_domain_and_odd_partition():
    """Non-cube domain with a partition count that is not a power of two
    (greedy bisection ties, ref regions.py:92-111): same counts and estimates
    as the oracle for a few iterations."""
    import paper_2511_01573_b200 as hb
    from oracle import hcub_oracle as orc
    lo, hi = np.array([-1.5, 0.25, 2.0, 0.0]), np.array([0.5, 0.75, 5.0, 0.125])
    f = hb.make_product_peak(4, center=[-0.2, 0.5, 3.1, 0.05], sharpness=20.0)[0]
    tr = []
    r = hb.integrate(f, hb.HyperRect(lo, hi), hb.DriverConfig(1e-7, max_iterations=9), trace=tr.append,
                     initial_regions=11)
    o = orc.integrate(orc.product_peak(4, [-0.2, 0.5, 3.1, 0.05], 20.0), 4, 1e-7, lo, hi, init=11, max_iterations=9)
    assert [t.active_regions for t in tr] == [t[1] for t in o.trace]
    for a, b in zip(tr, o.trace):
        assert math.isclose(a.integral, b[2], rel_tol=1e-12) and math.isclose(a.error, b[3], rel_tol=1e-9)
