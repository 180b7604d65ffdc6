"""Degree-9 fully symmetric rule with an embedded degree-7 rule, as a
loadable table for `parse_rule_table` (the paper's "9-order"
rule, ref PAPER.md:59, table format ref
pkg/src/hcub/rules.py:377-405).

Node structure and generators: the degree-9 rule of DCUHRE (Berntsen,
Espelid & Genz, ACM TOMS 17 (1991) 437-451, Algorithm 698, subroutine
D09HRE), the Genz-Berntsen fully symmetric family the paper cites.  In the
squared-generator variables lam = g^2:

    lam0 = 0.4707
    lam1 = 4 / (15 - 5/lam0)
    r    = (1 - lam1/lam0) / 27
    lam2 = (5 - 7 lam1 - 35 r) / (7 - 35 lam1/3 - 35 r/lam0)
    r    = r (1 - lam2/lam0) / 3
    lam3 = (7 - 9 (lam2 + lam1) + 63 lam2 lam1/5 - 63 r)
           / (9 - 63 (lam2 + lam1)/5 + 21 lam2 lam1 - 63 r/lam0)

orbits (generator magnitudes on [-1, 1]^d):
    center; (g0), (g1), (g2), (g3) on the axes; (g1, g1), (g1, g2);
    (g1, g1, g1) for d >= 3; (g0, ..., g0) at the 2^d corners
node count 1 + 8d + 6d(d-1) + 4d(d-1)(d-2)/3 + 2^d (d=5: 273, d=8: 1105).

The generators are restated from that algorithm (no network here to re-check
the printed source), so nothing below is trusted on that basis: every lam is
an exact rational function of lam0 = 4707/10000, and the weights are the
UNIQUE exact rational solution of the fully symmetric moment equations
sum_nodes w * x^(2 alpha) = 2^d prod_j 1/(2 alpha_j + 1) for every even
monomial of degree <= 9 (12 pattern equations, 9 weights: the system is
over-determined and is consistent only because of the lam relations above -
its zero residual is the proof that the node set supports a degree-9 rule).
The embedded degree-7 rule is the unique solution of the degree-7 equations
on the same nodes without the (g0) / (g3) axis orbits and the 3-nonzero
orbit.  Weights follow the reference convention (x 2^d, rules.py:270-281).
tests/test_rule9.py re-derives the exactness numerically from the parsed
table (monomials of degree <= 9 / <= 7, d = 2..8).

As in the GM rule the lam0 axis orbit carries zero weight in both rules; it
exists for error estimation: the reference's axis bookkeeping
(rules.py:206-250) takes the two smallest on-axis magnitudes, here g2
(lam_in) and g0 (lam_out), for the fourth-difference scores and the degree-3
companion of the error cascade.
"""
from __future__ import annotations

import math
from fractions import Fraction
from functools import lru_cache
from collections import Counter

from .rules import RuleTable, UnsupportedDimensionError, parse_rule_table

__all__ = ["gm9_lambdas", "gm9_weights", "gm9_rule_text", "build_gm9_rule"]


def gm9_lambdas() -> tuple[Fraction, Fraction, Fraction, Fraction]:
    """(lam0, lam1, lam2, lam3) = squared generators, exact rationals."""
    l0 = Fraction(4707, 10000)
    l1 = 4 / (15 - 5 / l0)
    r = (1 - l1 / l0) / 27
    l2 = (5 - 7 * l1 - 35 * r) / (7 - Fraction(35, 3) * l1 - 35 * r / l0)
    r = r * (1 - l2 / l0) / 3
    l3 = (7 - 9 * (l2 + l1) + Fraction(63, 5) * l2 * l1 - 63 * r) / (
        9 - Fraction(63, 5) * (l2 + l1) + 21 * l2 * l1 - 63 * r / l0)
    return l0, l1, l2, l3


def _orbits(d: int):
    l0, l1, l2, l3 = gm9_lambdas()

    def g(*v):
        return tuple(list(v) + [Fraction(0)] * (d - len(v)))

    orb = [("center", g()), ("axis0", g(l0)), ("axis1", g(l1)), ("axis2", g(l2)), ("axis3", g(l3)),
           ("pair11", g(l1, l1)), ("pair12", g(l1, l2))]
    if d >= 3:
        orb.append(("triple111", g(l1, l1, l1)))
    orb.append(("corner0", tuple([l0] * d)))
    return orb


def _patterns(degree: int, d: int):
    """Even monomials x^(2 alpha) up to `degree`, one per symmetry class
    (alpha non-increasing, at most d parts)."""
    out = []

    def rec(cur, rem, mx):
        out.append(tuple(cur))
        if len(cur) == d:
            return
        for k in range(min(rem, mx), 0, -1):
            rec(cur + [k], rem - k, k)

    rec([], degree // 2, degree // 2)
    return out


def _orbit_moment(lams, alpha) -> Fraction:
    """sum over the orbit's nodes of prod_j x_j^(2 alpha_j): sign flips give
    2^nnz identical terms; the distinct permutations are counted by
    assigning values to the len(alpha) constrained coordinates and
    multiplying by the number of distinct arrangements of the rest."""
    counts = Counter(lams)
    nnz = sum(1 for v in lams if v != 0)

    def arrangements(cnt) -> int:
        n = sum(cnt.values())
        out = math.factorial(n)
        for c in cnt.values():
            out //= math.factorial(c)
        return out

    def rec(j, cnt) -> Fraction:
        if j == len(alpha):
            return Fraction(arrangements(cnt))
        s = Fraction(0)
        for v in list(cnt):
            if cnt[v] == 0:
                continue
            cnt[v] -= 1
            s += v ** alpha[j] * rec(j + 1, cnt)
            cnt[v] += 1
        return s

    return 2 ** nnz * rec(0, counts)


def _solve_exact(A, b):
    """Exact least squares over the rationals (normal equations, Gauss-Jordan);
    returns (x, max residual)."""
    n = len(A[0])
    M = [[sum(A[k][i] * A[k][j] for k in range(len(A))) for j in range(n)]
         + [sum(A[k][i] * b[k] for k in range(len(A)))] for i in range(n)]
    for c in range(n):
        p = next((r for r in range(c, n) if M[r][c] != 0), None)
        if p is None:
            raise ArithmeticError("moment system is singular")
        M[c], M[p] = M[p], M[c]
        for r in range(n):
            if r != c and M[r][c] != 0:
                f = M[r][c] / M[c][c]
                M[r] = [x - f * y for x, y in zip(M[r], M[c])]
    x = [M[i][n] / M[i][i] for i in range(n)]
    res = max(abs(sum(A[k][i] * x[i] for i in range(n)) - b[k]) for k in range(len(A)))
    return x, res


def _rule_weights(d: int, degree: int, use) -> dict[str, Fraction]:
    orb = [o for o in _orbits(d) if o[0] in use]
    pats = _patterns(degree, d)
    A = [[_orbit_moment(g, al) for _, g in orb] for al in pats]
    b = [Fraction(2 ** d) * math.prod(Fraction(1, 2 * a + 1) for a in al) for al in pats]
    x, res = _solve_exact(A, b)
    if res != 0:
        raise ArithmeticError(f"degree-{degree} moment equations inconsistent at d={d} (residual {float(res)})")
    return dict(zip((n for n, _ in orb), x))


@lru_cache(maxsize=None)
def gm9_weights(d: int):
    """[(orbit name, squared generator, main weight, embedded weight)] with
    exact rational weights (x 2^d convention)."""
    if not 2 <= d <= 13:
        raise UnsupportedDimensionError(f"degree-9 table defined for 2 <= d <= 13, got {d}")
    orb = _orbits(d)
    names = [n for n, _ in orb]
    w9 = _rule_weights(d, 9, names)
    w7 = _rule_weights(d, 7, [n for n in names if n not in ("axis0", "axis3", "triple111")])
    return [(n, g, w9[n], w7.get(n, Fraction(0))) for n, g in orb]


def gm9_rule_text(d: int) -> str:
    """The rule in the reference's plain-text table format (one orbit per
    line: d generator magnitudes, weight, embedded weight)."""
    lines = [f"# degree-9 fully symmetric rule (DCUHRE D09HRE node set), embedded degree 7, d={d}"]
    for name, g, w, we in gm9_weights(d):
        coords = [repr(math.sqrt(v)) if v else "0.0" for v in (float(x) for x in g)]
        lines.append(" ".join(coords + [repr(float(w)), repr(float(we))]) + f"  # {name}")
    return "\n".join(lines) + "\n"


@lru_cache(maxsize=None)
def build_gm9_rule(d: int) -> RuleTable:
    """The degree-9 table parsed through `parse_rule_table` (so it carries
    exactly the bookkeeping the reference derives for a loaded table)."""
    t = parse_rule_table(gm9_rule_text(d), name="gm9", degree=9, embedded_degree=7)
    t.family = "gm9"  # the device evaluates it in generator form (csrc/k1_gm9.cuh), not as a node table
    return t
