"""Cubature rule tables and batched rule application on the B200.

Rule construction is host metadata (ref pkg/src/hcub/rules.py:71-282): the
Genz-Malik degree-7/5 rule is carried in generator form (four lambdas and
five weight pairs) and handed to the device, which generates every node on
the fly.  The expanded node table (`RuleTable.points`) is materialised only
on request for API compatibility - no kernel reads it.

`apply_rule_batch` (ref rules.py:459-536) runs kernel K1 (`k1_gm_eval`) via
the C ABI; there is no host evaluation path.
"""

from __future__ import annotations

import ctypes as C
import functools
import math
import threading
from dataclasses import dataclass, field
from pathlib import Path
from typing import Sequence

import numpy as np

from . import _lib
from .regions import HyperRect

__all__ = [
    "UnsupportedDimensionError", "Orbit", "RuleTable", "RuleEvaluation", "build_gm_rule", "build_gk_tensor_rule",
    "get_rule", "load_rule_table", "parse_rule_table", "expand_orbit", "apply_rule", "apply_rule_batch",
    "select_axis", "NONFINITE_ERROR_SCALE",
]

GM_MIN_DIM, GM_MAX_DIM, GK_MAX_DIM = 2, 13, 6
NONFINITE_ERROR_SCALE = 1e30
_DESCRIPTOR_LOCK = threading.Lock()
GM9_GENERATOR_MAX_D = 10  # csrc/k1_gm9.cuh instantiations (larger d: the node-table kernel)


class UnsupportedDimensionError(ValueError):
    """Requested rule does not exist for this dimension (ref rules.py:67-68)."""


@dataclass(frozen=True)
class Orbit:
    generator: tuple
    weight: float
    embedded_weight: float
    size: int


@dataclass
class RuleEvaluation:
    integral: float
    error: float
    axis_scores: np.ndarray
    f_evals: int


def _orbit_size(gen) -> int:
    mags = [abs(float(g)) for g in gen]
    n = math.factorial(len(mags))
    for v in set(mags):
        n //= math.factorial(mags.count(v))
    return n * 2 ** sum(1 for m in mags if m != 0.0)


def expand_orbit(generator: Sequence[float]) -> np.ndarray:
    """Distinct permutations (lexicographic) x sign flips of the nonzero
    entries in binary order, all-plus first (ref rules.py:154-175)."""
    gen = [float(g) for g in generator]
    if not gen:
        raise ValueError("generator must be a 1-D point")
    if any(g < 0 for g in gen):
        raise ValueError("generator coordinates must be non-negative magnitudes")
    keys = sorted(set(gen))
    left = {k: gen.count(k) for k in keys}
    rows = []
    cur: list[float] = []

    def walk():
        if len(cur) == len(gen):
            nz = [i for i, v in enumerate(cur) if v != 0.0]
            for mask in range(1 << len(nz)):
                p = list(cur)
                for b, i in enumerate(nz):
                    if mask >> b & 1:
                        p[i] = -p[i]
                rows.append(p)
            return
        for k in keys:
            if left[k]:
                left[k] -= 1
                cur.append(k)
                walk()
                cur.pop()
                left[k] += 1

    walk()
    return np.asarray(rows, dtype=np.float64).reshape(len(rows), len(gen))


@dataclass
class RuleTable:
    """Rule metadata.  For the GM family the generator data in `orbits` plus
    the axis bookkeeping is all the device needs; `points`/`weights` expand
    lazily."""

    d: int
    name: str
    kind: str
    node_count: int
    degree: int
    embedded_degree: int
    orbits: list = field(default_factory=list)
    fourth_diff_ratio: float | None = None
    null_center_weight: float | None = None
    null_axis_weight: float | None = None
    lambdas: tuple | None = None  # (lam2, lam3, lam4, lam5) for the GM family
    family: str | None = None     # "gm9": the rule9.py degree-9 table (evaluated in generator form)

    @property
    def has_null_cascade(self) -> bool:
        return self.null_center_weight is not None

    @functools.cached_property
    def points(self) -> np.ndarray:
        return np.vstack([expand_orbit(o.generator) for o in self.orbits])

    @functools.cached_property
    def weights(self) -> np.ndarray:
        return np.concatenate([np.full(o.size, o.weight) for o in self.orbits])

    @functools.cached_property
    def embedded_weights(self) -> np.ndarray:
        return np.concatenate([np.full(o.size, o.embedded_weight) for o in self.orbits])

    def _table_descriptor(self) -> _lib.hcub_rule:
        """Explicit node table for custom fully symmetric rules (device kernel
        k1_table_eval); arrays are kept alive on the table object."""
        if not 1 <= self.d <= _lib.MAX_DIM:
            raise UnsupportedDimensionError(f"rule tables support 1 <= d <= {_lib.MAX_DIM}, got {self.d}")
        # the host arrays the descriptor points into are built once per table and
        # kept on it: worker threads creating stores concurrently (the concurrent
        # backend) must never see an earlier descriptor's arrays freed under them
        keep = self.__dict__.get("_keep")
        if keep is None:
            with _DESCRIPTOR_LOCK:
                keep = self.__dict__.get("_keep")
                if keep is None:
                    pts = np.ascontiguousarray(self.points, dtype=np.float64)
                    keep = (pts, np.ascontiguousarray(self.weights, dtype=np.float64),
                            np.ascontiguousarray(self.embedded_weights, dtype=np.float64),
                            _axis_bookkeeping(pts, self.orbits, self.d))
                    self._keep = keep
        pts, w, we, book = keep
        r = _lib.hcub_rule()
        r.d = self.d
        r.node_count = self.node_count
        # 3: k1_gm9_eval, the generator form of this very table (compiled for d <= 8)
        r.kind = 3 if self.family == "gm9" and self.d <= GM9_GENERATOR_MAX_D else 1
        r.K = pts.shape[0]
        r.points, r.weights, r.embedded_weights = _lib.dptr(pts), _lib.dptr(w), _lib.dptr(we)
        if book:
            r.has_axis_pairs = 1
            r.center_index = book["center"]
            for k in range(self.d):
                for q in range(4):
                    r.axis_pairs[k][q] = int(book["pairs"][k, q])
            r.fourth_diff_ratio = book["ratio"]
            r.null_center_weight = book["null_center"]
            r.null_axis_weight = book["null_axis"]
        else:
            r.center_index = -1
        return r

    def descriptor(self) -> _lib.hcub_rule:
        if self.kind == "symmetric" and self.lambdas is None:
            return self._table_descriptor()
        if self.kind == "tensor_gk":  # k1_gk_partial / k1_gk_finalize
            r = _lib.hcub_rule()
            r.d = self.d
            r.node_count = self.node_count
            r.kind = 2
            return r
        if self.kind != "symmetric" or self.name != "gm":
            raise NotImplementedError(f"rule {self.name!r} ({self.kind}) has no B200 kernel")
        r = _lib.hcub_rule()
        r.d = self.d
        r.node_count = self.node_count
        r.lam2, r.lam3, r.lam4, r.lam5 = self.lambdas
        for i, o in enumerate(self.orbits):
            r.w[i] = o.weight
            r.we[i] = o.embedded_weight
        r.fourth_diff_ratio = self.fourth_diff_ratio
        r.null_center_weight = self.null_center_weight
        r.null_axis_weight = self.null_axis_weight
        return r


def _axis_bookkeeping(points: np.ndarray, orbits, d: int) -> dict:
    """Center node, per-axis inner/outer on-axis node pairs and the degree-3
    companion weights, as ref rules.py:206-250 derives them (empty if the
    table lacks the structure)."""
    center = np.flatnonzero((points == 0.0).all(axis=1))
    if center.size != 1:
        return {}
    lambdas = sorted({float(max(abs(g) for g in o.generator)) for o in orbits
                      if sum(1 for g in o.generator if g != 0.0) == 1})
    if len(lambdas) < 2:
        return {}
    lam_in, lam_out = lambdas[0], lambdas[1]
    pairs = np.zeros((d, 4), dtype=np.int32)
    for ax in range(d):
        rest = np.delete(points, ax, axis=1)
        for j, lam in enumerate((lam_in, lam_out)):
            hit = np.flatnonzero((np.abs(np.abs(points[:, ax]) - lam) < 1e-14) & (rest == 0.0).all(axis=1))
            plus, minus = hit[points[hit, ax] > 0], hit[points[hit, ax] < 0]
            if plus.size != 1 or minus.size != 1:
                return {}
            pairs[ax, 2 * j], pairs[ax, 2 * j + 1] = plus[0], minus[0]
    w_axis = 2.0 ** d / (6.0 * lam_out ** 2)
    return dict(center=int(center[0]), pairs=pairs, ratio=(lam_in / lam_out) ** 2,
                null_center=2.0 ** d - 2 * d * w_axis, null_axis=w_axis)


@functools.lru_cache(maxsize=None)
def build_gm_rule(d: int) -> RuleTable:
    """Genz-Malik degree 7 with embedded degree 5, 2 <= d <= 13
    (ref rules.py:257-282; constants as in the reference)."""
    if not GM_MIN_DIM <= d <= GM_MAX_DIM:
        raise UnsupportedDimensionError(
            f"fully symmetric rule supports {GM_MIN_DIM} <= d <= {GM_MAX_DIM}, got {d}")
    lam2 = math.sqrt(9.0 / 70.0)
    lam3 = math.sqrt(9.0 / 10.0)
    lam4 = lam3
    lam5 = math.sqrt(9.0 / 19.0)
    t = 2.0 ** d
    zeros = (0.0,) * d
    gens = [
        (zeros, t * (12824 - 9120 * d + 400 * d * d) / 19683.0, t * (729 - 950 * d + 50 * d * d) / 729.0),
        ((lam2,) + zeros[1:], t * 980 / 6561.0, t * 245 / 486.0),
        ((lam3,) + zeros[1:], t * (1820 - 400 * d) / 19683.0, t * (265 - 100 * d) / 1458.0),
        ((lam4, lam4) + zeros[2:], t * 200 / 19683.0, t * 25 / 729.0),
        ((lam5,) * d, 6859 / 19683.0, 0.0),
    ]
    orbits = [Orbit(tuple(g), w, we, _orbit_size(g)) for g, w, we in gens]
    # axis bookkeeping (ref rules.py:206-250): inner/outer on-axis magnitudes
    lam_in, lam_out = lam2, lam3
    w_axis = t / (6.0 * lam_out ** 2)
    return RuleTable(
        d=d, name="gm", kind="symmetric", node_count=sum(o.size for o in orbits), degree=7, embedded_degree=5,
        orbits=orbits, fourth_diff_ratio=(lam_in / lam_out) ** 2, null_center_weight=t - 2 * d * w_axis,
        null_axis_weight=w_axis, lambdas=(lam2, lam3, lam4, lam5))


@functools.lru_cache(maxsize=None)
def build_gk_tensor_rule(d: int) -> RuleTable:
    """Tensor G7/K15 rule, 15^d nodes, d <= 6 (ref rules.py:332-357); the
    device decodes nodes from their index (kernels in csrc/k1_gk.cuh)."""
    if d < 1:
        raise UnsupportedDimensionError("dimension must be at least 1")
    if d > GK_MAX_DIM:
        raise UnsupportedDimensionError(
            f"tensor Gauss-Kronrod rule is capped at d <= {GK_MAX_DIM} "
            f"(15^d nodes are impractical beyond that), got {d}")
    return RuleTable(d=d, name="gk-tensor", kind="tensor_gk", node_count=15 ** d, degree=22, embedded_degree=13)


def get_rule(name, d: int) -> RuleTable:
    """ref rules.py:360-370.  B200 extra: a RuleTable (e.g. from
    parse_rule_table) is accepted as-is, so DriverConfig(rule=table) runs a
    custom family through integrate / run_distributed."""
    if isinstance(name, RuleTable):
        if name.d != d:
            raise UnsupportedDimensionError(f"table is for d={name.d}, problem has d={d}")
        return name
    if name == "gm":
        return build_gk_tensor_rule(1) if d == 1 else build_gm_rule(d)
    if name in ("gk-tensor", "gk_tensor", "gk"):
        return build_gk_tensor_rule(d)
    if name == "gm9":  # B200 extra: the degree-9 table of rule9.py through parse_rule_table
        from .rule9 import build_gm9_rule
        return build_gm9_rule(d)
    raise ValueError(f"unknown rule {name!r}; expected 'gm' or 'gk-tensor'")


def parse_rule_table(text: str, name: str = "custom", degree: int = -1, embedded_degree: int = -1) -> RuleTable:
    """Plain-text orbit table (ref rules.py:377-400): one orbit per line,
    ``g_1..g_d weight embedded_weight``; '#' comments, commas tolerated."""
    rows = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip().replace(",", " ")
        if not line:
            continue
        try:
            rows.append([float(tok) for tok in line.split()])
        except ValueError as exc:
            raise ValueError(f"line {lineno}: {exc}") from exc
    if not rows:
        raise ValueError("no orbits found in rule table text")
    width = len(rows[0])
    if width < 3 or any(len(r) != width for r in rows):
        raise ValueError("every orbit line needs d coordinates plus two weights")
    d = width - 2
    orbits = [Orbit(tuple(r[:d]), r[d], r[d + 1], _orbit_size(r[:d])) for r in rows]
    return RuleTable(d=d, name=name, kind="symmetric", node_count=sum(o.size for o in orbits), degree=degree,
                     embedded_degree=embedded_degree, orbits=orbits)


def load_rule_table(path, name=None) -> RuleTable:
    path = Path(path)
    return parse_rule_table(path.read_text(), name=name or path.stem)


def _rows(a, d=None):
    a = np.ascontiguousarray(np.atleast_2d(np.asarray(a, dtype=np.float64)))
    return a


def apply_rule_batch(table: RuleTable, lo, hi, f):
    """Per-region integrals, errors, (n, d) axis scores and the evaluation
    count (ref rules.py:459-536), computed by K1 on the device."""
    from .integrands import device_descriptor

    lo = _rows(lo)
    hi = _rows(hi)
    n, d = lo.shape
    if hi.shape != lo.shape:
        raise ValueError("lo/hi shape mismatch")
    if d != table.d:
        raise UnsupportedDimensionError(f"table is for d={table.d}, regions have d={d}")
    rd = table.descriptor()
    fd = device_descriptor(f, d)
    integral = np.empty(n)
    error = np.empty(n)
    scores = np.empty((n, d))
    axis = np.empty(n, dtype=np.int64)
    ev = C.c_int64(0)
    _lib.check(_lib.lib().hcub_apply_rule_batch(
        _lib.current_device(), C.byref(rd), C.byref(fd), _lib.dptr(lo), _lib.dptr(hi), n,
        _lib.dptr(integral), _lib.dptr(error), _lib.dptr(scores), _lib.iptr(axis), C.byref(ev)))
    return integral, error, scores, int(ev.value)


def apply_rule_batch_axes(table: RuleTable, lo, hi, f):
    """apply_rule_batch plus the device-chosen split axes (argmax of scores)."""
    from .integrands import device_descriptor

    lo = _rows(lo)
    hi = _rows(hi)
    n, d = lo.shape
    rd = table.descriptor()
    fd = device_descriptor(f, d)
    integral = np.empty(n)
    error = np.empty(n)
    scores = np.empty((n, d))
    axis = np.empty(n, dtype=np.int64)
    ev = C.c_int64(0)
    _lib.check(_lib.lib().hcub_apply_rule_batch(
        _lib.current_device(), C.byref(rd), C.byref(fd), _lib.dptr(lo), _lib.dptr(hi), n,
        _lib.dptr(integral), _lib.dptr(error), _lib.dptr(scores), _lib.iptr(axis), C.byref(ev)))
    return integral, error, scores, axis, int(ev.value)


def apply_rule(table: RuleTable, rect: HyperRect, f) -> RuleEvaluation:
    integral, error, scores, evals = apply_rule_batch(table, rect.lo[None, :], rect.hi[None, :], f)
    return RuleEvaluation(float(integral[0]), float(error[0]), scores[0], evals)


def select_axis(evaluation: RuleEvaluation) -> int:
    """Largest fourth-difference score, lowest axis on ties (ref rules.py:454-456)."""
    return int(np.argmax(evaluation.axis_scores))
