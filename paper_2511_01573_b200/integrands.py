"""Genz benchmark integrands as device functors (ref pkg/src/hcub/integrands.py).

The device cannot call back into Python per node, so an integrand is
identified by its kind and constants and evaluated inside the kernels
(`Fn<FN,D>` in csrc/hcub_device.cuh).  `BenchmarkIntegrand.__call__` and
`ProductPeak.__call__` evaluate on the GPU too.  Exact reference values are
host-side closed forms / exact rationals, computed as the reference does
(ref integrands.py:102-178).
"""

from __future__ import annotations

import cmath
import ctypes as C
import functools
import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _lib

__all__ = ["FUNCTION_IDS", "BenchmarkIntegrand", "ProductPeak", "make_integrand", "reference_integral",
           "make_product_peak", "device_descriptor"]

FUNCTION_IDS = ("f1", "f2", "f3", "f4", "f5", "f6", "f7")


def _eval_on_device(desc: _lib.hcub_integrand, d: int, pts) -> np.ndarray:
    pts = np.ascontiguousarray(np.atleast_2d(np.asarray(pts, dtype=np.float64)))
    if pts.shape[1] != d:
        raise ValueError(f"points must be (m, {d})")
    out = np.empty(pts.shape[0])
    _lib.check(_lib.lib().hcub_eval_points(_lib.current_device(), C.byref(desc), _lib.dptr(pts), pts.shape[0],
                                           _lib.dptr(out)))
    return out


@dataclass(frozen=True)
class BenchmarkIntegrand:
    """One Genz function at a fixed dimension (ref integrands.py:35-46)."""

    id: str
    d: int
    reference_value: float
    reference_provenance: str

    def descriptor(self) -> _lib.hcub_integrand:
        f = _lib.hcub_integrand()
        f.kind = _lib.KIND[self.id]
        f.d = self.d
        f.a = 50.0 ** -2
        return f

    def evaluate(self, pts) -> np.ndarray:
        return _eval_on_device(self.descriptor(), self.d, pts)

    def __call__(self, pts) -> np.ndarray:
        return self.evaluate(pts)


class ProductPeak:
    """Movable product peak prod_j 1/(a + (x_j - c_j)^2), a = 1/sharpness^2
    (ref integrands.py:194-210)."""

    def __init__(self, d: int, center, sharpness: float):
        if not 1 <= d <= _lib.MAX_DIM:
            raise ValueError(f"product peak supports 1 <= d <= {_lib.MAX_DIM}")
        self.d = d
        self.center = np.broadcast_to(np.asarray(center, dtype=np.float64), (d,)).copy()
        self.sharpness = float(sharpness)
        self.a = 1.0 / self.sharpness ** 2

    def descriptor(self) -> _lib.hcub_integrand:
        f = _lib.hcub_integrand()
        f.kind = _lib.KIND["product_peak"]
        f.d = self.d
        f.a = self.a
        for j, c in enumerate(self.center):
            f.center[j] = float(c)
        return f

    def __call__(self, pts) -> np.ndarray:
        return _eval_on_device(self.descriptor(), self.d, pts)

    def __repr__(self):
        return f"ProductPeak(d={self.d}, center={self.center.tolist()}, sharpness={self.sharpness})"


def device_descriptor(f, d: int) -> _lib.hcub_integrand:
    """Device functor descriptor for ``f``; anything the device cannot
    identify is rejected (no CPU fallback)."""
    if isinstance(f, (BenchmarkIntegrand, ProductPeak)):
        if f.d != d:
            raise ValueError(f"integrand is for d={f.d}, regions have d={d}")
        return f.descriptor()
    raise TypeError(
        "the B200 path evaluates integrands on the device and accepts only BenchmarkIntegrand "
        "(make_integrand) or ProductPeak (make_product_peak) objects; arbitrary Python callables "
        f"cannot run inside the kernels (got {type(f).__name__})")


# ---------------------------------------------------------------------------
# exact values (host, ref integrands.py:102-178)


def _f1_exact(d):
    z = complex(1.0, 0.0)
    for i in range(1, d + 1):
        z *= (cmath.exp(1j * i) - 1.0) / (1j * i)
    return z.real


def _f3_exact(d):
    acc = Fraction(0)
    for mask in range(1 << d):
        s = sum(i + 1 for i in range(d) if mask >> i & 1)
        acc += Fraction((-1) ** bin(mask).count("1"), 1 + s)
    return float(acc / Fraction(math.factorial(d)) ** 2)


def _f7_exact(d):
    # sum over exponent partitions of 11 into at most d parts
    def parts(n, cap, slots):
        if n == 0:
            yield ()
            return
        if slots == 0:
            return
        for p in range(min(n, cap), 0, -1):
            for rest in parts(n - p, p, slots - 1):
                yield (p,) + rest

    total = Fraction(0)
    for part in parts(11, 11, d):
        ks = list(part) + [0] * (d - len(part))
        coef = Fraction(math.factorial(11))
        for k in ks:
            coef /= math.factorial(k) * (2 * k + 1)
        mult = Fraction(math.factorial(d))
        for v in set(ks):
            mult /= math.factorial(ks.count(v))
        total += coef * mult
    return float(total)


@functools.lru_cache(maxsize=None)
def reference_integral(id: str, d: int) -> tuple[float, str]:
    if id not in FUNCTION_IDS:
        raise ValueError(f"unknown integrand {id!r}")
    if d < 1:
        raise ValueError("dimension must be at least 1")
    if id == "f1":
        return _f1_exact(d), "closed_form"
    if id == "f2":
        return (100.0 * math.atan(25.0)) ** d, "closed_form"
    if id == "f3":
        # "oracle" is the reference's provenance label for exact-rational values
        # (ref integrands.py:43, 167) - not the repo's test oracle/
        return _f3_exact(d), "oracle"
    if id == "f4":
        return (math.sqrt(math.pi) / 25.0 * math.erf(12.5)) ** d, "closed_form"
    if id == "f5":
        return ((1.0 - math.exp(-5.0)) / 5.0) ** d, "closed_form"
    if id == "f6":
        v = 1.0
        for i in range(1, d + 1):
            t = min(1.0, (3.0 + i) / 10.0)
            v *= (math.exp((i + 4.0) * t) - 1.0) / (i + 4.0)
        return v, "closed_form"
    return _f7_exact(d), "oracle"


@functools.lru_cache(maxsize=None)
def make_integrand(id: str, d: int) -> BenchmarkIntegrand:
    value, prov = reference_integral(id, d)
    if d > _lib.MAX_DIM:
        raise ValueError(f"device integrands support d <= {_lib.MAX_DIM}")
    return BenchmarkIntegrand(id=id, d=d, reference_value=value, reference_provenance=prov)


def make_product_peak(d: int, center=0.5, sharpness: float = 50.0):
    """(evaluator, exact integral over [0,1]^d) (ref integrands.py:194-210)."""
    f = ProductPeak(d, center, sharpness)
    exact = 1.0
    for c in f.center:
        exact *= sharpness * (math.atan(sharpness * (1.0 - c)) - math.atan(sharpness * (0.0 - c)))
    return f, exact
