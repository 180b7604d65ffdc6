"""Single-worker batch adaptive integration on one B200 (ref pkg/src/hcub/driver.py).

`integrate` hands the whole loop to the device (`hcub_integrate`): the
region store stays in HBM, each iteration runs K1 (rule evaluation) -> K2
(exact global sums) -> K3 (classify / finalize / split / compact), and only
the per-iteration trace scalars cross PCIe (one 128-byte read per
iteration).  Termination logic and results mirror ref driver.py:237-323.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import Enum
from typing import Callable

import numpy as np

from . import _lib
from .regions import HyperRect, partition_arrays

__all__ = ["TerminationReason", "DriverConfig", "VolumeBudgetClassifier", "GlobalEstimate", "IntegrationResult",
           "IterationTrace", "check_convergence", "integrate", "exact_sum"]


def exact_sum(values) -> float:
    """math.fsum of ``values`` (ref driver.py:43-45); host utility."""
    return math.fsum(np.asarray(values, dtype=np.float64).tolist())


def device_exact_sum(values, carry: float = 0.0) -> float:
    """fsum([carry, *values]) computed by the device superaccumulator that
    K2/K3 use (exactly rounded, so equal to math.fsum bit for bit)."""
    x = np.ascontiguousarray(np.asarray(values, dtype=np.float64).ravel())
    out = C.c_double(0.0)
    _lib.check(_lib.lib().hcub_exact_sum(_lib.current_device(), _lib.dptr(x), x.size, float(carry), C.byref(out)))
    return out.value


class TerminationReason(str, Enum):
    TOLERANCE = "tolerance"
    MAX_ITERATIONS = "max_iterations"
    MAX_REGIONS = "max_regions"
    WIDTH_GUARD_EXHAUSTED = "width_guard_exhausted"


_REASON = [TerminationReason.TOLERANCE, TerminationReason.MAX_ITERATIONS, TerminationReason.MAX_REGIONS,
           TerminationReason.WIDTH_GUARD_EXHAUSTED]


@dataclass(frozen=True)
class VolumeBudgetClassifier:
    """A region is negligible once error <= max(floor, |I| tau) * safety *
    vol/vol_domain (ref driver.py:60-76); evaluated inside K3 on the device."""

    safety: float = 0.5

    def thresholds(self, estimate, cfg, volumes, domain_volume):
        budget = max(cfg.abs_floor, abs(estimate.integral) * cfg.tau_rel)
        return budget * self.safety * (np.asarray(volumes) / domain_volume)


@dataclass(frozen=True)
class DriverConfig:
    """ref driver.py:79-102."""

    tau_rel: float
    abs_floor: float = 1e-16
    max_iterations: int = 1000
    max_regions: int = 1 << 24
    min_width_ulp_factor: float = 8.0
    rule: str = "gm"
    classifier: VolumeBudgetClassifier = field(default_factory=VolumeBudgetClassifier)

    def __post_init__(self):
        if not self.tau_rel > 0:
            raise ValueError("tau_rel must be positive")
        if self.max_regions < 1 or self.max_iterations < 1:
            raise ValueError("max_regions and max_iterations must be >= 1")

    def descriptor(self) -> _lib.hcub_driver_cfg:
        if type(self.classifier) is not VolumeBudgetClassifier:
            raise TypeError("the device classifier implements VolumeBudgetClassifier(safety) only")
        c = _lib.hcub_driver_cfg()
        c.tau_rel = self.tau_rel
        c.abs_floor = self.abs_floor
        c.min_width_ulp_factor = self.min_width_ulp_factor
        c.safety = self.classifier.safety
        c.max_iterations = int(self.max_iterations)
        c.max_regions = int(min(self.max_regions, (1 << 62)))
        return c


@dataclass
class GlobalEstimate:
    integral: float
    error: float
    finalized_integral: float
    finalized_error: float
    active_regions: int


@dataclass
class IntegrationResult:
    integral: float
    error: float
    converged: bool
    iterations: int
    total_f_evals: int
    peak_regions: int
    termination_reason: TerminationReason


@dataclass(frozen=True)
class IterationTrace:
    iteration: int
    active_regions: int
    integral: float
    error: float
    f_evals: int


def check_convergence(estimate: GlobalEstimate, cfg: DriverConfig) -> bool:
    return estimate.error <= max(cfg.abs_floor, abs(estimate.integral) * cfg.tau_rel)


def integrate(f, domain: HyperRect, cfg: DriverConfig, trace: Callable[[IterationTrace], None] | None = None,
              initial_regions: int | None = None, *, capacity: int = 0, stats: dict | None = None
              ) -> IntegrationResult:
    """Adaptive integration of ``f`` over ``domain`` on the current device
    (ref driver.py:237-323).  ``capacity`` (regions per store buffer, 0 =
    from cfg.max_regions and free HBM) and ``stats`` (filled with device
    timings) are B200 extras."""
    from .integrands import device_descriptor
    from .rules import get_rule

    d = domain.dim
    table = get_rule(cfg.rule, d)
    rd = table.descriptor()
    fd = device_descriptor(f, d)
    k = initial_regions if initial_regions is not None else 2 * d
    lo0, hi0 = partition_arrays(domain, k)
    dlo = np.ascontiguousarray(domain.lo, dtype=np.float64)
    dhi = np.ascontiguousarray(domain.hi, dtype=np.float64)
    cd = cfg.descriptor()
    res = _lib.hcub_result()
    err_box = []

    def _cb(user, it, n, I, E, ev):
        try:
            trace(IterationTrace(int(it), int(n), float(I), float(E), int(ev)))
            return 0
        except BaseException as exc:  # stop the device loop now, re-raise below
            err_box.append(exc)
            return 1

    cb = _lib.TRACE_FN(_cb) if trace is not None else _lib.TRACE_FN()
    rc = _lib.lib().hcub_integrate(_lib.current_device(), C.byref(rd), C.byref(fd), _lib.dptr(dlo),
                                   _lib.dptr(dhi), _lib.dptr(lo0), _lib.dptr(hi0), k, C.byref(cd), int(capacity),
                                   cb, None, C.byref(res))
    if err_box:  # the reference propagates a trace exception immediately
        raise err_box[0]
    _lib.check(rc)
    if stats is not None:
        stats.update(device_ms=res.device_ms, k1_ms=res.k1_ms, k2_ms=res.k2_ms, k3_ms=res.k3_ms,
                     k1_launches=res.k1_launches, launches=res.launches, capacity_limited=bool(res.capacity_limited))
    return IntegrationResult(
        integral=res.integral, error=res.error, converged=bool(res.converged), iterations=int(res.iterations),
        total_f_evals=int(res.total_f_evals), peak_regions=int(res.peak_regions),
        termination_reason=_REASON[res.termination_reason])
