"""The reference package's own objects -> the B200 engine, and back.

This is what a ``"b200"`` backend registered inside the reference calls
(INTEGRATION.md section 2): the reference passes its own ``DriverConfig``,
``RedistributionConfig``, ``HyperRect`` and - from its CLI and experiment
runner - the bare ``BenchmarkIntegrand.evaluate`` lambda
(ref cli.py:126-134, experiments.py:136-143).  The kernels cannot call a
Python lambda per node, so the integrand is identified:

  * an object with ``id`` / ``d`` (the reference's or this package's
    ``BenchmarkIntegrand``, ref integrands.py:35-46) -> ``make_integrand``;
  * the evaluator lambda of ``_EVALUATORS[id](d)`` (ref integrands.py:53-99;
    qualname ``_f<k>.<locals>.<lambda>`` or ``.evaluate``) -> ``make_integrand(f<k>, d)``;
  * the ``evaluate`` closure of ``make_product_peak`` (ref integrands.py:194-210)
    -> a device product peak with the closure's own ``a`` and center (bit-equal
    constants, not re-derived from the sharpness);
  * this package's integrand objects pass through.

Anything else raises ``TypeError`` (no CPU fallback).  Results come back as
the reference module's own dataclasses (``IntegrationResult``,
``IterationTrace``, ``TimeBreakdown``, ``DistributedResult``).
"""

from __future__ import annotations

import functools
import math
import re

import numpy as np

from . import distributed as _dist
from . import driver as _drv
from .integrands import BenchmarkIntegrand, ProductPeak, make_integrand
from .regions import HyperRect

_LAMBDA = re.compile(r"^_(f[1-7])\.<locals>\.(<lambda>|evaluate)$")


def _closure(fn) -> dict:
    cells = getattr(fn, "__closure__", None) or ()
    return dict(zip(fn.__code__.co_freevars, (c.cell_contents for c in cells)))


def to_integrand(f, d: int):
    """Device integrand for one of the reference's integrand objects."""
    if isinstance(f, (BenchmarkIntegrand, ProductPeak)):
        return f
    fid, fd = getattr(f, "id", None), getattr(f, "d", None)
    if isinstance(fid, str) and isinstance(fd, int):  # ref BenchmarkIntegrand
        if fd != d:
            raise ValueError(f"integrand is for d={fd}, domain has d={d}")
        return make_integrand(fid, d)
    qn = getattr(f, "__qualname__", "")
    m = _LAMBDA.match(qn)
    if m and getattr(f, "__module__", "").endswith("integrands"):
        return make_integrand(m.group(1), d)
    if qn == "make_product_peak.<locals>.evaluate" and getattr(f, "__module__", "").endswith("integrands"):
        cl = _closure(f)
        a, c = float(cl["a"]), np.asarray(cl["c"], dtype=np.float64)
        if c.shape != (d,):
            raise ValueError(f"product peak center has shape {c.shape}, domain has d={d}")
        pp = ProductPeak(d, c, 1.0 / math.sqrt(a))
        pp.a = a  # the closure's constant itself (ref :202), not 1/sharpness^2 recomputed
        return pp
    raise TypeError(
        "the b200 backend evaluates integrands on the device: pass a BenchmarkIntegrand, its "
        "`evaluate`, or a make_product_peak evaluator (got " + (qn or type(f).__name__) + ")")


def to_domain(domain) -> HyperRect:
    return HyperRect(np.asarray(domain.lo, dtype=np.float64), np.asarray(domain.hi, dtype=np.float64))


def to_config(cfg) -> _drv.DriverConfig:
    """ref DriverConfig (driver.py:79-102) -> this package's."""
    cl = cfg.classifier
    if type(cl).__name__ != "VolumeBudgetClassifier" or not hasattr(cl, "safety"):
        raise TypeError("the device classifier implements VolumeBudgetClassifier(safety) only")
    return _drv.DriverConfig(tau_rel=cfg.tau_rel, abs_floor=cfg.abs_floor, max_iterations=cfg.max_iterations,
                             max_regions=cfg.max_regions, min_width_ulp_factor=cfg.min_width_ulp_factor,
                             rule=cfg.rule, classifier=_drv.VolumeBudgetClassifier(cl.safety))


def to_rcfg(rcfg) -> _dist.RedistributionConfig | None:
    """ref RedistributionConfig (distributed.py:77-103) -> this package's."""
    if rcfg is None:
        return None
    return _dist.RedistributionConfig(
        cap=rcfg.cap, initial_subdomains_per_rank=rcfg.initial_subdomains_per_rank, policy=rcfg.policy,
        delivery_latency=rcfg.delivery_latency, max_unacked_iterations=rcfg.max_unacked_iterations,
        msg_fixed_cost=rcfg.msg_fixed_cost, msg_cost_per_region=rcfg.msg_cost_per_region)


def to_ref_result(res, ref):
    return ref.IntegrationResult(res.integral, res.error, bool(res.converged), int(res.iterations),
                                 int(res.total_f_evals), int(res.peak_regions),
                                 ref.TerminationReason(res.termination_reason.value))


def integrate(f, domain, cfg, trace=None, initial_regions=None, *, ref):
    """ref driver.integrate (driver.py:237-243) on the device."""
    d = len(domain.lo)
    sink = None
    if trace is not None:
        def sink(t):
            trace(ref.IterationTrace(t.iteration, t.active_regions, t.integral, t.error, t.f_evals))
    r = _drv.integrate(to_integrand(f, d), to_domain(domain), to_config(cfg), trace=sink,
                       initial_regions=initial_regions)
    return to_ref_result(r, ref)


def run_distributed(f, domain, cfg, rcfg=None, workers: int = 1, backend: str = "b200", collect_log: bool = False,
                    *, ref):
    """ref distributed.run_distributed (distributed.py:854-877) for backend
    "b200": this package's threaded engine, one device worker per rank (rank r
    on visible device r mod count), returning the reference's dataclasses."""
    d = len(domain.lo)
    dr = _dist.run_distributed(to_integrand(f, d), to_domain(domain), to_config(cfg), to_rcfg(rcfg),
                               workers=workers, backend="concurrent", collect_log=collect_log)
    timings = [ref.TimeBreakdown(t.rank, t.iterations, t.compute_seconds, t.idle_seconds, t.messages_out,
                                 t.regions_out) for t in dr.timings]
    return ref.DistributedResult(to_ref_result(dr.result, ref), timings, dr.messages_total,
                                 dr.regions_transferred_total, dr.final_reduce_integral, dr.final_reduce_error,
                                 dr.iteration_log)


def bind(ref_package):
    """(integrate, run_distributed) taking and returning the objects of the
    imported reference package ``ref_package`` (the ``hcub`` module)."""
    return (functools.partial(integrate, ref=ref_package), functools.partial(run_distributed, ref=ref_package))
