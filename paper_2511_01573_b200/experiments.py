"""Benchmark sweeps on the B200 backend (ref pkg/src/hcub/experiments.py).

Same sweep definition (`ExperimentSpec`, ref :45-83), CSV schemas
(ACCURACY/SCALING/IDLE_COLUMNS, ref :86-118) and manifest (ref :303-314) as
the reference, so downstream tooling reads either.  Every run goes through
`run_distributed` on device stores; on `deterministic_sim` the time columns
are the reference's virtual units, on `concurrent`/`nccl` seconds.
"""

from __future__ import annotations

import csv
import dataclasses
import json
from dataclasses import dataclass
from datetime import datetime, timezone
from pathlib import Path

from .distributed import BACKENDS, RedistributionConfig, run_distributed
from .driver import DriverConfig
from .integrands import FUNCTION_IDS, make_integrand
from .regions import HyperRect
from .rules import UnsupportedDimensionError

__all__ = ["SpecError", "ExperimentSpec", "ACCURACY_COLUMNS", "SCALING_COLUMNS", "IDLE_COLUMNS",
           "run_accuracy_sweep", "run_scaling_sweep", "run_idle_breakdown", "write_rows", "write_manifest"]


class SpecError(ValueError):
    """The sweep definition itself is unusable."""


@dataclass(frozen=True)
class ExperimentSpec:
    functions: tuple
    dims: tuple
    tolerances: tuple
    workers: tuple = (1,)
    rule: str = "gm"
    backend: str = "deterministic_sim"
    repetitions: int = 1
    seed: int = 0
    output_path: str = "results.csv"
    cap: int = 512
    init_per_rank: int = 8
    max_iterations: int = 1000

    def __post_init__(self):
        if not (self.functions and self.dims and self.tolerances and self.workers):
            raise SpecError("every sweep axis needs at least one entry")
        unknown = [f for f in self.functions if f not in FUNCTION_IDS]
        if unknown:
            raise SpecError(f"unknown functions {unknown}; valid ids are {list(FUNCTION_IDS)}")
        if min(self.dims) < 1:
            raise SpecError("dimensions must be >= 1")
        if not all(t > 0 for t in self.tolerances):
            raise SpecError("tolerances must be positive")
        if min(self.workers) < 1:
            raise SpecError("worker counts must be >= 1")
        if self.repetitions < 1:
            raise SpecError("repetitions must be >= 1")
        if self.backend not in BACKENDS:
            raise SpecError(f"unknown backend {self.backend!r}; expected one of {BACKENDS}")
        if self.rule not in ("gm", "gk-tensor", "gm9"):  # gm9: B200 extra (rule9.py)
            raise SpecError(f"unknown rule {self.rule!r}")


_CFG_TAIL = ["rule", "backend", "cap", "init_per_rank", "repetition", "seed"]
ACCURACY_COLUMNS = ["function", "d", "tau_rel", "I", "eps", "rel_error_vs_exact", "iterations", "f_evals",
                    "wall_or_virtual_time", "termination_reason", "workers"] + _CFG_TAIL
SCALING_COLUMNS = ["function", "d", "tau_rel", "P", "time", "iterations", "regions_transferred", "messages",
                   "termination_reason"] + _CFG_TAIL
IDLE_COLUMNS = ["function", "d", "tau_rel", "P", "rank", "compute_fraction", "idle_fraction"] + _CFG_TAIL


def _grid(spec: ExperimentSpec):
    for fid in spec.functions:
        for d in spec.dims:
            for tau in spec.tolerances:
                for workers in spec.workers:
                    for rep in range(spec.repetitions):
                        yield fid, d, tau, workers, rep


def _tail(spec: ExperimentSpec, rep: int) -> dict:
    return {"rule": spec.rule, "backend": spec.backend, "cap": spec.cap, "init_per_rank": spec.init_per_rank,
            "repetition": rep, "seed": spec.seed}


def _execute(spec: ExperimentSpec, fid: str, d: int, tau: float, workers: int):
    """One engine run (ref :133-144); raises UnsupportedDimensionError for
    configurations without a rule."""
    f = make_integrand(fid, d)
    cfg = DriverConfig(tau_rel=tau, rule=spec.rule, max_iterations=spec.max_iterations)
    rcfg = RedistributionConfig(cap=spec.cap, initial_subdomains_per_rank=spec.init_per_rank)
    try:
        run = run_distributed(f, HyperRect.unit_cube(d), cfg, rcfg, workers=workers, backend=spec.backend)
    except NotImplementedError as exc:  # rule tables without a device kernel count as unsupported
        raise UnsupportedDimensionError(str(exc)) from exc
    return f, run


def _elapsed(run) -> float:
    return max((t.compute_seconds + t.idle_seconds for t in run.timings), default=0.0)


def run_accuracy_sweep(spec: ExperimentSpec) -> list[dict]:
    rows = []
    for fid, d, tau, workers, rep in _grid(spec):
        row = {"function": fid, "d": d, "tau_rel": tau, "workers": workers} | _tail(spec, rep)
        try:
            f, run = _execute(spec, fid, d, tau, workers)
        except UnsupportedDimensionError:
            rows.append(row | dict.fromkeys(["I", "eps", "rel_error_vs_exact", "iterations", "f_evals",
                                             "wall_or_virtual_time"], "") | {"termination_reason": "unsupported"})
            continue
        r = run.result
        rows.append(row | {"I": r.integral, "eps": r.error,
                           "rel_error_vs_exact": abs(r.integral - f.reference_value) / abs(f.reference_value),
                           "iterations": r.iterations, "f_evals": r.total_f_evals,
                           "wall_or_virtual_time": _elapsed(run), "termination_reason": r.termination_reason.value})
    return rows


def run_scaling_sweep(spec: ExperimentSpec) -> list[dict]:
    rows = []
    for fid, d, tau, workers, rep in _grid(spec):
        row = {"function": fid, "d": d, "tau_rel": tau, "P": workers} | _tail(spec, rep)
        try:
            _, run = _execute(spec, fid, d, tau, workers)
        except UnsupportedDimensionError:
            rows.append(row | dict.fromkeys(["time", "iterations", "regions_transferred", "messages"], "")
                        | {"termination_reason": "unsupported"})
            continue
        rows.append(row | {"time": _elapsed(run), "iterations": run.result.iterations,
                           "regions_transferred": run.regions_transferred_total, "messages": run.messages_total,
                           "termination_reason": run.result.termination_reason.value})
    return rows


def run_idle_breakdown(spec: ExperimentSpec) -> list[dict]:
    rows = []
    for fid, d, tau, workers, rep in _grid(spec):
        _, run = _execute(spec, fid, d, tau, workers)
        total = _elapsed(run) or 1.0
        for t in run.timings:
            rows.append({"function": fid, "d": d, "tau_rel": tau, "P": workers, "rank": t.rank,
                         "compute_fraction": t.compute_seconds / total, "idle_fraction": t.idle_seconds / total}
                        | _tail(spec, rep))
    return rows


def _cell(x) -> str:
    return repr(x) if isinstance(x, float) else str(x)


def write_rows(rows: list[dict], columns: list[str], path) -> Path:
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(columns)
        for row in rows:
            w.writerow([_cell(row[c]) for c in columns])
    return path


def write_manifest(spec: ExperimentSpec, path) -> Path:
    from . import __version__

    path = Path(path)
    out = path.with_suffix(path.suffix + ".manifest.json")
    out.parent.mkdir(parents=True, exist_ok=True)
    out.write_text(json.dumps({"spec": dataclasses.asdict(spec), "engine_version": __version__,
                               "backend": spec.backend, "created": datetime.now(timezone.utc).isoformat()},
                              indent=2) + "\n", encoding="utf-8")
    return out
