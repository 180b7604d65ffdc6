"""Experiments / CLI surface (ref experiments.py, cli.py): spec validation,
CSV schema, exit codes - CPU; sweeps against the reference's CSVs - GPU."""
import csv
import math
import os

import pytest

from conftest import GOLDEN

import paper_2511_01573_b200 as hb
from paper_2511_01573_b200 import cli, experiments as ex


def test_spec_validation():
    with pytest.raises(ex.SpecError):
        ex.ExperimentSpec(functions=("f9",), dims=(3,), tolerances=(1e-3,))
    with pytest.raises(ex.SpecError):
        ex.ExperimentSpec(functions=("f1",), dims=(3,), tolerances=(0.0,))
    with pytest.raises(ex.SpecError):
        ex.ExperimentSpec(functions=("f1",), dims=(3,), tolerances=(1e-3,), backend="mpi")
    ex.ExperimentSpec(functions=("f1",), dims=(3,), tolerances=(1e-3,), workers=(1, 2))


def test_columns_match_reference_schema():
    for name, cols in (("accuracy_f4_d3", ex.ACCURACY_COLUMNS), ("scaling_f2_d3", ex.SCALING_COLUMNS),
                       ("idle_f6_d3", ex.IDLE_COLUMNS)):
        with open(os.path.join(GOLDEN, f"sweep_{name}.csv")) as fh:
            assert next(csv.reader(fh)) == cols


def test_cli_bad_spec_exit_code(tmp_path):
    assert cli.main(["accuracy", "--function", "f1", "--dim", "0", "--tol-exp-range", "3",
                     "--out", str(tmp_path / "x.csv"), "--no-plot"]) == cli.EXIT_BAD_SPEC
    assert cli._tol_range("3:5") == (1e-3, 1e-4, 1e-5)
    assert cli._tol_range("2:6:2") == (1e-2, 1e-4, 1e-6)


def _read(path):
    with open(path) as fh:
        return list(csv.DictReader(fh))


@pytest.mark.gpu
@pytest.mark.parametrize("kind,name", [("accuracy", "accuracy_f4_d3"), ("scaling", "scaling_f2_d3"),
                                        ("idle", "idle_f6_d3")])
def test_sweeps_match_reference_csv(tmp_path, kind, name):
    ref = _read(os.path.join(GOLDEN, f"sweep_{name}.csv"))
    fn, d = ref[0]["function"], int(ref[0]["d"])
    tols = sorted({float(r["tau_rel"]) for r in ref}, reverse=True)
    workers = sorted({int(r.get("workers") or r.get("P")) for r in ref})
    exps = [round(-math.log10(t)) for t in tols]
    rng = f"{exps[0]}:{exps[-1]}" if len(exps) > 1 else str(exps[0])
    out = tmp_path / "out.csv"
    rc = cli.main([kind, "--function", fn, "--dim", str(d), "--tol-exp-range", rng,
                   "--workers", ",".join(map(str, workers)), "--out", str(out), "--no-plot"])
    assert rc == 0
    mine = _read(out)
    assert len(mine) == len(ref)
    for a, b in zip(mine, ref):
        for k in b:
            if k in ("I", "eps", "compute_fraction", "idle_fraction"):
                assert math.isclose(float(a[k]), float(b[k]), rel_tol=1e-9, abs_tol=1e-300), (k, a[k], b[k])
            elif k == "rel_error_vs_exact":  # |I - exact|/|exact| magnifies last-bit differences of I
                assert abs(float(a[k]) - float(b[k])) < 1e-12, (k, a[k], b[k])
            else:
                assert a[k] == b[k], (k, a[k], b[k])
