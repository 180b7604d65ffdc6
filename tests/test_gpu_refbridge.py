"""The reference package itself, unmodified apart from the `b200` backend
INTEGRATION.md section 2 documents, driving the B200 engine: its CLI
(`hcub integrate --backend b200`, ref cli.py:121-152), `integrate` through
`hcub.b200.integrate_b200`, and `run_distributed(backend="b200")` with the
reference's own integrand objects (the bare `evaluate` lambdas, a
make_product_peak closure).  Results equal this package's and the
reference's own goldens."""
import json
import os
import subprocess
import sys

import pytest

from refstage import ROOT, reference_source, stage

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(reference_source() is None, reason="reference package not staged (baseline/_ref)")]

RUN = r'''
import contextlib, io, json, sys
import hcub
import hcub.cli
from hcub.distributed import run_distributed
import paper_2511_01573_b200 as hb
out = {}
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    rc = hcub.cli.main(["integrate", "--function", "f4", "--dim", "3", "--tol", "1e-6", "--workers", "2",
                        "--backend", "b200"])
out["cli_rc"] = rc
out["cli"] = dict(line.split(None, 1) for line in buf.getvalue().splitlines() if line.startswith(("integral", "iterations", "integrand", "termination")))
mine = hb.run_distributed(hb.make_integrand("f4", 3), hb.HyperRect.unit_cube(3), hb.DriverConfig(1e-6), workers=2,
                          backend="concurrent")
out["mine_cli"] = [repr(mine.result.integral), mine.result.iterations, mine.result.total_f_evals]
tr = []
r = hcub.b200.integrate_b200(hcub.make_integrand("f2", 5).evaluate, hcub.HyperRect.unit_cube(5),
                             hcub.DriverConfig(1e-6, max_iterations=14), trace=tr.append)
out["integrate"] = [type(r).__module__, r.termination_reason.value, r.iterations, r.total_f_evals, r.integral,
                    r.error, r.peak_regions, type(tr[0]).__module__,
                    [[t.iteration, t.active_regions, t.integral, t.error, t.f_evals] for t in tr]]
ev, _ = hcub.make_product_peak(4, center=0.1)
dr = run_distributed(ev, hcub.HyperRect.unit_cube(4), hcub.DriverConfig(1e-6), hcub.RedistributionConfig(),
                     workers=4, backend="b200", collect_log=True)
res = dr.result
out["dist"] = [type(dr).__module__, res.termination_reason.value, res.iterations, res.total_f_evals, res.integral,
               res.error, dr.messages_total, dr.regions_transferred_total, len(dr.timings), len(dr.iteration_log)]
try:
    run_distributed(lambda x: x.sum(1), hcub.HyperRect.unit_cube(2), hcub.DriverConfig(1e-3), backend="b200")
    out["lambda"] = "accepted"
except TypeError:
    out["lambda"] = "TypeError"
print(json.dumps(out))
'''


def _rel(a, b):
    return abs(a - b) / abs(b)


def test_reference_package_runs_on_b200_backend(tmp_path):
    stage(str(tmp_path))
    env = dict(os.environ, PYTHONPATH=f"{tmp_path}{os.pathsep}{ROOT}", PYTHONDONTWRITEBYTECODE="1")
    p = subprocess.run([sys.executable, "-c", RUN], env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    out = json.loads(p.stdout.strip().splitlines()[-1])
    gold = lambda n: json.load(open(os.path.join(ROOT, "tests", "golden", n)))  # noqa: E731

    # CLI (ref cli.py:121-152) on the b200 backend = this package's engine = the reference's log
    assert out["cli_rc"] == 0
    assert out["cli"]["integral"] == out["mine_cli"][0]
    assert int(out["cli"]["iterations"]) == out["mine_cli"][1]
    g = gold("dist_f4_d3_P2.json")["result"]
    assert out["mine_cli"][1] == g["iterations"] and out["mine_cli"][2] == g["total_f_evals"]
    assert _rel(float(out["cli"]["integral"]), g["integral"]) <= 1e-12

    # integrate_b200 with the bare f2 lambda vs the reference's own trace (ref driver.py:237-323)
    mod, reason, its, evals, I, E, peak, trmod, trace = out["integrate"]
    g = gold("trace_f2_d5.json")
    assert mod == "hcub.driver" and trmod == "hcub.driver"
    assert (reason, its, evals, peak) == (g["result"]["termination_reason"], g["result"]["iterations"],
                                         g["result"]["total_f_evals"], g["result"]["peak_regions"])
    assert _rel(I, g["result"]["integral"]) <= 1e-12 and _rel(E, g["result"]["error"]) <= 1e-12
    for a, b in zip(trace, g["trace"]):
        assert a[0] == b[0] and a[1] == b[1] and a[4] == b[4]
        assert _rel(a[2], b[2]) <= 1e-12 and _rel(a[3], b[3]) <= 1e-12

    # run_distributed(backend="b200") with a make_product_peak closure vs the reference's log
    mod, reason, its, evals, I, E, msgs, moved, ntim, nlog = out["dist"]
    g = gold("dist_pp_d4_c01_P4.json")
    assert mod == "hcub.distributed"
    assert (reason, its, evals) == (g["result"]["termination_reason"], g["result"]["iterations"],
                                    g["result"]["total_f_evals"])
    assert (msgs, moved) == (g["messages_total"], g["regions_transferred_total"])
    assert ntim == 4 and nlog == len(g["log"])
    # the settled error sums |main - emb|-dominated estimates whose BLAS-order cancellation the
    # device does not reproduce: 1e-9, as in test_gpu_distributed
    assert _rel(I, g["result"]["integral"]) <= 1e-12 and _rel(E, g["result"]["error"]) <= 1e-9
    assert out["lambda"] == "TypeError"
