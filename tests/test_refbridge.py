"""The reference-side `b200` backend on CPU:
the documented stub applies to an unmodified copy of the reference, and the
bridge identifies the reference's own integrand objects, configs and
domains (no device calls here; tests/test_gpu_refbridge.py runs them)."""
import json
import os
import subprocess
import sys

import pytest

from refstage import ROOT, reference_source, stage

pytestmark = pytest.mark.skipif(reference_source() is None, reason="reference package not staged")

CHECK = r'''
import json, sys
import numpy as np
import hcub
from hcub import distributed as D
from paper_2511_01573_b200 import refbridge as rb
import paper_2511_01573_b200 as hb
out = {"backends": list(D.BACKENDS), "b200_file": hcub.b200.__name__ if hasattr(hcub, "b200") else None}
import hcub.b200
out["bound"] = [hcub.b200.integrate_b200.func.__name__, hcub.b200.run_distributed_b200.func.__name__]
ids = {}
for fid in ("f1", "f2", "f3", "f4", "f5", "f6", "f7"):
    g = rb.to_integrand(hcub.make_integrand(fid, 4).evaluate, 4)
    ids[fid] = [g.id, g.d]
    assert rb.to_integrand(hcub.make_integrand(fid, 4), 4) is g
out["ids"] = ids
ev, exact = hcub.make_product_peak(3, center=[0.1, 0.2, 0.3], sharpness=37.0)
pp = rb.to_integrand(ev, 3)
out["pp"] = [pp.a == 1.0 / 37.0 ** 2, pp.center.tolist()]
try:
    rb.to_integrand(lambda x: x.sum(1), 3)
    out["lambda"] = "accepted"
except TypeError:
    out["lambda"] = "TypeError"
cfg = rb.to_config(hcub.DriverConfig(1e-5, max_iterations=7, max_regions=99, abs_floor=1e-12,
                                     min_width_ulp_factor=4.0, classifier=hcub.VolumeBudgetClassifier(0.25)))
out["cfg"] = [cfg.tau_rel, cfg.max_iterations, cfg.max_regions, cfg.abs_floor, cfg.min_width_ulp_factor,
              cfg.classifier.safety, type(cfg).__module__]
rc = rb.to_rcfg(hcub.RedistributionConfig(cap=16, initial_subdomains_per_rank=3, delivery_latency=2))
out["rcfg"] = [rc.cap, rc.initial_subdomains_per_rank, rc.delivery_latency]
dom = rb.to_domain(hcub.HyperRect.unit_cube(3))
out["dom"] = [dom.lo.tolist(), dom.hi.tolist()]
print(json.dumps(out))
'''


def test_stub_applies_and_bridge_identifies_reference_objects(tmp_path):
    stage(str(tmp_path))
    env = dict(os.environ, PYTHONPATH=f"{tmp_path}{os.pathsep}{ROOT}", PYTHONDONTWRITEBYTECODE="1")
    p = subprocess.run([sys.executable, "-c", CHECK], env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-3000:]
    out = json.loads(p.stdout.strip().splitlines()[-1])
    assert out["backends"] == ["deterministic_sim", "concurrent", "b200"]
    assert out["bound"] == ["integrate", "run_distributed"]
    assert out["ids"] == {f"f{k}": [f"f{k}", 4] for k in range(1, 8)}
    assert out["pp"] == [True, [0.1, 0.2, 0.3]]
    assert out["lambda"] == "TypeError"
    assert out["cfg"] == [1e-5, 7, 99, 1e-12, 4.0, 0.25, "paper_2511_01573_b200.driver"]
    assert out["rcfg"] == [16, 3, 2]
    assert out["dom"] == [[0.0] * 3, [1.0] * 3]
